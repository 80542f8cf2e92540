// Grid-barrier latency probe: the engine's single-word flip barrier (thread 0 arrives and polls)
// against variants with several staggered pollers per CTA.  592 CTAs x 256 threads (the remedy's
// grid), back-to-back barriers.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bp barrier_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned atom_add_acq_rel_gpu(unsigned *a, unsigned v)
{
    unsigned old;
    asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(old) : "l"(a), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_acquire_gpu(const unsigned *a)
{
    unsigned v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory");
    return v;
}

template <int NP, int SPIN, int STAG>
__global__ void k(unsigned *bar, int iters, unsigned *sink)
{
    __shared__ unsigned s_old;
    __shared__ volatile unsigned s_done;
    if (threadIdx.x == 0) {
        s_old = 0;
        s_done = 0;
    }
    unsigned acc = 0;
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        if (threadIdx.x == 0) {
            const unsigned add = blockIdx.x == 0 ? 0x80000000u - (gridDim.x - 1u) : 1u;
            s_old = atom_add_acq_rel_gpu(bar, add) | 1u;  // |1: never 0 (armed marker below)
        }
        if (NP == 1) {
            if (threadIdx.x == 0) {
                const unsigned old = s_old;
                while (((old ^ ld_acquire_gpu(bar)) & 0x80000000u) == 0u)
                    if (SPIN) __nanosleep(SPIN);
            }
        } else if ((threadIdx.x & 31) == 0 && (threadIdx.x >> 5) < NP) {
            const unsigned w = threadIdx.x >> 5;
            unsigned old;
            while ((old = *(volatile unsigned *)&s_old) == 0u) {
            }
            if (w) __nanosleep(w * STAG);
            while (!s_done) {
                if (((old ^ ld_acquire_gpu(bar)) & 0x80000000u) != 0u) {
                    s_done = 1;
                    break;
                }
                if (SPIN) __nanosleep(SPIN);
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_old = 0;
            s_done = 0;
        }
        acc += threadIdx.x;
    }
    if (acc == 0xffffffffu) *sink = acc;
}

template <int NP, int SPIN, int STAG>
void run(const char *name, unsigned *bar, unsigned *sink)
{
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    void *args1[] = {&bar, nullptr, &sink};
    int w = 20, n = 2000;
    args1[1] = &w;
    cudaLaunchCooperativeKernel((const void *)k<NP, SPIN, STAG>, 592, 256, args1, 0, 0);
    cudaEventRecord(a);
    args1[1] = &n;
    cudaLaunchCooperativeKernel((const void *)k<NP, SPIN, STAG>, 592, 256, args1, 0, 0);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    printf("%-40s %.3f us per barrier  (%s)\n", name, ms * 1e3 / n, cudaGetErrorString(cudaGetLastError()));
}

int main()
{
    unsigned *bar, *sink;
    cudaMalloc(&bar, 256);
    cudaMalloc(&sink, 4);
    cudaMemset(bar, 0, 256);
    for (int rep = 0; rep < 2; ++rep) {
        run<1, 32, 0>("1 poller, nanosleep 32 (engine)", bar, sink);
        run<1, 0, 0>("1 poller, no sleep", bar, sink);
        run<2, 32, 150>("2 pollers, stagger 150 ns", bar, sink);
        run<4, 32, 100>("4 pollers, stagger 100 ns", bar, sink);
        run<4, 0, 100>("4 pollers, stagger 100 ns, no sleep", bar, sink);
        run<8, 32, 60>("8 pollers, stagger 60 ns", bar, sink);
    }
    return 0;
}
