// Same-address atomicAdd (with return) from every CTA vs per-group addresses: the cost of the
// remedy's per-CTA list reservation.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ac atom_contention.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k(unsigned *ctr, int stride_groups, int iters, unsigned long long *t_out)
{
    __shared__ unsigned s;
    unsigned long long t0, t1;
    for (int it = 0; it < iters; ++it) {
        __syncthreads();
        if (threadIdx.x == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
            unsigned *a = ctr + (stride_groups ? (blockIdx.x / stride_groups) * 32 : 0);
            s = atomicAdd(a, 1u + (threadIdx.x & 1));
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
            atomicAdd(t_out, t1 - t0);
        }
        __syncthreads();
        if (s == 0xffffffffu) t_out[1] = 1;
    }
}

int main()
{
    unsigned *ctr;
    unsigned long long *t;
    cudaMalloc(&ctr, 4096 * 4);
    cudaMalloc(&t, 16);
    for (int g : {0, 64, 32, 16, 8, 1}) {
        cudaMemset(ctr, 0, 4096 * 4);
        cudaMemset(t, 0, 16);
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        k<<<592, 256>>>(ctr, g, 10, t);
        cudaEventRecord(a);
        k<<<592, 256>>>(ctr, g, 100, t);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        unsigned long long h[2];
        cudaMemcpy(h, t, 16, cudaMemcpyDeviceToHost);
        printf("group %3d: %.3f us per round (kernel), mean atomic latency %.1f ns\n", g, ms * 1e3 / 100,
               (double)h[0] / (592.0 * 110));
    }
    return 0;
}
