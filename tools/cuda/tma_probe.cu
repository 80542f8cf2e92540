// TMA mechanics probe (design tool): a 3D float64 box with a halo (negative start coordinates,
// zero fill outside), a 1D bulk copy, mbarrier expect_tx/try_wait, tensor map passed as a
// __grid_constant__ parameter after a large by-value struct (like the engine's KP).
// nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o /tmp/tma_probe tools/cuda/tma_probe.cu
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

struct Big {
    char pad[616];
};

__device__ __forceinline__ unsigned sa(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }

#ifndef V_GLOBAL_MAP
#define V_GLOBAL_MAP 0
#endif
#ifndef V_TMA
#define V_TMA 1
#endif
#ifndef V_BULK
#define V_BULK 1
#endif
#ifndef V_ORIGIN
#define V_ORIGIN -1
#endif
#ifndef V_OX
#define V_OX V_ORIGIN
#endif
#ifndef V_BW
#define V_BW 34
#endif
#ifndef V_INITFENCE
#define V_INITFENCE 1
#endif
__global__ void probe(Big big, const unsigned *flag, const __grid_constant__ CUtensorMap tmp, const CUtensorMap *tmg,
                      const double *src, double *out, int *status)
{
    const CUtensorMap *tmx = V_GLOBAL_MAP ? tmg : &tmp;
    extern __shared__ __align__(1024) unsigned char raw[];
    unsigned char *sm = raw + ((1024u - (sa(raw) & 1023u)) & 1023u);
    double *box = (double *)sm;
    double *lin = (double *)(sm + 29696);
    unsigned long long *bar = (unsigned long long *)(sm + 29696 + 512);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(bar)), "r"(1) : "memory");
        if (V_INITFENCE) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned tx = (V_TMA ? V_BW * 10 * 10 * 8 : 0) + (V_BULK ? 256 : 0);
        asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(bar)), "r"(tx) : "memory");
        if (V_TMA) asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
            ::"r"(sa(box)), "l"(tmx), "r"(V_OX), "r"(V_ORIGIN), "r"(V_ORIGIN), "r"(sa(bar))
            : "memory");
        if (V_BULK) asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"(sa(lin)), "l"(src + 64), "r"(256), "r"(sa(bar))
                     : "memory");
    }
    unsigned ok = 0;
    while (!ok) {
        asm volatile(
            "{\n .reg .pred q;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%1], %2;\n"
            " selp.u32 %0, 1, 0, q;\n}"
            : "=r"(ok)
            : "r"(sa(bar)), "r"(0)
            : "memory");
    }
    for (int i = threadIdx.x; i < V_BW * 100; i += blockDim.x) out[i] = box[i];
    for (int i = threadIdx.x; i < 32; i += blockDim.x) out[3700 + i] = lin[i];
    if (threadIdx.x == 0) *status = 1 + big.pad[0] + (flag ? 0 : 0);
}

int main()
{
    const int nx = 64, ny = 16, nz = 16, n = nx * ny * nz;
    std::vector<double> h(n);
    for (int i = 0; i < n; ++i) h[i] = i + 1;
    double *d, *o;
    int *st;
    cudaMalloc(&d, n * 8);
    cudaMalloc(&o, 4096 * 8);
    cudaMalloc(&st, 4);
    cudaMemcpy(d, h.data(), n * 8, cudaMemcpyHostToDevice);
    cudaMemset(st, 0, 4);
    void *f = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    CUtensorMap tm;
    const cuuint64_t dims[3] = {nx, ny, nz}, strides[2] = {nx * 8, nx * ny * 8};
    const cuuint32_t box[3] = {V_BW, 10, 10}, es[3] = {1, 1, 1};
    CUresult r = ((PFN_cuTensorMapEncodeTiled_v12000)f)(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, es,
                                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d\n", (int)r);
    Big big{};
    const int smem = 29696 + 512 + 64 + 1024;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    CUtensorMap *tg;
    cudaMalloc(&tg, sizeof(CUtensorMap));
    cudaMemcpy(tg, &tm, sizeof(CUtensorMap), cudaMemcpyHostToDevice);
    probe<<<1, 128, smem>>>(big, nullptr, tm, tg, d, o, st);
    cudaError_t e = cudaDeviceSynchronize();
    printf("kernel: %s\n", cudaGetErrorString(e));
    std::vector<double> got(3732);
    cudaMemcpy(got.data(), o, 3732 * 8, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int k = 0; k < 10; ++k)
        for (int j = 0; j < 10; ++j)
            for (int i = 0; i < V_BW; ++i) {
                const int x = i + V_OX, y = j + V_ORIGIN, z = k + V_ORIGIN;
                const double want = (x < 0 || y < 0 || z < 0 || x >= nx) ? 0.0 : h[(z * ny + y) * nx + x];
                if (got[(k * 10 + j) * V_BW + i] != want && bad++ < 5)
                    printf("box (%d,%d,%d) got %g want %g\n", i, j, k, got[(k * 10 + j) * V_BW + i], want);
            }
    if (!V_TMA) bad = 0;
    for (int i = 0; i < 32 && V_BULK; ++i)
        if (got[3700 + i] != h[64 + i] && bad++ < 10) printf("lin %d got %g\n", i, got[3700 + i]);
    printf("TMA_PROBE %s (%d bad)\n", bad ? "FAIL" : "OK", bad);
    return 0;
}
