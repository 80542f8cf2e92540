// Exhaustive-ish check of the FMA form of x / 3.0 used by the 3D local solver
// (div3_rn in eik_ifim.cu) against IEEE division: random bit patterns over the
// finite positive range plus mantissas near every rounding boundary.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -fmad=false -o /tmp/check_div3 tools/cuda/check_div3.cu
#include <cstdio>
#include <cstdint>

__device__ __forceinline__ double div3_rn(double x)
{
    if (!(x >= 0x1p-900) || !(x < INFINITY)) return x / 3.0;
    const double inv3 = 0x1.5555555555555p-2;
    const double q = __dmul_rn(x, inv3);
    const double r = __fma_rn(-q, 3.0, x);
    return __fma_rn(r, inv3, q);
}

__device__ __forceinline__ uint64_t mix(uint64_t z)
{
    z += 0x9e3779b97f4a7c15ull;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

__global__ void k(uint64_t base, uint64_t n, unsigned long long *bad, unsigned long long *first)
{
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t h = mix(base + i);
        uint64_t bits;
        const int mode = (int)(h & 3);
        if (mode == 0) {
            bits = h >> 1;  // any positive finite
        } else if (mode == 1) {  // exponent near 1, random mantissa
            bits = ((uint64_t)(1023 + ((h >> 2) & 63) - 32) << 52) | ((h >> 8) & ((1ull << 52) - 1));
        } else if (mode == 2) {  // integers and multiples of 3 (exact quotients), scaled
            bits = __double_as_longlong((double)((h >> 10) & ((1ull << 53) - 1)) * (double)(1ull << ((h >> 2) & 15)));
        } else {  // mantissas with long runs (rounding-boundary patterns)
            const uint64_t run = ((h >> 8) & 1) ? ((1ull << 52) - 1) : 0ull;
            const uint64_t flip = 1ull << ((h >> 9) & 51);
            bits = ((uint64_t)(1023 + ((h >> 20) & 1023) - 512) << 52) | ((run ^ flip ^ ((h >> 40) & 7)) & ((1ull << 52) - 1));
        }
        const double x = __longlong_as_double((long long)(bits & 0x7fffffffffffffffull));
        if (!(x < INFINITY)) continue;
        const double a = div3_rn(x), b = x / 3.0;
        if (__double_as_longlong(a) != __double_as_longlong(b)) {
            if (atomicAdd(bad, 1ull) == 0) *first = bits;
        }
    }
}

int main()
{
    unsigned long long *d;
    cudaMalloc(&d, 16);
    cudaMemset(d, 0, 16);
    const uint64_t per = 1ull << 32;
    for (int r = 0; r < 8; ++r) k<<<148 * 16, 256>>>((uint64_t)r * per, per, d, d + 1);
    unsigned long long h[2];
    cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
    printf("checked %llu values, mismatches %llu (first bits %llx) %s\n", (unsigned long long)(8 * per), h[0], h[1],
           cudaGetErrorString(cudaGetLastError()));
    return h[0] != 0;
}
