// eik_ifim.cu -- B200 (sm_100a) engine for the improved fast iterative method.
//
// Implements the C ABI declared in include/eik_ifim.h.  The reference path it
// replaces is E/ifim.py (E = /root/reference/pkg/src/eikonal):
//
//   update step  (E/ifim.py:75-134)  -> k_update   persistent, one thread per active cell
//   build pass   (E/ifim.py:137-161) -> k_build    one pass, one warp per bitmap word
//   remedy step  (E/ifim.py:164-218) -> k_remedy   persistent; per round the member list is
//                                                  rebuilt from the decrease bitmap, then one
//                                                  thread per member
//                                     or k_remedy_b (eik_remedy_tma.cuh) TMA brick pipeline for
//                                                  dense remedy sets, chosen on the device from
//                                                  |R_0| (k_choose_remedy)
// plus the fixpoint ground truth (E/oracle.py, k_fixpoint), max_residual
// (E/harness.py, k_residual), the FIM baseline (E/fim.py, k_fim) and the
// multi-rank z-slab variants of the update / remedy kernels (peer memory).
//
// Data layout in HBM:
//   * phi: the caller's array (row-major, x fastest) plus one workspace copy.
//     The two form a Jacobi double buffer: iteration k reads P[k&1]; every
//     processed cell whose value changes, or changed in iteration k-1 (CARRY
//     bit of its list entry), writes P[(k+1)&1].  That keeps the snapshot
//     semantics of padded_phi (E/_kernels.py:21-26) without an O(N) copy per
//     iteration; at termination both buffers are equal.
//   * d = delta / F precomputed per cell (bit-identical to the per-call
//     division at E/_kernels.py:48 and E/local_solver.py:105).
//   * Sets are bitmaps with one 32-bit word per 32 consecutive cells of one
//     x-row (word w <-> row w / W, x = 32*(w % W) + bit); rows are padded to
//     whole words.  Worklists hold cell indices (< 2^31, bit 31 = CARRY).
//
// Arithmetic is IEEE with FMA contraction disabled (-fmad=false) and the
// reference's operation order, so the float64 build is bit-identical to the
// reference: phi and every RunStats integer (iterations, solver_calls, peaks,
// active_history).  The same source compiled with -DEIK_SINGLE=1 is the
// float32 perf mode (names suffixed _f32).
//
// Termination is device-side: the persistent kernels loop over iterations
// with a software grid barrier (co-residency guaranteed by a cooperative
// launch, 10 s watchdog) and read the global set size after each barrier;
// the host sees only the final statistics.

#include <cuda.h>          // CUtensorMap (TMA descriptors)
#include <cudaTypedefs.h>  // PFN_cuTensorMapEncodeTiled
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <string>
#include <vector>

#include "eik_ifim.h"

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: named ranges for nsys / ncu --nvtx

// Field precision: float64 (parity mode, libeik_ifim.so) or float32 (perf mode,
// libeik_ifim_f32.so: -DEIK_SINGLE=1, exported names carry the _f32 suffix).
#ifndef EIK_SINGLE
#define EIK_SINGLE 0
#endif
#if EIK_SINGLE
typedef float real_t;
#define EIK_FN(name) name##_f32
#define EIK_DTYPE EIK_F32
#else
typedef double real_t;
#define EIK_FN(name) name
#define EIK_DTYPE EIK_F64
#endif

namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef EIK_BLOCK
#define EIK_BLOCK 256
#endif
constexpr int BLOCK = EIK_BLOCK;
constexpr int WPB = BLOCK / 32;
constexpr uint8_t ST_SOURCE = 2, ST_BLOCKED = 4;  // E/grid.py:21-26
enum { SOL_U2 = 0, SOL_A2 = 1, SOL_U3 = 2 };

// E/_kernels.py:18 (math.sqrt(2.0)) and E/local_solver.py:28
constexpr real_t kSqrt2 = (real_t)1.4142135623730951;
constexpr real_t DISC_CLAMP = (real_t)1e-12;
constexpr real_t R_HALF = (real_t)0.5, R_ONE = (real_t)1.0, R_TWO = (real_t)2.0, R_THREE = (real_t)3.0, R_ZERO = (real_t)0.0;

// IEEE bits of a non-negative value, ordered like the value (atomicMax reductions)
#if EIK_SINGLE
__device__ __forceinline__ unsigned long long bits_of(float x) { return (unsigned long long)__float_as_uint(x); }
#else
__device__ __forceinline__ unsigned long long bits_of(double x) { return (unsigned long long)__double_as_longlong(x); }
#endif
__device__ __forceinline__ real_t real_of_bits(unsigned long long b)
{
#if EIK_SINGLE
    return __uint_as_float((unsigned)b);
#else
    return __longlong_as_double((long long)b);
#endif
}

struct Ctl {
    unsigned len[3];
    unsigned err;
    unsigned long long cnt[3];
    unsigned long long sum;     // sum of set sizes over iterations (solver calls)
    unsigned long long peak;    // peak set size
    unsigned long long writes;  // phi writes
    unsigned long long conv;    // cells converged (update)
    unsigned long long iters;   // iterations / rounds executed
    unsigned long long free_cells;  // build: #free
    unsigned long long flagged;     // build: |R0|
    unsigned long long dsum[3];     // remedy: |D_r| per rotating slot
    unsigned long long nz_words;    // remedy diagnostics: non-empty member words / 4-cell sectors
    unsigned long long nz_sectors;
    unsigned stale;                 // remedy: a hand-built set has members outside its work list (St)
    unsigned engine;                // remedy: engine chosen on the device (1 member list, 3 brick)
    unsigned wcount;                // multi-rank: world-barrier arrivals (rank 0's copy is used)
    unsigned wgen;                  // multi-rank: this rank's world-barrier generation
    unsigned fc[3];                 // FIM: check-list length per rotating slot
    // grid barrier word on its own 128-byte line (the arrivals and the polls do not share a
    // line with the round counters)
    alignas(128) unsigned bar_count;
    alignas(128) unsigned bar_gen;  // multi-rank release generation
#ifdef EIK_DIAG
    unsigned long long dg[4][26];   // remedy rounds by log2|R_r|: count, phase B ns, phase A ns, members
    unsigned long long dgw[3][5];   // per round slot: max / sum of the CTAs' phase-B work ns, max / min start, max end
    unsigned long long dg2[7][26];  // by log2|R_r|: sum of max-CTA B work, of mean-CTA B work, start skew, barrier tail,
                                    // slowest CTA's members, rounds whose slowest CTA is CTA 0, its traversal share
    unsigned long long dgk[3];      // per round slot: (B work ns << 24) | (members << 10) | CTA of the slowest CTA
    unsigned long long du[3][26];   // update iterations by log2|A_k|: count, ns, cells
    unsigned long long duw[3][2];   // per iteration slot: max / sum of the CTAs' work ns (start -> arrival)
    unsigned long long du2[2][26];  // by log2|A_k|: sum of slowest-CTA work, of mean-CTA work
#endif
};

constexpr int EIK_MAX_RANKS = 16;

// A neighbour rank's buffers, addressable from this device (same GPU, or an
// NVLink peer mapping).  Multi-rank (peer-slab) mode reads its boundary planes
// of phi and of the decrease bitmap directly and activates cells on its
// boundary plane with atomics on its touched bitmap and next worklist.
struct Peer {
    real_t *P0, *P1;
    uint32_t *Bt, *L0, *L1, *D0b, *D1b;
    Ctl *ctl;
    uint32_t nz;     // its owned planes
    uint32_t valid;
};

// Division by a runtime-invariant divisor for dividends < 2^31 (round-up
// multiplier method): q = umulhi(n, mul) >> shr.
struct FastDiv {
    uint32_t d, mul, shr;
};

FastDiv make_fastdiv(uint32_t d)
{
    FastDiv f{d, 0u, 0u};
    if (d <= 1) return f;
    uint32_t l = 0;
    while ((1ull << l) < d) ++l;  // ceil(log2 d)
    const uint32_t p = 31 + l;
    f.mul = (uint32_t)(((1ull << p) + d - 1) / d);
    f.shr = p - 32;
    return f;
}

__device__ __forceinline__ uint32_t fdiv(uint32_t n, const FastDiv &f)
{
    return f.d == 1 ? n : (__umulhi(n, f.mul) >> f.shr);
}

struct KP {
    int64_t nx, ny, nz, plane;
    uint32_t W, nwords, nrows, ncells;  // ncells < 2^31
    uint32_t nx32, plane32;  // cell indices are < 2^31 (make_layout)
    uint32_t npos, nty4;     // remedy member-list traversal: positions (padded bricks), 4-row tiles in y
    FastDiv fnx, fny, fW, fnty4;
    real_t dx, dy, delta, tol;
    int32_t slab;            // 1: z-slab of a sharded 3D grid, planes 0 and nz-1 are ghosts
    int32_t pad1;
    int64_t it0, max_it;     // iteration window of one persistent launch (slab mode: one step)
    real_t *P0, *P1;         // P0 = caller phi, P1 = workspace copy
    const real_t *F;         // speed
    real_t *dd;              // delta / F (uniform solvers)
    uint8_t *lab;            // FIM labels (one byte per cell)
    const uint8_t *state;
    uint32_t *Bt;                 // touched bitmap (update step labels: not FAR)
    uint32_t *L0, *L1;            // update-step cell worklists
    uint32_t *L2;                 // FIM: check list
    Ctl *ctl;
    int64_t *hist;
    int64_t hist_cap;
    int64_t cap;
    // remedy step: row-major bitmaps (one word per 32 cells of an x-row)
    uint32_t *R0b;       // R_0 (build / load)
    uint32_t *D0b, *D1b;  // D_r (decreased cells), double-buffered by round parity
    uint32_t *Fb;        // fixed = blocked | source | outside the row
    // remedy tile engine (k_remedy_t, single device): tile-major bitmaps (one 128-byte line of 32
    // row words per tile), per-tile D stamps by round parity, sharded chunk counters
    uint32_t nty, ntz, ntiles, rt_shs;  // tiles in y / z, tiles, tiles per shard
    FastDiv fnty;
    uint32_t *Ft;                // fixed, tile-major (rows outside the grid: all fixed)
    uint32_t *St;                // hand-built sets: members outside the work list, tile-major
    uint32_t *Dt0, *Dt1;         // D_r, tile-major, by round parity
    uint32_t *stamp0, *stamp1;   // per tile: (round + 1) << 7 | faces of its D_r line, by round parity
    unsigned *grab;              // [3 slots][RT_SHARDS] chunk counters, one 128-byte line each
    // remedy brick engine (k_remedy_b, single device 3D; eik_remedy_tma.cuh): 32 x 8 x 8 bricks,
    // brick-major D records by round parity, fixed words, per-round masks and brick lists
    uint32_t nbx, nby, nbz, nbricks;
    FastDiv fnbx, fnby;
    uint32_t *brec0, *brec1;     // [nbricks][128 words]: own D rows + face summaries
    uint32_t *bfix;              // [nbricks][64 words]: fixed rows (outside the grid: all ones)
    uint32_t *bmask;             // [3 slots][nbricks]: which records a brick reads next round
    uint32_t *blist0, *blist1;   // [nbricks]: active bricks of a round, by parity
    unsigned *bcnt;              // [3 slots] list lengths, [3 slots] grab counters (128-byte lines)
    unsigned *bsel;              // engine selection: [0] skip word of the list kernel, [32] of the brick kernel
    // multi-rank (peer slabs): this rank owns planes [zg0, zg0 + nz) of the global grid
    int32_t mr, q, R, pad2;
    uint32_t gb0, gnb;     // this rank's CTAs: blockIdx.x in [gb0, gb0 + gnb)
    Peer lo, hi;
    Ctl *rank_ctl[EIK_MAX_RANKS];
};



// Remedy tile engine geometry (k_remedy_t below)
#ifndef REMEDY_TILE_DEFAULT
#define REMEDY_TILE_DEFAULT 0  // single-device remedy: 1 = tile engine, 0 = member-list kernel
#endif
#ifndef RT_SHARDS
#define RT_SHARDS 32
#endif
#ifndef RT_CHUNK
#define RT_CHUNK 4  // tiles per grab (<= 4: 7 stamp lanes per tile)
#endif
#ifndef RT_MINB
#define RT_MINB 4
#endif
#ifndef RT_ISO
#define RT_ISO 1  // skip the solve of members whose neighbours did not change last round
#endif
constexpr int RT_GS = 32;  // grab counter stride (uint32): one 128-byte line per shard and slot
enum { FS_SELF = 1, FS_XL = 2, FS_XH = 4, FS_YL = 8, FS_YH = 16, FS_ZL = 32, FS_ZH = 64 };

template <int DIM>
struct TileGeo {
    static constexpr int LY = DIM == 3 ? 3 : 5, LZ = DIM == 3 ? 2 : 0;
    static constexpr int TY = 1 << LY, TZ = 1 << LZ;
    // lanes on the tile's faces
    static constexpr unsigned YL = DIM == 3 ? 0x01010101u : 0x00000001u;
    static constexpr unsigned YH = DIM == 3 ? 0x80808080u : 0x80000000u;
    static constexpr unsigned ZL = DIM == 3 ? 0x000000ffu : 0u;
    static constexpr unsigned ZH = DIM == 3 ? 0xff000000u : 0u;
};

// ---------------------------------------------------------------------------
// Local solvers (bit-exact restatements; no FMA contraction)
// ---------------------------------------------------------------------------

__device__ __forceinline__ real_t dmin(real_t a, real_t b) { return a <= b ? a : b; }
__device__ __forceinline__ real_t dmax(real_t a, real_t b) { return a >= b ? a : b; }

// sqrt(max(x, 0)) for the roots: x <= 0 (or NaN) yields +0 without feeding the
// IEEE slow path (sqrt of 0/negative/NaN); the reference's clamp
// `x if x > 0 else 0` (E/local_solver.py) gives exactly +0 there too.  Where
// the numpy form would propagate NaN (E/_kernels.py:56, NaN disc) the root is
// never selected (take_two / isfinite guards), so the result is unchanged.
__device__ __forceinline__ real_t sqrt_rn(real_t x)
{
    real_t r;  // opaque to the optimizer, so the operand select below is not folded away
#if EIK_SINGLE
    asm("sqrt.rn.f32 %0, %1;" : "=f"(r) : "f"(x));
#else
    asm("sqrt.rn.f64 %0, %1;" : "=d"(r) : "d"(x));
#endif
    return r;
}
__device__ __forceinline__ real_t sqrt_pos(real_t x) { return x > R_ZERO ? sqrt_rn(x > R_ZERO ? x : R_ONE) : R_ZERO; }

// x / 3.0 correctly rounded without the division sequence (Markstein): inv3 =
// RN(1/3) has relative error 2^-54, so q = RN(x * inv3) is within 3/4 ulp of
// x/3 (faithful), r = x - 3q is exact under FMA, and RN(q + r * inv3) is the
// correctly rounded quotient; x/3 is never a rounding tie.  Tiny (subnormal
// quotient), zero and non-finite dividends take the IEEE division.  Checked
// bit-exact against x / 3.0 on 3.4e10 values (tools/cuda/check_div3.cu).
__device__ __forceinline__ real_t div3_rn(real_t x)
{
#if EIK_SINGLE
    return x / R_THREE;
#else
    if (!(x >= 0x1p-900) || !(x < INFINITY)) return x / 3.0;
    const real_t inv3 = 0x1.5555555555555p-2;
    const real_t q = __dmul_rn(x, inv3);
    const real_t r = __fma_rn(-q, 3.0, x);
    return __fma_rn(r, inv3, q);
#endif
}

// E/_kernels.py:47-58 (_update_uniform_batch), d = delta / f
__device__ __forceinline__ real_t upd2u(real_t a, real_t b, real_t d)
{
    const real_t lo = dmin(a, b);
    const real_t hi = dmax(a, b);
    const real_t one = lo + d;
    const real_t diff = hi - lo;
    const bool take_two = diff <= kSqrt2 * d;
    const real_t disc = R_TWO * d * d - diff * diff;
    const real_t root = R_HALF * (a + b + sqrt_pos(disc));
    const bool valid = take_two && (disc >= -DISC_CLAMP * (R_TWO * d * d)) && (root >= hi);
    return valid ? root : one;
}

// E/_kernels.py:61-88 (_update_aniso_batch)
__device__ __forceinline__ real_t upd2a(real_t a, real_t b, real_t f, real_t dx, real_t dy)
{
    const real_t one_x = a + dx / f;
    const real_t one_y = b + dy / f;
    const real_t dx2 = dx * dx;
    const real_t dy2 = dy * dy;
    const real_t s2 = (dx2 + dy2) / (f * f);
    const real_t s = sqrt(s2);
    const real_t diff = a - b;
    const real_t disc = s2 - diff * diff;
    const real_t root = (a * dy2 + b * dx2 + (dx * dy) * sqrt_pos(disc)) / (dx2 + dy2);
    const real_t drop_larger = (a > b) ? one_y : one_x;
    const bool valid = isfinite(a) && isfinite(b) && !(diff > s) && !(-diff > s) &&
                       (disc >= -DISC_CLAMP * s2) && (root >= a) && (root >= b);
    real_t out = valid ? root : drop_larger;
    if (isinf(a) && isfinite(b)) out = one_y;
    if (isfinite(a) && isinf(b)) out = one_x;
    if (isinf(a) && isinf(b)) out = INFINITY;
    return out;
}

// E/local_solver.py:91-157 (update_3d_uniform), verified branch walk; d = delta / f.
//
// Every branch's root is a pure function of the sorted neighbours and d, and
// the walk only compares those roots with the neighbours, so its outcome can
// be written in closed form.  With F3/F2 = "branch 3/2 demotes on its
// discriminant (or a2 = inf)", G3 = r3 >= a3, L2 = r2 < a2, H2 = r2 > a3,
// H1 = r1 > a2, and k0 the guard's entry branch, the walk returns
//   k0 = 3:  (!F3 && G3) ? r3 : (F2 || L2) ? r1 : r2
//   k0 = 2:  (F2 || L2) ? r1 : M2
//   k0 = 1:  (!H1 || F2) ? r1 : M2,     M2 = H2 ? (F3 ? r2 : r3) : r2
// (walk 3 -> 2 -> 1 stops at 1 because 2 was visited; 2 -> 3 accepts r3
// because 2 was visited, or falls back to 2 which then returns r2; 1 -> 2
// ignores L2 because 1 was visited).  The selected value is produced by the
// reference's own expression: bit-identical.  When every lane of the warp
// takes the common "k0 = 3 and r3 valid" exit, branch 2 is not evaluated.
__device__ __forceinline__ real_t upd3u(real_t px, real_t py, real_t pz, real_t d, real_t delta)
{
    real_t a1 = px, a2 = py, a3 = pz, t;
    if (a2 < a1) { t = a1; a1 = a2; a2 = t; }
    if (a3 < a2) { t = a2; a2 = a3; a3 = t; }
    if (a2 < a1) { t = a1; a1 = a2; a2 = t; }
    const int k0 = (a3 - a1 < delta) ? 3 : ((a2 - a1 < delta) ? 2 : 1);
    // branch 3 (E/local_solver.py:119-134)
    const real_t b2 = a2 - a1;
    const real_t b3 = a3 - a1;
    const real_t s3 = b2 + b3;
    const real_t disc3 = s3 * s3 - R_THREE * (b2 * b2 + b3 * b3 - d * d);
    const bool F3 = disc3 < -DISC_CLAMP * (R_THREE * d * d);
    // r3 is only ever selected with a3 finite; an infinite dividend would take
    // the division slow path for a value nobody reads
    const real_t x3 = s3 + sqrt_pos(disc3);
    const real_t r3 = a1 + div3_rn(x3 < INFINITY ? x3 : R_ZERO);
    const bool quick = (a1 == INFINITY) || (k0 == 3 && !F3 && r3 >= a3);
    if (__all_sync(__activemask(), quick)) return a1 == INFINITY ? INFINITY : r3;
    // branch 2 (E/local_solver.py:136-151) and branch 1 (:152-157)
    const real_t disc2 = R_TWO * d * d - b2 * b2;
    const bool F2 = (a2 == INFINITY) || (disc2 < -DISC_CLAMP * (R_TWO * d * d));
    const real_t r2 = R_HALF * (a1 + a2 + sqrt_pos(disc2));
    const real_t r1 = a1 + d;
    const bool L2 = r2 < a2, H2 = r2 > a3, H1 = r1 > a2;
    const real_t M2 = H2 ? (F3 ? r2 : r3) : r2;
    real_t out;
    if (k0 == 3) out = (!F3 && r3 >= a3) ? r3 : ((F2 || L2) ? r1 : r2);
    else if (k0 == 2) out = (F2 || L2) ? r1 : M2;
    else out = (!H1 || F2) ? r1 : M2;
    return a1 == INFINITY ? INFINITY : out;
}

// ---------------------------------------------------------------------------
// small helpers
// ---------------------------------------------------------------------------

// Tolerance of the converge / build / decrease tests at value x.  float64: the
// caller's absolute tol (E/ifim.py:121,157,203).  float32 perf mode: at least
// 4 ulps of x, since a float32 Jacobi pair can otherwise alternate between
// neighbouring floats forever (|v - old| = 1 ulp > 1e-12).
__device__ __forceinline__ real_t tol_at(real_t tol, real_t x)
{
#if EIK_SINGLE
    const real_t r = x * (real_t)0x1p-21;
    return (r > tol && r < INFINITY) ? r : tol;  // an infinite old value keeps the absolute tol
#else
    (void)x;
    return tol;
#endif
}

__device__ __forceinline__ real_t ldcg(const real_t *p) { return __ldcg(p); }
__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T vload(const T *p) { return *(const volatile T *)p; }

__device__ __forceinline__ unsigned long long globaltimer()
{
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

constexpr unsigned EIK_EHANG = 5;  // device-side watchdog tripped (reported as a CUDA error)

// Software barrier over this rank's CTAs (co-resident: cooperative launch) and,
// in multi-rank mode, across ranks: the last CTA of a rank arrives at the world
// counter (rank 0's control block), the last rank releases every rank's
// generation word, each rank then releases its CTAs.  System-scope fences make
// the data written before the barrier visible to peer GPUs.  Returns false if
// the watchdog fired (nobody arrived within ~10 s); callers then leave the
// kernel so a logic error cannot wedge the GPU.
#ifndef SPIN_NS
#define SPIN_NS 32  // back-off between polls of a barrier word
#endif
__device__ __forceinline__ bool spin_until_change(volatile unsigned *w, unsigned old, Ctl *ctl)
{
    const unsigned long long t0 = globaltimer();
    for (unsigned k = 0; *w == old; ++k) {
        if (SPIN_NS) __nanosleep(SPIN_NS);
        if ((k & 15u) == 15u &&  // watchdog checks every 16 polls
            (*(volatile unsigned *)&ctl->err == EIK_EHANG || globaltimer() - t0 > 10000000000ull)) {
            atomicExch(&ctl->err, EIK_EHANG);
            return false;
        }
    }
    return true;
}

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

// Software grid barrier over the nblocks CTAs of this rank (and, in multi-rank
// mode, across ranks).  Thread 0 of each CTA arrives with an acq_rel atomic
// (releasing the CTA's writes, ordered before it by bar.sync), the last arriver
// releases the generation word and the others acquire it; the watchdog turns a
// missing arrival into EIK_EHANG instead of a wedged GPU.
__device__ __forceinline__ bool grid_barrier_n(Ctl *ctl, unsigned nblocks, const KP *p)
{
    __shared__ unsigned s_ok;
    __syncthreads();
    if (!p || !p->mr || p->R == 1) {
        // single rank: one acq_rel add per CTA on one word; CTA 0 adds 2^31 - (n - 1), the others
        // 1, so the last arrival flips bit 31 and leaves the low bits as they were (no reset, no
        // separate release); everyone waits for the flip with acquire loads
        if (threadIdx.x == 0) {
            const unsigned add = blockIdx.x == (p ? p->gb0 : 0u) ? 0x80000000u - (nblocks - 1u) : 1u;
            const unsigned old = atom_add_acq_rel_gpu(&ctl->bar_count, add);
            unsigned ok = 1;
            const unsigned long long t0 = globaltimer();
            for (unsigned k = 0; ((old ^ ld_acquire_gpu(&ctl->bar_count)) & 0x80000000u) == 0u; ++k) {
                if (SPIN_NS) __nanosleep(SPIN_NS);
                if ((k & 15u) == 15u &&  // watchdog checks every 16 polls
                    (*(volatile unsigned *)&ctl->err == EIK_EHANG || globaltimer() - t0 > 10000000000ull)) {
                    atomicExch(&ctl->err, EIK_EHANG);
                    ok = 0;
                    break;
                }
            }
            s_ok = ok;
        }
        __syncthreads();
        return s_ok != 0;
    }
    // multi-rank: arrivals count on bar_count; the rank's last arriver meets the other ranks
    // (system-scope counter at rank 0, then every rank's wgen) and releases its rank through the
    // generation word bar_gen, which the others poll
    if (threadIdx.x == 0) {
        volatile unsigned *vgen = &ctl->bar_gen;
        const unsigned gen = *vgen;
        __threadfence();  // gpu-scope release; the last arriver publishes system-wide below
        unsigned ok = 1;
        if (atomicAdd(&ctl->bar_count, 1u) == nblocks - 1u) {
            atomicExch(&ctl->bar_count, 0u);
            volatile unsigned *wg = &ctl->wgen;
            const unsigned wgen = *wg;
            __threadfence_system();
            Ctl *c0 = p->rank_ctl[0];
            if (atomicAdd_system(&c0->wcount, 1u) == (unsigned)p->R - 1) {
                atomicExch_system(&c0->wcount, 0u);
                __threadfence_system();
                for (int r = 0; r < p->R; ++r) atomicAdd_system(&p->rank_ctl[r]->wgen, 1u);
            } else {
                ok = spin_until_change(wg, wgen, ctl);
            }
            __threadfence_system();
            __threadfence();
            atomicAdd(&ctl->bar_gen, 1u);
        } else {
            ok = spin_until_change(vgen, gen, ctl);
        }
        __threadfence();
        s_ok = ok;
    }
    __syncthreads();
    return s_ok != 0;
}

__device__ __forceinline__ bool grid_barrier(Ctl *ctl) { return grid_barrier_n(ctl, gridDim.x, nullptr); }

template <typename T>
__device__ __forceinline__ T warp_sum(T v)
{
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    return v;
}

// Sum a per-thread value over the block of NT threads; result valid in thread 0.
template <int NT = BLOCK>
__device__ __forceinline__ unsigned long long block_sum(unsigned long long v, unsigned long long *sm)
{
    v = warp_sum(v);
    const int w = threadIdx.x >> 5;
    __syncthreads();
    if (lane_id() == 0) sm[w] = v;
    __syncthreads();
    unsigned long long t = 0;
    if (threadIdx.x == 0)
        for (int i = 0; i < NT / 32; ++i) t += sm[i];
    __syncthreads();
    return t;
}

// Per-cell coefficient of the local solver: d = delta/F (uniform) or F (anisotropic).
template <int SOL>
__device__ __forceinline__ real_t coef(const KP &p, uint32_t c)
{
    return (SOL == SOL_A2) ? __ldg(p.F + c) : __ldg(p.dd + c);
}

// Traversal order of the remedy member list: x-word columns of 4x4 (y, z) row
// tiles (3D) or 16-row tiles (2D), so a CTA's consecutive members cover their
// own y +- 1 / z +- 1 neighbour rows (L1 reuse).  Positions beyond the grid
// (tile padding) map to an out-of-range word.
#ifndef TILE_LY
#define TILE_LY 2  // log2 rows per tile in y (3D)
#endif
#ifndef TILE_LZ
#define TILE_LZ 2  // log2 rows per tile in z (3D)
#endif
#ifndef TILE_L2D
#define TILE_L2D 4  // log2 rows per tile (2D)
#endif
template <int DIM>
__device__ __forceinline__ uint32_t word_at(const KP &p, uint32_t l)
{
    constexpr uint32_t LT = DIM == 3 ? TILE_LY + TILE_LZ : TILE_L2D;
    const uint32_t in = l & ((1u << LT) - 1u), t = l >> LT;
    const uint32_t tile = fdiv(t, p.fW), wx = t - tile * p.W;
    uint32_t y, z;
    if (DIM == 3) {
        const uint32_t tz = fdiv(tile, p.fnty4), ty = tile - tz * p.nty4;
        y = (ty << TILE_LY) + (in & ((1u << TILE_LY) - 1u));
        z = (tz << TILE_LZ) + (in >> TILE_LY);
    } else {
        y = (tile << TILE_L2D) + in;
        z = 0;
    }
    if (y >= (uint32_t)p.ny || z >= (uint32_t)p.nz) return 0xffffffffu;
    return (z * (uint32_t)p.ny + y) * p.W + wx;
}

struct WPos {
    uint32_t row, wx, y, z;
    uint32_t x0, c0;
    uint32_t rowm;  // lanes inside the row
};

template <int DIM>
__device__ __forceinline__ WPos wpos(const KP &p, uint32_t w)
{
    WPos q;
    q.row = fdiv(w, p.fW);
    q.wx = w - q.row * p.W;
    if (DIM == 3) {
        q.z = fdiv(q.row, p.fny);
        q.y = q.row - q.z * (uint32_t)p.ny;
    } else {
        q.z = 0;
        q.y = q.row;
    }
    q.x0 = q.wx * 32u;
    q.c0 = q.row * p.nx32 + q.x0;
    const uint32_t nv = p.nx32 - q.x0;
    q.rowm = nv >= 32 ? FULL : ((1u << nv) - 1u);
    return q;
}

// Jacobi snapshot around one cell (E/_kernels.py:29-38: out-of-grid reads
// are +inf) plus the cell's coefficient (d = delta/F, or F for the
// anisotropic solver).
struct Sten {
    real_t c, w, e, s, n, d, u, k;
    real_t edge;  // word layout: lane 0 / lane 31 x-neighbour outside the word
};

// Word layout, stage 1: issue every load of the word at once (one memory
// round trip).  Lanes adjacent to an active lane load their own value so the
// x-neighbours come from shuffles in stage 2.
template <int DIM, int SOL>
__device__ __forceinline__ void gather_issue(const KP &p, const real_t *__restrict__ Pc, const WPos &q, uint32_t bits,
                                             Sten &s)
{
    const unsigned lane = lane_id();
    const bool act = (bits >> lane) & 1u;
    const uint32_t need = (bits | (bits << 1) | (bits >> 1)) & q.rowm;
    const uint32_t c = q.c0 + lane;
    s.c = s.edge = s.s = s.n = s.d = s.u = INFINITY;
    s.k = 1.0;
    if ((need >> lane) & 1u) s.c = ldcg(Pc + c);
    if (act) {
        if (lane == 0 && q.wx > 0) s.edge = ldcg(Pc + (c - 1));
        if (lane == 31 && q.x0 + 32 < p.nx32) s.edge = ldcg(Pc + (c + 1));
        if (q.y > 0) s.s = ldcg(Pc + (c - p.nx32));
        if (q.y + 1 < p.ny) s.n = ldcg(Pc + (c + p.nx32));
        if (DIM == 3) {
            if (q.z > 0) s.d = ldcg(Pc + (c - p.plane32));
            else if (p.mr && p.lo.valid)  // multi-rank: neighbour's top plane, same buffer parity
                s.d = ldcg((Pc == p.P0 ? p.lo.P0 : p.lo.P1) + (((p.lo.nz - 1) * (uint32_t)p.ny + q.y) * p.nx32 + q.x0 + lane));
            if (q.z + 1 < p.nz) s.u = ldcg(Pc + (c + p.plane32));
            else if (p.mr && p.hi.valid)
                s.u = ldcg((Pc == p.P0 ? p.hi.P0 : p.hi.P1) + (q.y * p.nx32 + q.x0 + lane));
        }
        s.k = coef<SOL>(p, c);
    }
}

// Word layout, stage 2: x-neighbours by shuffle.
__device__ __forceinline__ void gather_finish(const KP &p, const WPos &q, Sten &s)
{
    const unsigned lane = lane_id();
    real_t w = __shfl_up_sync(FULL, s.c, 1);
    real_t e = __shfl_down_sync(FULL, s.c, 1);
    if (lane == 0) w = s.edge;
    if (lane == 31) e = s.edge;
    else if (q.x0 + lane + 1 >= p.nx32) e = INFINITY;
    s.w = w;
    s.e = e;
}

template <int DIM, int SOL>
__device__ __forceinline__ void gather(const KP &p, const real_t *__restrict__ Pc, const WPos &q, uint32_t bits,
                                       Sten &s)
{
    gather_issue<DIM, SOL>(p, Pc, q, bits, s);
    gather_finish(p, q, s);
}

// One local-solver call on the gathered stencil (E/ifim.py:57-59).
template <int DIM, int SOL>
__device__ __forceinline__ real_t solve(const KP &p, const Sten &s)
{
    const real_t xm = dmin(s.w, s.e);
    const real_t ym = dmin(s.s, s.n);
    if (SOL == SOL_U2) return upd2u(xm, ym, s.k);
    if (SOL == SOL_A2) return upd2a(xm, ym, s.k, p.dx, p.dy);
    return upd3u(xm, ym, dmin(s.d, s.u), s.k, p.delta);
}

// Worklist entries: cell index | CARRY.  CARRY marks cells that changed in the
// previous iteration/round; only they must rewrite an unchanged value into the
// other phi buffer to keep the Jacobi double buffer consistent (every other
// cell already holds its current value there).  Cell indices are < 2^31.
constexpr uint32_t CARRY = 0x80000000u;

// Block-wide exclusive scan of a per-thread count plus one global reservation:
// returns this thread's first slot in the global list whose length is *glen.
template <bool SYS = false, int NT = BLOCK>
__device__ __forceinline__ unsigned block_reserve(unsigned v, unsigned *glen, unsigned *sscan)
{
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    unsigned inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned t = __shfl_up_sync(FULL, inc, o);
        if (lane >= (unsigned)o) inc += t;
    }
    if (lane == 31) sscan[warp] = inc;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned acc = 0;
        for (int i = 0; i < (NT / 32); ++i) {
            const unsigned t = sscan[i];
            sscan[i] = acc;
            acc += t;
        }
        sscan[(NT / 32)] = acc ? (SYS ? atomicAdd_system(glen, acc) : atomicAdd(glen, acc)) : 0u;
    }
    __syncthreads();
    const unsigned pos = sscan[(NT / 32)] + sscan[warp] + inc - v;
    __syncthreads();
    return pos;
}

// ---------------------------------------------------------------------------
// Preparation kernels
// ---------------------------------------------------------------------------

// Slab mode: ghost planes (neighbour ranks' boundary planes) are read, never computed.
__device__ __forceinline__ bool ghost_plane(const KP &p, uint32_t z) { return p.slab && (z == 0 || z + 1 == (uint32_t)p.nz); }

// apply_boundary writes (E/grid.py:212-215); validation is done by the caller.
__global__ void k_seed(real_t *phi, uint8_t *state, const int64_t *idx, const double *val, int64_t n)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        phi[idx[s]] = val[s];
        state[idx[s]] = ST_SOURCE;
    }
}


// One pass over all words: copy phi into the second buffer, d = delta / F,
// touched = blocked, fixed = blocked | source, optionally clear set bitmaps.
template <int DIM, bool UNIFORM>
__global__ void __launch_bounds__(BLOCK) k_prep(KP p, bool copy_phi, bool build_touched)
{
    const unsigned lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t GW = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = gw; w < p.nwords; w += GW) {
        const WPos q = wpos<DIM>(p, w);
        const bool in = (q.rowm >> lane) & 1u;
        const uint32_t c = q.c0 + lane;
        uint8_t st = 0;
        if (in) {
            st = p.state[c];
            if (copy_phi) p.P1[c] = p.P0[c];
            if (UNIFORM) p.dd[c] = p.delta / p.F[c];
        }
        const uint32_t blk = __ballot_sync(FULL, in && st == ST_BLOCKED);
        const uint32_t src = __ballot_sync(FULL, in && st == ST_SOURCE);
        if (lane == 0) {
            const bool gh = ghost_plane(p, q.z);
            const uint32_t fw = gh ? FULL : (blk | src | ~q.rowm);  // lanes outside the row count as fixed
            p.Fb[w] = fw;
            if (p.Ft) {  // tile-major copy for the remedy tile engine
                constexpr int LY = TileGeo<DIM>::LY, LZ = TileGeo<DIM>::LZ;
                const uint32_t t = (((q.z >> LZ) * p.nty + (q.y >> LY)) * p.W + q.wx);
                p.Ft[t * 32u + (((q.z & ((1u << LZ) - 1u)) << LY) | (q.y & ((1u << LY) - 1u)))] = fw;
            }
            if (build_touched) p.Bt[w] = gh ? 0u : blk;   // ghost bits record activation requests
        }
    }
}

// Multi-rank: write the seeds this rank owns (global linear index -> local).
#if !EIK_SINGLE
__global__ void k_seed_mr(real_t *phi, uint8_t *state, const int64_t *idx, const double *val, int64_t n, int64_t zg0,
                          int64_t nzl, int64_t plane)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = idx[s] / plane;
        if (z < zg0 || z >= zg0 + nzl) continue;
        const int64_t c = idx[s] - zg0 * plane;
        phi[c] = val[s];
        state[c] = ST_SOURCE;
    }
}
#endif

// Multi-rank initial activation: every seed (global index) activates the free
// FAR neighbours this rank owns (E/ifim.py:97-102).
#if !EIK_SINGLE
__global__ void k_init_active_mr(KP p, const int64_t *seeds, int64_t nseeds, int64_t zg0, int64_t nz_global)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseeds; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t g = seeds[s];
        const int64_t i = g % p.nx, r = g / p.nx, j = r % p.ny, k = r / p.ny;
        const int64_t nb[6][3] = {{i - 1, j, k}, {i + 1, j, k}, {i, j - 1, k}, {i, j + 1, k}, {i, j, k - 1}, {i, j, k + 1}};
        for (int t = 0; t < 6; ++t) {
            const int64_t x = nb[t][0], y = nb[t][1], z = nb[t][2];
            if (x < 0 || x >= p.nx || y < 0 || y >= p.ny || z < 0 || z >= nz_global) continue;
            if (z < zg0 || z >= zg0 + p.nz) continue;  // owned by another rank
            const int64_t e = ((z - zg0) * p.ny + y) * p.nx + x;
            const uint8_t st = p.state[e];
            if (st == ST_BLOCKED || st == ST_SOURCE) continue;
            const uint32_t w = (uint32_t)(((z - zg0) * p.ny + y) * p.W + (x >> 5));
            const uint32_t bit = 1u << (x & 31);
            if (atomicOr(p.Bt + w, bit) & bit) continue;  // label != FAR
            p.L0[atomicAdd(&p.ctl->len[0], 1u)] = (uint32_t)e;
        }
    }
}
#endif

// Initial Active = free FAR axis neighbours of the seeds (E/ifim.py:97-102).
template <int DIM>
__global__ void k_init_active(KP p, const int64_t *seeds, int64_t nseeds)
{
    for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < nseeds; s += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = seeds[s];
        const int64_t i = c % p.nx;
        const int64_t r = c / p.nx;
        const int64_t j = r % p.ny;
        const int64_t k = r / p.ny;
        int64_t nb[6];
        int m = 0;
        if (i > 0) nb[m++] = c - 1;
        if (i < p.nx - 1) nb[m++] = c + 1;
        if (j > 0) nb[m++] = c - p.nx;
        if (j < p.ny - 1) nb[m++] = c + p.nx;
        if (DIM == 3) {
            if (k > 0) nb[m++] = c - p.plane;
            if (k < p.nz - 1) nb[m++] = c + p.plane;
        }
        for (int t = 0; t < m; ++t) {
            const int64_t e = nb[t];
            if (DIM == 3 && ghost_plane(p, (uint32_t)(e / p.plane))) continue;  // owned by a neighbour rank
            const uint8_t st = p.state[e];
            if (st == ST_BLOCKED || st == ST_SOURCE) continue;
            const int64_t row = e / p.nx;
            const int64_t x = e - row * p.nx;
            const uint32_t w = (uint32_t)(row * p.W + (x >> 5));
            const uint32_t bit = 1u << (x & 31);
            const uint32_t old = atomicOr(p.Bt + w, bit);
            if (old & bit) continue;  // label != FAR
            p.L0[atomicAdd(&p.ctl->len[0], 1u)] = (uint32_t)e;
        }
    }
}

// ---------------------------------------------------------------------------
// Update step: persistent kernel, one iteration per grid barrier.
// The active list is a compacted list of cell indices processed one thread per
// cell (a thin 3D wavefront leaves ~1 active cell per 32-cell row segment, so
// a word layout would idle 31 of 32 lanes).  Next list = non-converged cells
// + newly activated FAR neighbours; each cell enters it at most once (an
// active cell is "touched", activation is an atomicOr on the touched bitmap),
// so its length is exactly |A_{k+1}|.
// ---------------------------------------------------------------------------

#ifndef UPD_MU
#define UPD_MU 1  // active cells per thread per pass (2 measured slower: 47 vs 37 ms at 512^3)
#endif
#ifndef UPD_PREF
#define UPD_PREF 1  // first-pass list entry loaded with the list length after each barrier
#endif
// Sum of a worklist-length slot over all ranks (multi-rank) or this rank.
template <bool MR>
__device__ __forceinline__ unsigned long long ranks_len(const KP &p, int slot)
{
    if (!MR) return vload(&p.ctl->len[slot]);
    unsigned long long t = 0;
    for (int r = 0; r < p.R; ++r) t += __ldcg(&p.rank_ctl[r]->len[slot]);
    return t;
}

template <bool MR>
__device__ __forceinline__ unsigned long long ranks_sum(const KP &p, const unsigned long long Ctl::*field, int slot)
{
    if (!MR) return vload(&(p.ctl->*field)) ;
    unsigned long long t = 0;
    for (int r = 0; r < p.R; ++r) t += vload(&(p.rank_ctl[r]->*field));
    return t;
}

template <int DIM, int SOL, bool MR>
__device__ __forceinline__ void update_body(const KP &p)
{
    __shared__ unsigned sscan[WPB + 1];
    __shared__ unsigned long long sred[WPB];
    Ctl *ctl = p.ctl;
    const unsigned gb = blockIdx.x - p.gb0, gnb = p.gnb ? p.gnb : gridDim.x;
    const bool lead = gb == 0 && threadIdx.x == 0 && (!MR || p.q == 0);  // writes the global stats
    unsigned long long a_writes = 0, a_conv = 0;
    if (MR && !grid_barrier_n(ctl, gnb, &p)) return;  // every rank's initial list is complete
    if (!p.slab) {
        const unsigned long long n0 = ranks_len<MR>(p, (int)(p.it0 % 3));
        if (n0 == 0) return;  // no initial active cell: zero iterations
        if (lead) {
            if (p.hist_cap > 0) p.hist[0] = (int64_t)n0;
            ctl->sum = n0;
            ctl->peak = n0;
        }
    }
    const uint32_t nx = (uint32_t)p.nx, ny = (uint32_t)p.ny, nz = (uint32_t)p.nz;
    unsigned nnext = ~0u;  // next iteration's list length when already read
    // UPD_PREF: this thread's first list entry of the next iteration, loaded right after the barrier
    // together with the list length (the two L2 round trips overlap); entries past the length are
    // stale and masked by `live`
    uint32_t pre = 0;
    bool have_pre = false;
    for (int64_t it = p.it0; it < p.it0 + p.max_it; ++it) {
#ifdef EIK_DIAG
        unsigned long long duc0 = 0;
        if (threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(duc0));
#endif
        const int par = (int)(it & 1);
        const real_t *__restrict__ Pc = par ? p.P1 : p.P0;
        real_t *__restrict__ Pn = par ? p.P0 : p.P1;
        const uint32_t *__restrict__ Lc = par ? p.L1 : p.L0;
        uint32_t *Ln = par ? p.L0 : p.L1;
        unsigned *lenN = &ctl->len[(it + 1) % 3];
        // this rank's list length (single rank: the global count read after the last barrier)
        const unsigned n = nnext != ~0u ? nnext : vload(&ctl->len[it % 3]);
        for (unsigned base = gb * (BLOCK * UPD_MU); base < n; base += gnb * (BLOCK * UPD_MU)) {
            uint32_t c[UPD_MU], x[UPD_MU], y[UPD_MU], z[UPD_MU], r[UPD_MU];
            unsigned emit[UPD_MU];  // bit 0: stay; bits 1..6: activate W, E, S, N, D, U
            bool carry[UPD_MU], live[UPD_MU];
            Sten s[UPD_MU];
            // issue every load of this thread's cells before any solve
#pragma unroll
            for (int u = 0; u < UPD_MU; ++u) {
                const unsigned i = base + u * BLOCK + threadIdx.x;
                live[u] = i < n;
                emit[u] = 0;
                if (UPD_PREF && u == 0 && have_pre && base == gb * (BLOCK * UPD_MU)) c[u] = live[u] ? pre : 0u;
                else c[u] = live[u] ? __ldcg(Lc + i) : 0u;
                carry[u] = (c[u] & CARRY) != 0;  // non-converged in the previous iteration
                c[u] &= ~CARRY;
                r[u] = fdiv(c[u], p.fnx);
                x[u] = c[u] - r[u] * nx;
                if (DIM == 3) {
                    z[u] = fdiv(r[u], p.fny);
                    y[u] = r[u] - z[u] * ny;
                } else {
                    z[u] = 0;
                    y[u] = r[u];
                }
                Sten &t = s[u];
                t.c = t.w = t.e = t.s = t.n = t.d = t.u = INFINITY;
                t.k = 1.0;
                if (live[u]) {
                    const uint32_t cc = c[u];
                    t.c = __ldca(Pc + cc);
                    if (x[u] > 0) t.w = __ldca(Pc + (cc - 1));
                    if (x[u] + 1 < nx) t.e = __ldca(Pc + (cc + 1));
                    if (y[u] > 0) t.s = __ldca(Pc + (cc - nx));
                    if (y[u] + 1 < ny) t.n = __ldca(Pc + (cc + nx));
                    if (DIM == 3) {
                        if (z[u] > 0) t.d = __ldca(Pc + (cc - p.plane32));
                        else if (MR && p.lo.valid)  // neighbour rank's top plane (peer memory)
                            t.d = __ldcg((par ? p.lo.P1 : p.lo.P0) + (((p.lo.nz - 1) * ny + y[u]) * nx + x[u]));
                        if (z[u] + 1 < nz) t.u = __ldca(Pc + (cc + p.plane32));
                        else if (MR && p.hi.valid)  // neighbour rank's bottom plane
                            t.u = __ldcg((par ? p.hi.P1 : p.hi.P0) + (y[u] * nx + x[u]));
                    }
                    t.k = coef<SOL>(p, cc);
                }
            }
#pragma unroll
            for (int u = 0; u < UPD_MU; ++u) {
                if (!live[u]) continue;
                const Sten &t = s[u];
                const real_t v = solve<DIM, SOL>(p, t);
                // E/ifim.py:121: converged iff v == old or |v - old| <= tol
                const bool conv = (v == t.c) || fabs(v - t.c) <= tol_at(p.tol, t.c);
                if (!conv) Pn[c[u]] = v;              // E/ifim.py:128
                else if (carry[u]) Pn[c[u]] = t.c;    // changed last iteration: carry into the other buffer
                if (!conv) {
                    emit[u] = 1u;
                    ++a_writes;
                } else {
                    ++a_conv;
                    // activate +inf, unblocked, FAR neighbours (E/ifim.py:123-126)
                    const real_t nv[6] = {t.w, t.e, t.s, t.n, t.d, t.u};
                    uint32_t old[6];
#pragma unroll
                    for (int k = 0; k < (DIM == 3 ? 6 : 4); ++k) {
                        old[k] = 0xffffffffu;
                        const bool inb = k == 0 ? x[u] > 0 : k == 1 ? x[u] + 1 < nx : k == 2 ? y[u] > 0
                                         : k == 3 ? y[u] + 1 < ny : k == 4 ? z[u] > 0 : z[u] + 1 < nz;
                        if (MR && DIM == 3 && k >= 4 && !inb && nv[k] == INFINITY) {
                            // the neighbour lies on an adjacent rank: activate it there (E/ifim.py:123-126)
                            const Peer &pr = k == 4 ? p.lo : p.hi;
                            if (pr.valid) {
                                const uint32_t ze = k == 4 ? pr.nz - 1 : 0u;
                                const uint32_t bit = 1u << (x[u] & 31);
                                const uint32_t old2 = atomicOr_system(pr.Bt + (ze * ny + y[u]) * p.W + (x[u] >> 5), bit);
                                if (!(old2 & bit)) {
                                    uint32_t *Lp = par ? pr.L0 : pr.L1;
                                    Lp[atomicAdd_system(&pr.ctl->len[(it + 1) % 3], 1u)] = (ze * ny + y[u]) * nx + x[u];
                                    // the only remote plain store: publish it system-wide before this
                                    // CTA arrives at the (gpu-scope) barrier
                                    __threadfence_system();
                                }
                            }
                            continue;
                        }
                        if (inb && nv[k] == INFINITY) {
                            const uint32_t xe = k == 0 ? x[u] - 1 : k == 1 ? x[u] + 1 : x[u];
                            const uint32_t re = k == 2 ? r[u] - 1 : k == 3 ? r[u] + 1 : k == 4 ? r[u] - ny
                                                : k == 5 ? r[u] + ny : r[u];
                            const uint32_t bit = 1u << (xe & 31);
                            // boundary planes are also activated by the neighbouring ranks: system scope
                            old[k] = ((MR && (z[u] <= 1u || z[u] + 2u >= nz)) ? atomicOr_system(p.Bt + re * p.W + (xe >> 5), bit)
                                                                               : atomicOr(p.Bt + re * p.W + (xe >> 5), bit)) | ~bit;
                            // slab mode: a ghost-plane target is an activation request for its owner
                            if (DIM == 3 && k >= 4 && ghost_plane(p, k == 4 ? z[u] - 1 : z[u] + 1)) old[k] = 0xffffffffu;
                        }
                    }
#pragma unroll
                    for (int k = 0; k < (DIM == 3 ? 6 : 4); ++k)
                        if (old[k] != 0xffffffffu) emit[u] |= 2u << k;
                }
            }
            unsigned tot = 0;
#pragma unroll
            for (int u = 0; u < UPD_MU; ++u) tot += __popc(emit[u]);
            unsigned pos = block_reserve<MR>(tot, lenN, sscan);  // peers append to lenN too
#pragma unroll
            for (int u = 0; u < UPD_MU; ++u) {
                if (emit[u] & 1u) Ln[pos++] = c[u] | CARRY;
#pragma unroll
                for (int k = 0; k < (DIM == 3 ? 6 : 4); ++k) {
                    const uint32_t e = k == 0 ? c[u] - 1 : k == 1 ? c[u] + 1 : k == 2 ? c[u] - nx : k == 3 ? c[u] + nx
                                       : k == 4 ? c[u] - p.plane32 : c[u] + p.plane32;
                    if (emit[u] & (2u << k)) Ln[pos++] = e;
                }
            }
        }
        if (gb == 0 && threadIdx.x == 0) {
            ctl->len[(it + 2) % 3] = 0;
#ifdef EIK_DIAG
            ctl->duw[(it + 1) % 3][0] = ctl->duw[(it + 1) % 3][1] = 0;
#endif
        }
#ifdef EIK_DIAG
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long duc1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(duc1));
            atomicMax(&ctl->duw[it % 3][0], duc1 - duc0);
            atomicAdd(&ctl->duw[it % 3][1], duc1 - duc0);
        }
#endif
        if (!grid_barrier_n(ctl, gnb, MR ? &p : nullptr)) return;
        if (UPD_PREF && !MR) {
            const unsigned i0 = gb * (BLOCK * UPD_MU) + threadIdx.x;
            pre = i0 < (unsigned)p.ncells ? __ldcg(Ln + i0) : 0u;
            have_pre = true;
        }
        const unsigned long long m = ranks_len<MR>(p, (int)((it + 1) % 3));
        nnext = MR ? ~0u : (unsigned)m;
#ifdef EIK_DIAG
        if (lead) {
            unsigned long long tnow;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tnow));
            const int bk = n ? min(25, 31 - __clz(n)) : 0;
            if (it > p.it0) {
                ctl->du[0][bk] += 1;
                ctl->du[1][bk] += tnow - ctl->du[2][25];
                ctl->du[2][bk] += n;
                ctl->du2[0][bk] += ctl->duw[it % 3][0];
                ctl->du2[1][bk] += ctl->duw[it % 3][1] / gnb;
            }
            ctl->du[2][25] = tnow;  // last barrier time (bucket 25 of cells is never reached)
        }
#endif
        if (p.slab) continue;  // the host reduces the counts and decides
        if (lead) {
            ctl->iters = it + 1;
            if (m) {
                if (it + 1 < p.hist_cap) p.hist[it + 1] = (int64_t)m;
                ctl->sum += m;
                if (m > ctl->peak) ctl->peak = m;
            }
        }
        if (m == 0) break;
        if (it + 1 >= p.cap) {  // E/ifim.py:106-110
            if (gb == 0 && threadIdx.x == 0) ctl->err = EIK_ECAP;
            break;
        }
    }
    const unsigned long long tw = block_sum(a_writes, sred);
    const unsigned long long tc = block_sum(a_conv, sred);
    if (threadIdx.x == 0) {
        atomicAdd(&ctl->writes, tw);
        atomicAdd(&ctl->conv, tc);
    }
}

#ifndef UPD_2D_PER_SM
#define UPD_2D_PER_SM 1  // update step CTAs per SM on 2D grids (thin O(n) fronts)
#endif
#ifndef UPD_MINB
#define UPD_MINB 3  // update step: CTAs per SM the register budget is sized for
#endif
template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK, UPD_MINB) k_update(KP p)
{
    update_body<DIM, SOL, false>(p);
}

// Multi-rank: rank groups of one launch (emulation on one GPU, kps[] in device
// memory) or one rank per GPU (kps[0]); peers through device-visible pointers.
template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK, UPD_MINB) k_update_mr(const KP *__restrict__ kps, uint32_t per_group)
{
    update_body<DIM, SOL, true>(kps[blockIdx.x / per_group]);
}

// One rank per launch (one process per GPU): the rank's parameters stay in the
// kernel parameter space instead of being read through a pointer.
template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK, UPD_MINB) k_update_mr1(KP p)
{
    update_body<DIM, SOL, true>(p);
}

// ---------------------------------------------------------------------------
// Build pass (E/ifim.py:137-161): one value per free cell, flag |v - phi| > tol.
// Writes R_0 as a row-major bitmap (every word) and counts it.
// ---------------------------------------------------------------------------

template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK) k_build(KP p, const real_t *__restrict__ Pc, const unsigned *skip)
{
    __shared__ unsigned long long sred[WPB];
    if (skip && *skip) return;
    const unsigned lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t GW = (gridDim.x * blockDim.x) >> 5;
    Ctl *ctl = p.ctl;
    unsigned long long a_free = 0, a_flag = 0;
    for (uint32_t w = gw; w < p.nwords; w += GW) {
        const WPos q = wpos<DIM>(p, w);
        const uint32_t freem = q.rowm & ~__ldg(p.Fb + w);
        uint32_t mm = 0;
        if (freem) {
            Sten s;
            gather<DIM, SOL>(p, Pc, q, freem, s);
            bool moved = false;
            if ((freem >> lane) & 1u) {
                const real_t v = solve<DIM, SOL>(p, s);
                moved = fabs(v - s.c) > tol_at(p.tol, s.c);  // NaN (inf - inf) is not flagged
            }
            mm = __ballot_sync(FULL, moved);
        }
        if (lane == 0) {
            p.R0b[w] = mm;
            a_free += __popc(freem);
            a_flag += __popc(mm);
        }
    }
    const unsigned long long tf = block_sum(a_free, sred);
    const unsigned long long tg = block_sum(a_flag, sred);
    if (threadIdx.x == 0) {
        atomicAdd(&ctl->free_cells, tf);
        atomicAdd(&ctl->flagged, tg);
    }
}

// Remedy set from uint8 masks (a RemedySet built elsewhere): the work list `cells` becomes R_0;
// members outside it (`member` & ~cells, E/ifim.py:64-72: RemedySet.member vs .cells) never get
// relaxed and never get enqueued (E/ifim.py:211), so they go to the tile-major St bitmap the
// remedy's dilation excludes.
template <int DIM>
__global__ void __launch_bounds__(BLOCK) k_remedy_load(KP p, const uint8_t *cells, const uint8_t *member)
{
    const unsigned lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t GW = (gridDim.x * blockDim.x) >> 5;
    unsigned long long cnt = 0;
    unsigned any_stale = 0;
    for (uint32_t w = gw; w < p.nwords; w += GW) {
        const WPos q = wpos<DIM>(p, w);
        const bool in = (q.rowm >> lane) & 1u;
        const bool wk = in && cells[q.c0 + lane] != 0;
        const uint32_t m = __ballot_sync(FULL, wk);
        const uint32_t sm = member ? __ballot_sync(FULL, in && !wk && member[q.c0 + lane] != 0) : 0u;
        if (lane == 0) {
            p.R0b[w] = m;
            cnt += __popc(m);
            if (member) {
                constexpr int LY = TileGeo<DIM>::LY, LZ = TileGeo<DIM>::LZ;
                const uint32_t t = (((q.z >> LZ) * p.nty + (q.y >> LY)) * p.W + q.wx);
                p.St[t * 32u + (((q.z & ((1u << LZ) - 1u)) << LY) | (q.y & ((1u << LY) - 1u)))] = sm;
                any_stale |= sm;
            }
        }
    }
    if (lane == 0 && cnt) atomicAdd(&p.ctl->flagged, cnt);
    if (lane == 0 && any_stale) atomicOr(&p.ctl->stale, 1u);
}

template <int DIM>
__global__ void k_remedy_export(KP p, uint8_t *member)
{
    const unsigned lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t GW = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t w = gw; w < p.nwords; w += GW) {
        const uint32_t m = p.R0b[w];
        if (m == 0) continue;
        const WPos q = wpos<DIM>(p, w);
        if ((m >> lane) & 1u) member[q.c0 + lane] = 1;
    }
}

// ---------------------------------------------------------------------------
// Remedy step (E/ifim.py:164-218): persistent kernel, two grid barriers per
// round.
//   B: R_r = R_0 (round 0) or D_{r-1} | (N(D_{r-1}) & ~fixed) (E/ifim.py:209-214
//      in set form: membership only deduplicates), one thread per bitmap word;
//      the members are compacted, in word order, into a cell list.
//   A: one thread per member: v from the snapshot; v < phi - tol writes P_next
//      and sets the member's D_r bit, otherwise the member drops
//      (E/ifim.py:199-208).
// |R_r| is the list length, |D_r| a counter; the loop ends when D_r is empty.
// ---------------------------------------------------------------------------

#ifndef REM_PER
#define REM_PER 4  // bitmap words per thread in phase B
#endif
#ifndef REM_MU
#define REM_MU 2            // phase A: members per lane in flight
#endif
// phase B: member words expanded per warp step.  2D: 4 (cfg2 remedy -6 %: a warp whose stretch
// of the traversal is dense walks up to 128 words, and the slowest warp holds the grid barrier);
// 3D: 1 (the extra registers spill in the 64-register list kernel and cost phase A more)
#ifndef REM_XU2
#define REM_XU2 4
#endif
// Phase B member expansion through per-warp shared-memory staging (3D: cfg4 remedy 263.0 ->
// 257.5 ms, cfg3 4.30 -> 4.15 ms; 2D with 8 words per step: cfg2 49.6 -> 48.4 ms against the
// shuffle form with REM_XU2 words per step, which REM_STAGE / REM_STAGE2 = 0 select)
#ifndef REM_STAGE
#define REM_STAGE 1
#endif
#ifndef REM_STAGE2
#define REM_STAGE2 1
#endif
// CTA-wide staging: the CTA's member words of a sweep go to one shared-memory queue and all its
// warps walk it round-robin (REM_CSXU per step), so the warps share a dense stretch instead of
// its owner walking it alone while the grid barrier waits (2D: cfg2 remedy 48.3 -> 36.2 ms;
// 3D: cfg3 4.12 -> 3.76 ms, cfg4 256.7 -> 255.3 ms)
#ifndef REM_CSTAGE2
#define REM_CSTAGE2 1
#endif
// Phase B work assignment: 0 = each CTA takes NT*REM_PER consecutive traversal positions per
// sweep; 1 = consecutive 32*REM_PER-position warp blocks go to different CTAs
#ifndef REM_WIL2
#define REM_WIL2 1
#endif
#ifndef REM_WIL3
#define REM_WIL3 2
#endif
#ifndef REM_CSTAGE3
#define REM_CSTAGE3 1
#endif
#ifndef REM_CSXU
#define REM_CSXU 4
#endif
#ifndef REM_SXU
#define REM_SXU 2   // staged words walked per step, 3D
#endif
#ifndef REM_SXU2
#define REM_SXU2 8  // staged words walked per step, 2D
#endif
#ifndef REM_XU3
#define REM_XU3 1
#endif


#ifdef EIK_DIAG
__shared__ unsigned dg_cta_members;
#endif
template <int DIM, bool MR, int NT>
__device__ __forceinline__ void rem_members(const KP &p, uint32_t r, const uint32_t *__restrict__ Dp,
                                            uint32_t *Dc, uint32_t *ML, unsigned *lenR, unsigned *sscan, unsigned gb,
                                            unsigned gnb)
{
    const unsigned lane = lane_id();
    const uint32_t chunk = NT * REM_PER;
    const uint32_t planeW = (uint32_t)p.ny * p.W;
    const int ppar = (int)((r + 1) & 1);  // parity of D_{r-1}
    // 3D (REM_WIL3 = 2): interleave only when one sweep covers the grid; with several sweeps the
    // strided chunks already spread a front over the CTAs and contiguous chunks keep phase A's
    // list segments local
    const bool WIL = DIM == 2 ? REM_WIL2 != 0 : (REM_WIL3 == 1 || (REM_WIL3 == 2 && p.npos <= gnb * chunk));
    const uint32_t wchunk = 32u * REM_PER, wrp = threadIdx.x >> 5;
    for (uint32_t it = 0;; ++it) {
        uint32_t pbase;  // this thread's first traversal position
        if (WIL) {
            if (((it * (NT / 32)) * gnb + gb) * wchunk >= p.npos) break;  // warp 0 holds the CTA's lowest block
            pbase = ((it * (NT / 32) + wrp) * gnb + gb) * wchunk + lane * REM_PER;
        } else {
            const uint32_t base = (gb + it * gnb) * chunk;
            if (base >= p.npos) break;
            pbase = base + threadIdx.x * REM_PER;
        }
        uint32_t R[REM_PER], C[REM_PER], WW[REM_PER];
        unsigned cnt = 0;
#pragma unroll
        for (int k = 0; k < REM_PER; ++k) {
            const uint32_t w = pbase + k < p.npos ? word_at<DIM>(p, pbase + k) : 0xffffffffu;  // brick order (see word_at)
            WW[k] = w;
            R[k] = C[k] = 0;
            if (w < p.nwords) {
                if (r == 0) {
                    R[k] = __ldcg(p.R0b + w);
                } else {
                    const uint32_t row = fdiv(w, p.fW);
                    const uint32_t wx = w - row * p.W;
                    uint32_t y, z;
                    if (DIM == 3) {
                        z = fdiv(row, p.fny);
                        y = row - z * (uint32_t)p.ny;
                    } else {
                        z = 0;
                        y = row;
                    }
                    const uint32_t c = __ldcg(Dp + w);
                    const uint32_t dw = wx > 0 ? __ldcg(Dp + w - 1) : 0u;
                    const uint32_t de = wx + 1 < p.W ? __ldcg(Dp + w + 1) : 0u;
                    const uint32_t ds = y > 0 ? __ldcg(Dp + w - p.W) : 0u;
                    const uint32_t dn = y + 1 < p.ny ? __ldcg(Dp + w + p.W) : 0u;
                    uint32_t dd = 0, du = 0;
                    if (DIM == 3) {
                        if (z > 0) dd = __ldcg(Dp + w - planeW);
                        else if (MR && p.lo.valid)  // neighbour rank's top-plane decreases (peer memory)
                            dd = __ldcg((ppar ? p.lo.D1b : p.lo.D0b) + ((p.lo.nz - 1) * (uint32_t)p.ny + y) * p.W + wx);
                        if (z + 1 < p.nz) du = __ldcg(Dp + w + planeW);
                        else if (MR && p.hi.valid)
                            du = __ldcg((ppar ? p.hi.D1b : p.hi.D0b) + y * p.W + wx);
                    }
                    const uint32_t dil = (c << 1) | (c >> 1) | (dw >> 31) | (de << 31) | ds | dn | dd | du;
                    const bool gh = DIM == 3 && ghost_plane(p, z);
                    R[k] = gh ? 0u : (c | (dil & ~__ldg(p.Fb + w)));
                    C[k] = gh ? 0u : c;
                }
                Dc[w] = 0;  // D_r is accumulated by phase A with atomicOr
                cnt += __popc(R[k]);
            }
        }
        unsigned pos = block_reserve<false, NT>(cnt, lenR, sscan);
#ifdef EIK_DIAG
        if (cnt) atomicAdd(&dg_cta_members, cnt);
#endif
        // warp-cooperative expansion: one word at a time, 32 coalesced entries per store; XU words
        // per step (their shuffles and stores are independent, so the steps overlap)
        constexpr int XU = DIM == 2 ? REM_XU2 : REM_XU3;
        if constexpr (DIM == 2 ? REM_CSTAGE2 : REM_CSTAGE3) {
            // the CTA stages all its member words in shared memory and its warps walk them
            // round-robin, so a CTA's dense stretch is shared by all its warps
            __shared__ uint4 s_c[NT * REM_PER];
            __shared__ unsigned s_n;
            const unsigned warp = threadIdx.x >> 5;
            const uint32_t lt = (1u << lane) - 1u;
            if (threadIdx.x == 0) s_n = 0;
            __syncthreads();
#pragma unroll
            for (int k = 0; k < REM_PER; ++k) {
                if (R[k]) {
                    const uint32_t row = fdiv(WW[k], p.fW);
                    s_c[atomicAdd(&s_n, 1u)] = make_uint4(R[k], C[k], row * p.nx32 + (WW[k] - row * p.W) * 32u, pos);
                }
                pos += __popc(R[k]);
            }
            __syncthreads();
            const unsigned n = s_n;
            for (unsigned j = warp; j < n; j += (NT / 32) * REM_CSXU) {
#pragma unroll
                for (int q = 0; q < REM_CSXU; ++q) {
                    const unsigned jj = j + q * (NT / 32);
                    if (jj < n) {
                        const uint4 e = s_c[jj];
                        if ((e.x >> lane) & 1u)
                            ML[e.w + __popc(e.x & lt)] = (e.z + lane) | (((e.y >> lane) & 1u) ? CARRY : 0u);
                    }
                }
            }
            __syncthreads();
        } else if (DIM == 3 ? REM_STAGE : REM_STAGE2) {
            // each warp stages its member words of step k in shared memory ({bits, carry,
            // first cell, first slot}) and walks them with broadcast loads, REM_SXU per step: no
            // shuffles, and the unrolled walk needs no per-word registers beyond the entry
            __shared__ uint4 s_q[NT / 32][32];
            const unsigned warp = threadIdx.x >> 5;
            const uint32_t lt = (1u << lane) - 1u;
#pragma unroll
            for (int k = 0; k < REM_PER; ++k) {
                const unsigned m = __ballot_sync(FULL, R[k] != 0);
                if (R[k]) {
                    const uint32_t row = fdiv(WW[k], p.fW);
                    s_q[warp][__popc(m & lt)] = make_uint4(R[k], C[k], row * p.nx32 + (WW[k] - row * p.W) * 32u, pos);
                }
                pos += __popc(R[k]);
                __syncwarp();
                const int n = __popc(m);
                constexpr int SXU = DIM == 2 ? REM_SXU2 : REM_SXU;
                for (int j = 0; j < n; j += SXU) {
#pragma unroll
                    for (int q = 0; q < SXU; ++q) {
                        if (j + q < n) {
                            const uint4 e = s_q[warp][j + q];
                            if ((e.x >> lane) & 1u)
                                ML[e.w + __popc(e.x & lt)] = (e.z + lane) | (((e.y >> lane) & 1u) ? CARRY : 0u);
                        }
                    }
                }
                __syncwarp();
            }
        } else {
#pragma unroll
        for (int k = 0; k < REM_PER; ++k) {
            unsigned todo = __ballot_sync(FULL, R[k] != 0);
            const uint32_t w = WW[k];
            const uint32_t row = fdiv(w, p.fW);
            const uint32_t c0 = row * p.nx32 + (w - row * p.W) * 32u;
            while (todo) {
                int src[XU];
                bool has[XU];
#pragma unroll
                for (int q = 0; q < XU; ++q) {
                    has[q] = todo != 0;
                    src[q] = has[q] ? __ffs(todo) - 1 : 0;
                    todo &= todo - 1;
                }
#pragma unroll
                for (int q = 0; q < XU; ++q) {
                    const uint32_t bits = __shfl_sync(FULL, R[k], src[q]);
                    const uint32_t carry = __shfl_sync(FULL, C[k], src[q]);
                    const uint32_t off = __shfl_sync(FULL, pos, src[q]);
                    const uint32_t cc0 = __shfl_sync(FULL, c0, src[q]);
                    if (has[q] && ((bits >> lane) & 1u))
                        ML[off + __popc(bits & ((1u << lane) - 1u))] = (cc0 + lane) | (((carry >> lane) & 1u) ? CARRY : 0u);
                }
            }
            pos += __popc(R[k]);
        }
        }
    }
}

#ifndef REM_MINB
#define REM_MINB 4
#endif
template <int DIM, int SOL, bool MR, int NT>
__device__ __forceinline__ void remedy_body(const KP &p, const unsigned *skip)
{
    __shared__ unsigned sscan[NT / 32 + 1];
    __shared__ unsigned long long sred[NT / 32];
    if (skip && *skip) return;
    Ctl *ctl = p.ctl;
    const unsigned lane = lane_id();
    const unsigned gb = blockIdx.x - p.gb0, gnb = p.gnb ? p.gnb : gridDim.x;
    const bool lead = gb == 0 && threadIdx.x == 0 && (!MR || p.q == 0);
    if (MR && !grid_barrier_n(ctl, gnb, &p)) return;  // every rank's build (R0) is complete
    if (!p.slab) {
        unsigned long long r0 = 0;
        if (MR) {
            for (int q = 0; q < p.R; ++q) r0 += vload(&p.rank_ctl[q]->flagged);
        } else {
            r0 = vload(&ctl->flagged);
        }
        if (r0 == 0) return;  // empty remedy set: zero rounds
        if (lead) {
            ctl->peak = r0;
            ctl->sum = 0;
        }
    }
    const uint32_t nx = p.nx32, ny = (uint32_t)p.ny, nz = (uint32_t)p.nz;
    uint32_t *ML = p.L0;
    for (int64_t rr = p.it0; rr < p.it0 + p.max_it; ++rr) {
        const uint32_t r = (uint32_t)rr;
#ifdef EIK_DIAG
        unsigned long long dgt0 = 0, dgt1 = 0, dgc0 = 0;
        int dgb = 0;
        if (lead) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dgt0));
        if (threadIdx.x == 0) {
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dgc0));
            dg_cta_members = 0;
        }
        __syncthreads();
#endif
        const int par = (int)(r & 1);
        const real_t *__restrict__ Pc = par ? p.P1 : p.P0;
        real_t *__restrict__ Pn = par ? p.P0 : p.P1;
        uint32_t *Dc = par ? p.D1b : p.D0b;
        const uint32_t *Dp = par ? p.D0b : p.D1b;
        unsigned *lenR = &ctl->len[r % 3];
        // ---- phase B: members of R_r ----
        rem_members<DIM, MR, NT>(p, r, Dp, Dc, ML, lenR, sscan, gb, gnb);
        if (gb == 0 && threadIdx.x == 0) {
            // slot (r+1)%3 of len / dsum was last read two rounds ago
            ctl->len[(r + 1) % 3] = 0;
            ctl->dsum[(r + 1) % 3] = 0;
#ifdef EIK_DIAG
            for (int q = 0; q < 5; ++q) ctl->dgw[(r + 1) % 3][q] = q == 3 ? ~0ull : 0ull;
            ctl->dgk[(r + 1) % 3] = 0;
#endif
        }
#ifdef EIK_DIAG
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long dgc1;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dgc1));
            atomicMax(&ctl->dgw[r % 3][0], dgc1 - dgc0);
            atomicAdd(&ctl->dgw[r % 3][1], dgc1 - dgc0);
            atomicMax(&ctl->dgw[r % 3][2], dgc0);
            atomicMin(&ctl->dgw[r % 3][3], dgc0);
            atomicMax(&ctl->dgw[r % 3][4], dgc1);
            atomicMax(&ctl->dgk[r % 3], ((dgc1 - dgc0) << 24) | ((unsigned long long)min(dg_cta_members, 16383u) << 10) | gb);
        }
#endif
        if (!grid_barrier_n(ctl, gnb, MR ? &p : nullptr)) return;
        const unsigned m = vload(lenR);  // this rank's |R_r| (list length)
        const unsigned long long mg = MR ? ranks_len<MR>(p, (int)(r % 3)) : m;  // global |R_r|
        if (!p.slab && rr > p.it0) {
            // R_r = D_{r-1} u (N(D_{r-1}) \ fixed) is empty exactly when round r-1 decreased
            // nothing: the loop ends here (no separate read of |D_{r-1}| after its barrier)
            if (mg == 0) break;
            if (r >= (uint32_t)p.cap) {  // E/ifim.py:185-189
                if (gb == 0 && threadIdx.x == 0) ctl->err = EIK_ECAP;
                break;
            }
        }
        if (lead) {
            ctl->iters = r + 1;
            ctl->sum += mg;
            if (mg > ctl->peak) ctl->peak = mg;
#ifdef EIK_DIAG
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dgt1));
            dgb = mg ? min(25, 63 - __clzll(mg)) : 0;
            ctl->dg[0][dgb] += 1;
            ctl->dg[1][dgb] += dgt1 - dgt0;
            ctl->dg[3][dgb] += mg;
            ctl->dg2[0][dgb] += ctl->dgw[r % 3][0];
            ctl->dg2[1][dgb] += ctl->dgw[r % 3][1] / gnb;
            ctl->dg2[2][dgb] += ctl->dgw[r % 3][2] - ctl->dgw[r % 3][3];
            ctl->dg2[3][dgb] += dgt1 > ctl->dgw[r % 3][4] ? dgt1 - ctl->dgw[r % 3][4] : 0ull;
            const unsigned long long kk = ctl->dgk[r % 3];
            ctl->dg2[4][dgb] += (kk >> 10) & 16383u;
            ctl->dg2[5][dgb] += (kk & 1023u) == 0u;
            ctl->dg2[6][dgb] += kk & 1023u;
#endif
        }
        // ---- phase A: one local solve per member, REM_MU members per lane in flight ----
        unsigned long long a_dec = 0;
        // one contiguous segment of the (brick-ordered) list per CTA: L1 reuse of neighbour rows
        const uint32_t seg = ((m + gnb - 1) / gnb + 32 * REM_MU - 1) / (32 * REM_MU) * (32 * REM_MU);
        const uint32_t sbeg = gb * seg, mend = min(m, sbeg + seg);
        const uint32_t wbase = sbeg + (threadIdx.x >> 5) * 32 * REM_MU, wstride = (NT / 32) * 32 * REM_MU;
        for (uint32_t i0 = wbase; i0 < mend; i0 += wstride) {
            uint32_t ent[REM_MU], rw[REM_MU], x[REM_MU];
            bool live[REM_MU];
            Sten s[REM_MU];
#pragma unroll
            for (int u = 0; u < REM_MU; ++u) {
                const uint32_t i = i0 + u * 32 + lane;
                live[u] = i < mend;
                ent[u] = live[u] ? __ldcg(ML + i) : 0u;
            }
#pragma unroll
            for (int u = 0; u < REM_MU; ++u) {
                const uint32_t c = ent[u] & ~CARRY;
                rw[u] = fdiv(c, p.fnx);
                x[u] = c - rw[u] * nx;
                uint32_t y, z = 0;
                if (DIM == 3) {
                    z = fdiv(rw[u], p.fny);
                    y = rw[u] - z * ny;
                } else {
                    y = rw[u];
                }
                Sten &t = s[u];
                t.c = t.w = t.e = t.s = t.n = t.d = t.u = INFINITY;
                t.k = 1.0;
                if (live[u]) {
                    t.c = __ldca(Pc + c);
                    if (x[u] > 0) t.w = __ldca(Pc + (c - 1));
                    if (x[u] + 1 < nx) t.e = __ldca(Pc + (c + 1));
                    if (y > 0) t.s = __ldca(Pc + (c - nx));
                    if (y + 1 < ny) t.n = __ldca(Pc + (c + nx));
                    if (DIM == 3) {
                        if (z > 0) t.d = __ldca(Pc + (c - p.plane32));
                        else if (MR && p.lo.valid)  // neighbour rank's top plane (peer memory)
                            t.d = __ldcg((par ? p.lo.P1 : p.lo.P0) + (((p.lo.nz - 1) * ny + y) * nx + x[u]));
                        if (z + 1 < nz) t.u = __ldca(Pc + (c + p.plane32));
                        else if (MR && p.hi.valid)
                            t.u = __ldcg((par ? p.hi.P1 : p.hi.P0) + (y * nx + x[u]));
                    }
                    t.k = coef<SOL>(p, c);
                }
            }
#pragma unroll
            for (int u = 0; u < REM_MU; ++u) {
                const uint32_t c = ent[u] & ~CARRY;
                bool dec = false;
                if (live[u]) {
                    const real_t v = solve<DIM, SOL>(p, s[u]);
                    dec = v < s[u].c - tol_at(p.tol, s[u].c);  // E/ifim.py:203
                    if (dec) Pn[c] = v;
                    else if (ent[u] & CARRY) Pn[c] = s[u].c;  // changed last round: carry into the other buffer
                }
                // D_r bits: a warp's members of one word are contiguous in the list, so a
                // segmented OR-scan leaves each word's bits in its first lane, which
                // issues a single atomicOr for the word.
                a_dec += __popc(__ballot_sync(FULL, dec));
                const uint32_t wi = live[u] ? rw[u] * p.W + (x[u] >> 5) : 0xffffffffu;
                uint32_t acc = dec ? (1u << (x[u] & 31)) : 0u;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t ov = __shfl_down_sync(FULL, acc, o);
                    const uint32_t ow = __shfl_down_sync(FULL, wi, o);
                    if (lane + o < 32 && ow == wi) acc |= ov;
                }
                const uint32_t pw = __shfl_up_sync(FULL, wi, 1);
                if (live[u] && acc && (lane == 0 || pw != wi)) atomicOr(Dc + wi, acc);
            }
        }
        const unsigned long long td = block_sum<NT>(lane == 0 ? a_dec : 0ull, sred);
        if (threadIdx.x == 0 && td) {
            atomicAdd(&ctl->dsum[r % 3], td);
            atomicAdd(&ctl->writes, td);
        }
        if (!grid_barrier_n(ctl, gnb, MR ? &p : nullptr)) return;
#ifdef EIK_DIAG
        if (lead) {
            unsigned long long dgt2;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(dgt2));
            ctl->dg[2][dgb] += dgt2 - dgt1;
        }
#endif
        // slab mode: the host reduces the counts and decides; otherwise the next round's
        // phase B finds R_{r+1} empty when D_r is
    }
}

// Single-device remedy kernel: REM_NT threads per CTA (512: two CTAs per SM at the 64-register
// budget, the same 1024 threads as 4 x 256 but half the CTAs at every grid barrier and block
// reservation; measured -2 % on cfg4 / cfg2).  The multi-rank kernels keep BLOCK.
#ifndef REM_NT
#define REM_NT 512
#endif
template <int DIM, int SOL>
__global__ void __launch_bounds__(REM_NT, REM_MINB * BLOCK / REM_NT) k_remedy(KP p, const unsigned *skip)
{
    remedy_body<DIM, SOL, false, REM_NT>(p, skip);
}

template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK, REM_MINB) k_remedy_mr(const KP *__restrict__ kps, uint32_t per_group)
{
    remedy_body<DIM, SOL, true, BLOCK>(kps[blockIdx.x / per_group], nullptr);
}

template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK, REM_MINB) k_remedy_mr1(KP p)
{
    remedy_body<DIM, SOL, true, BLOCK>(p, nullptr);
}

// ---------------------------------------------------------------------------
// Remedy step, tile engine (single device; E/ifim.py:164-218).  One grid
// barrier per round and no global member list.
//
// A tile is one bitmap word column (32 cells in x) times 32 rows: 8 (y) x 4 (z)
// in 3D, 32 (y) in 2D; lane l of a warp owns row l.  The remedy's bitmaps are
// tile-major, so a tile's 32 row words are one 128-byte line.  Round r:
//   * warps take chunks of RT_CHUNK consecutive tiles from RT_SHARDS sharded
//     counters (contiguous tile ranges, so concurrently processed tiles are
//     spatial neighbours), and skip tiles R_r cannot touch: R_r = D_{r-1} u
//     (N(D_{r-1}) \ fixed) meets tile t only if t's own D_{r-1} line, or a face
//     neighbour's line with bits on the shared face, is non-empty.  Each tile's
//     D line carries a stamp ((round + 1) << 7 | face bits), written with the
//     line, so stale lines of earlier rounds are never read and never cleared;
//   * the warp forms the tile's R_r rows (x-dilation in-register, y/z dilation
//     by shuffles plus the face rows of the neighbour lines), expands the
//     members into a warp-private shared-memory list, and relaxes them 32 at a
//     time: gather, local solve, decrease test (E/ifim.py:203), write, D bit by
//     a shared-memory atomicOr on the row word;
//   * the tile's D_r line and stamp are plain stores (the tile has one owner).
// |R_r| and |D_r| are summed per CTA and added once per round; the loop ends
// when D_r is empty (R_{r+1} = 0).  Round 0 reads R_0 from the build's
// row-major bitmap.
// ---------------------------------------------------------------------------
template <int DIM>
__device__ __forceinline__ void tile_xyz(const KP &p, uint32_t t, uint32_t &wx, uint32_t &ty, uint32_t &tz)
{
    const uint32_t tyz = fdiv(t, p.fW);
    wx = t - tyz * p.W;
    if (DIM == 3) {
        tz = fdiv(tyz, p.fnty);
        ty = tyz - tz * p.nty;
    } else {
        tz = 0;
        ty = tyz;
    }
}

template <int DIM, int SOL>
__device__ __forceinline__ void rt_tile(const KP &p, uint32_t t, uint32_t r, uint32_t vm, const real_t *__restrict__ Pc,
                                        real_t *__restrict__ Pn, const uint32_t *__restrict__ Dp,
                                        uint32_t *__restrict__ Dc, uint32_t *__restrict__ stc, uint16_t *buf,
                                        uint32_t *sD, const uint32_t *__restrict__ St, unsigned &a_mem,
                                        unsigned &a_dec)
{
    using G = TileGeo<DIM>;
    const unsigned lane = lane_id();
    uint32_t wx, ty, tz;
    tile_xyz<DIM>(p, t, wx, ty, tz);
    const uint32_t ny = (uint32_t)p.ny, nz = (uint32_t)p.nz, nx = p.nx32;
    const uint32_t ly = lane & (G::TY - 1), lz = lane >> G::LY;
    const uint32_t yb = ty << G::LY, zb = tz << G::LZ;
    const uint32_t y = yb + ly, z = zb + lz;
    const uint32_t WNTY = p.W * p.nty;
    uint32_t R, carry, iso = 0;
    if (r == 0) {
        R = (y < ny && z < nz) ? __ldcg(p.R0b + (z * ny + y) * p.W + wx) : 0u;
        carry = 0;
    } else {
        const uint32_t *L = Dp + t * 32u + lane;
        const uint32_t c = (vm & 1u) ? __ldcg(L) : 0u;
        const uint32_t dw = (vm & 2u) ? __ldcg(L - 32) : 0u;
        const uint32_t de = (vm & 4u) ? __ldcg(L + 32) : 0u;
        const uint32_t ys = ((vm & 8u) && ly == 0) ? __ldcg(L - p.W * 32u + (G::TY - 1)) : 0u;
        const uint32_t yn = ((vm & 16u) && ly == G::TY - 1) ? __ldcg(L + p.W * 32u - (G::TY - 1)) : 0u;
        uint32_t zd = 0, zu = 0;
        if (DIM == 3) {
            zd = ((vm & 32u) && lz == 0) ? __ldcg(L - WNTY * 32u + (G::TZ - 1) * G::TY) : 0u;
            zu = ((vm & 64u) && lz == G::TZ - 1) ? __ldcg(L + WNTY * 32u - (G::TZ - 1) * G::TY) : 0u;
        }
        const uint32_t F = __ldg(p.Ft + t * 32u + lane) | (St ? __ldg(St + t * 32u + lane) : 0u);
        uint32_t sv = __shfl_up_sync(FULL, c, 1), nv = __shfl_down_sync(FULL, c, 1);
        if (ly == 0) sv = ys;
        if (ly == G::TY - 1) nv = yn;
        uint32_t dil = (c << 1) | (c >> 1) | (dw >> 31) | (de << 31) | sv | nv;
        if (DIM == 3) {
            uint32_t dv = __shfl_up_sync(FULL, c, G::TY), uv = __shfl_down_sync(FULL, c, G::TY);
            if (lz == 0) dv = zd;
            if (lz == G::TZ - 1) uv = zu;
            dil |= dv | uv;
        }
        R = c | (dil & ~F);
        carry = c;
        // members that decreased last round while none of their neighbours did: their inputs are
        // the previous round's, so the solve returns their current value -- no decrease -- and
        // only the carry write remains (the call is still counted)
        iso = RT_ISO ? (c & ~dil) : 0u;
    }
    // members: warp scan of the row counts, expansion into the warp's shared list
    const uint32_t cnt = __popc(R);
    uint32_t inc = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, inc, o);
        if (lane >= (unsigned)o) inc += v;
    }
    const uint32_t T = __shfl_sync(FULL, inc, 31);
    if (T == 0) return;
    // non-isolated members first, isolated ones (carry only) last
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t Rs = R & ~iso, ns = __popc(Rs);
    uint32_t is = ns;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t v = __shfl_up_sync(FULL, is, o);
        if (lane >= (unsigned)o) is += v;
    }
    const uint32_t T1 = __shfl_sync(FULL, is, 31);
#pragma unroll 1
    for (int pass = 0; pass < 2; ++pass) {
        const uint32_t Rp = pass ? iso : Rs;
        const uint32_t off = pass ? T1 + (inc - cnt) - (is - ns) : is - ns;
        unsigned todo = __ballot_sync(FULL, Rp != 0);
        while (todo) {
            const int src = __ffs(todo) - 1;
            todo &= todo - 1;
            const uint32_t bits = __shfl_sync(FULL, Rp, src);
            const uint32_t cb = __shfl_sync(FULL, carry, src);
            const uint32_t o = __shfl_sync(FULL, off, src);
            if ((bits >> lane) & 1u)
                buf[o + __popc(bits & lt)] = (uint16_t)((((cb >> lane) & 1u) << 10) | ((uint32_t)src << 5) | lane);
        }
    }
    sD[lane] = 0;
    __syncwarp();
    const uint32_t x0 = wx * 32u;
    unsigned ndec = 0;
    for (uint32_t b = 0; b < T; b += 32) {
        const uint32_t i = b + lane;
        const bool live = i < T;
        const uint32_t e = live ? (uint32_t)buf[i] : 0u;
        const uint32_t row = (e >> 5) & 31u, bit = e & 31u;
        const uint32_t x = x0 + bit, yy = yb + (row & (G::TY - 1)), zz = zb + (row >> G::LY);
        const uint32_t c = DIM == 3 ? (zz * ny + yy) * nx + x : yy * nx + x;
        if (b >= T1) {  // isolated members only: carry the value over
            if (live) Pn[c] = __ldca(Pc + c);
            continue;
        }
        Sten s;
        s.c = s.w = s.e = s.s = s.n = s.d = s.u = INFINITY;
        s.k = R_ONE;
        if (live) {
            s.c = __ldca(Pc + c);
            if (x > 0) s.w = __ldca(Pc + (c - 1));
            if (x + 1 < nx) s.e = __ldca(Pc + (c + 1));
            if (yy > 0) s.s = __ldca(Pc + (c - nx));
            if (yy + 1 < ny) s.n = __ldca(Pc + (c + nx));
            if (DIM == 3) {
                if (zz > 0) s.d = __ldca(Pc + (c - p.plane32));
                if (zz + 1 < nz) s.u = __ldca(Pc + (c + p.plane32));
            }
            s.k = coef<SOL>(p, c);
        }
        bool dec = false;
        if (live) {
            const real_t v = solve<DIM, SOL>(p, s);
            dec = v < s.c - tol_at(p.tol, s.c);  // E/ifim.py:203
            if (dec) {
                Pn[c] = v;
                atomicOr(sD + row, 1u << bit);
            } else if (e >> 10) {
                Pn[c] = s.c;  // changed last round: carry into the other buffer
            }
        }
        ndec += __popc(__ballot_sync(FULL, dec));
    }
    __syncwarp();
    const uint32_t Dn = sD[lane];
    const unsigned anyb = __ballot_sync(FULL, Dn != 0);
    if (anyb) {
        Dc[t * 32u + lane] = Dn;
        const unsigned xl = __ballot_sync(FULL, Dn & 1u), xh = __ballot_sync(FULL, Dn >> 31);
        if (lane == 0) {
            const uint32_t faces = FS_SELF | (xl ? FS_XL : 0) | (xh ? FS_XH : 0) | ((anyb & G::YL) ? FS_YL : 0) |
                                   ((anyb & G::YH) ? FS_YH : 0) | ((anyb & G::ZL) ? FS_ZL : 0) |
                                   ((anyb & G::ZH) ? FS_ZH : 0);
            stc[t] = ((r + 1u) << 7) | faces;
        }
    }
    a_mem += T;
    a_dec += ndec;
}

template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK, RT_MINB) k_remedy_t(KP p, const unsigned *skip)
{
    __shared__ uint16_t s_buf[WPB][1024];
    __shared__ uint32_t s_D[WPB][32];
    __shared__ unsigned long long sred[WPB];
    if (skip && *skip) return;
    Ctl *ctl = p.ctl;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    const uint32_t *St = vload(&ctl->stale) ? p.St : nullptr;
    const unsigned long long r0 = vload(&ctl->flagged);
    if (r0 == 0) return;  // empty remedy set: zero rounds
    if (lead) {
        ctl->peak = r0;
        ctl->sum = 0;
    }
    const uint32_t K = RT_SHARDS, CH = RT_CHUNK;
    const uint32_t shs = p.rt_shs;
    // lane s: shard s's chunk count
    const uint32_t sb = min(p.ntiles, lane * shs), se = min(p.ntiles, (lane + 1) * shs);
    const uint32_t my_nch = (se - sb + CH - 1) / CH;
    const uint32_t gw = blockIdx.x * WPB + warp;
    const uint32_t WNTY = p.W * p.nty;
    uint16_t *buf = s_buf[warp];
    uint32_t *sD = s_D[warp];
    for (uint32_t r = 0;; ++r) {
        const int par = (int)(r & 1);
        const real_t *__restrict__ Pc = par ? p.P1 : p.P0;
        real_t *__restrict__ Pn = par ? p.P0 : p.P1;
        uint32_t *Dc = par ? p.Dt1 : p.Dt0;
        const uint32_t *Dp = par ? p.Dt0 : p.Dt1;
        uint32_t *stc = par ? p.stamp1 : p.stamp0;
        const uint32_t *stp = par ? p.stamp0 : p.stamp1;
        unsigned *Gc = p.grab + (r % 3) * K * RT_GS;
        unsigned a_mem = 0, a_dec = 0;
        uint32_t s = gw % K;
        while (true) {
            uint32_t k = 0;
            if (lane == 0) k = atomicAdd(Gc + s * RT_GS, 1u);
            k = __shfl_sync(FULL, k, 0);
            if (k >= __shfl_sync(FULL, my_nch, s)) {  // shard s is done: look for one with chunks left
                const uint32_t g = vload(Gc + lane * RT_GS);
                const unsigned left = __ballot_sync(FULL, g < my_nch);
                if (!left) break;
                const unsigned hi = left & (~0u << s);
                s = __ffs(hi ? hi : left) - 1;
                continue;
            }
            const uint32_t tb = s * shs + k * CH, te = min(tb + CH, min(p.ntiles, (s + 1) * shs));
            // activity: lanes 7j + n test neighbour n of tile tb + j (stamps of round r - 1)
            unsigned mask = 0;
            if (r > 0) {
                const uint32_t jj = lane / 7u, nn = lane - jj * 7u, tt = tb + jj;
                bool f = false;
                if (jj < CH && tt < te) {
                    uint32_t wx, ty, tz;
                    tile_xyz<DIM>(p, tt, wx, ty, tz);
                    uint32_t nb = tt, need = FS_SELF;
                    bool ex = true;
                    switch (nn) {
                        case 1: ex = wx > 0; nb = tt - 1; need = FS_XH; break;
                        case 2: ex = wx + 1 < p.W; nb = tt + 1; need = FS_XL; break;
                        case 3: ex = ty > 0; nb = tt - p.W; need = FS_YH; break;
                        case 4: ex = ty + 1 < p.nty; nb = tt + p.W; need = FS_YL; break;
                        case 5: ex = DIM == 3 && tz > 0; nb = tt - WNTY; need = FS_ZH; break;
                        case 6: ex = DIM == 3 && tz + 1 < p.ntz; nb = tt + WNTY; need = FS_ZL; break;
                        default: break;
                    }
                    if (ex) {
                        const uint32_t st = __ldcg(stp + nb);
                        f = (st >> 7) == r && (st & need);
                    }
                }
                mask = __ballot_sync(FULL, f);
            }
            for (uint32_t t = tb, j = 0; t < te; ++t, ++j) {
                const uint32_t vm = (mask >> (7 * j)) & 0x7fu;
                if (r > 0 && !vm) continue;
                rt_tile<DIM, SOL>(p, t, r, vm, Pc, Pn, Dp, Dc, stc, buf, sD, St, a_mem, a_dec);
            }
        }
        const unsigned long long tm = block_sum(lane == 0 ? (unsigned long long)a_mem : 0ull, sred);
        const unsigned long long td = block_sum(lane == 0 ? (unsigned long long)a_dec : 0ull, sred);
        if (threadIdx.x == 0) {
            if (tm) atomicAdd(&ctl->cnt[r % 3], tm);
            if (td) {
                atomicAdd(&ctl->dsum[r % 3], td);
                atomicAdd(&ctl->writes, td);
            }
        }
        if (blockIdx.x == 0) {
            // slot (r+1)%3 of the counts was last read at the start of round r-1; grab slot (r+2)%3
            // was last used in round r-1
            if (threadIdx.x == 0) {
                ctl->cnt[(r + 1) % 3] = 0;
                ctl->dsum[(r + 1) % 3] = 0;
            }
            if (threadIdx.x < K) p.grab[((r + 2) % 3) * K * RT_GS + threadIdx.x * RT_GS] = 0;
        }
        if (!grid_barrier(ctl)) return;
        const unsigned long long mg = vload(&ctl->cnt[r % 3]);  // |R_r|
        const unsigned long long dg = vload(&ctl->dsum[r % 3]);  // |D_r|
        if (lead) {
            ctl->iters = r + 1;
            ctl->sum += mg;
            if (mg > ctl->peak) ctl->peak = mg;
        }
        if (dg == 0) break;  // R_{r+1} is empty
        if (r + 1 >= (uint32_t)p.cap) {  // E/ifim.py:185-189
            if (lead) ctl->err = EIK_ECAP;
            break;
        }
    }
}

#include "eik_remedy_tma.cuh"

// ---------------------------------------------------------------------------
// Fixpoint reference (E/oracle.py:22-70): full-grid Jacobi passes
// phi <- min(phi, U(snapshot)) over every free cell until nothing decreases or
// the largest decrease is below tol; cap 10*(nx+ny[+nz]) passes.  Every free
// cell writes the other buffer each pass, so the double buffer stays exact.
// max_change is reduced with atomicMax on the IEEE bits (non-negative doubles
// order like their bit patterns; +inf for first reaches).
// ---------------------------------------------------------------------------

template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK) k_fixpoint(KP p)
{
    __shared__ unsigned long long sred[WPB];
    Ctl *ctl = p.ctl;
    const unsigned lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t GW = (gridDim.x * blockDim.x) >> 5;
    for (int64_t it = 0;; ++it) {
        const int par = (int)(it & 1);
        const real_t *__restrict__ Pc = par ? p.P1 : p.P0;
        real_t *__restrict__ Pn = par ? p.P0 : p.P1;
        unsigned long long a_dec = 0, a_max = 0;
        for (uint32_t w = gw; w < p.nwords; w += GW) {
            const WPos q = wpos<DIM>(p, w);
            const uint32_t freem = q.rowm & ~__ldg(p.Fb + w);
            if (freem == 0) continue;
            Sten s;
            gather<DIM, SOL>(p, Pc, q, freem, s);
            bool dec = false;
            if ((freem >> lane) & 1u) {
                const real_t cand = solve<DIM, SOL>(p, s);
                const real_t nw = dmin(s.c, cand);  // np.minimum(old, candidates)
                dec = nw < s.c;
                if (dec) {
                    const real_t ch = s.c - nw;
                    const unsigned long long b = bits_of(ch);
                    if (b > a_max) a_max = b;
                }
                Pn[q.c0 + lane] = nw;
            }
            const uint32_t bm = __ballot_sync(FULL, dec);
            if (lane == 0) a_dec += __popc(bm);
        }
        unsigned long long m = a_max;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long t = __shfl_xor_sync(FULL, m, o);
            m = t > m ? t : m;
        }
        const unsigned long long td = block_sum(a_dec, sred);
        if (lane == 0 && m) atomicMax(&ctl->cnt[(it % 3)], m);  // cnt[] slots hold max-change bits here
        if (threadIdx.x == 0) {
            if (td) atomicAdd(&ctl->dsum[it % 3], td);
            if (blockIdx.x == 0) {
                ctl->cnt[(it + 1) % 3] = 0;
                ctl->dsum[(it + 1) % 3] = 0;
            }
        }
        if (!grid_barrier(ctl)) return;
        const unsigned long long decs = vload(&ctl->dsum[it % 3]);
        const real_t maxch = real_of_bits(vload(&ctl->cnt[it % 3]));
        if (blockIdx.x == 0 && threadIdx.x == 0) ctl->iters = it + 1;
        if (decs == 0 || maxch < p.tol) break;  // E/oracle.py:59-62
        if (it + 1 >= p.cap) {                   // E/oracle.py:63-67
            if (blockIdx.x == 0 && threadIdx.x == 0) ctl->err = EIK_ECAP;
            break;
        }
    }
}

// ---------------------------------------------------------------------------
// FIM (E/fim.py:62-144): the paper's baseline, with the
// per-iteration neighbour checks iFIM drops.  One persistent launch, five
// grid barriers per iteration, phi updated in place between them:
//   1  values of the active list from the snapshot (stored per list slot)
//   2  settle (|v-old| <= tol -> SETTLED) or write and survive (:95-108)
//   3  every cell active this iteration examines its neighbours: fixed and
//      ACTIVE ones are skipped, +inf ones are activated once (claim bitmap),
//      finite ones are checks -- one counted call per examination, computed
//      once per distinct cell (:110-124)
//   4  values of the distinct checks from the post-phase-2 field
//   5  a check that drops by more than tol is written and re-activated (:126-138)
// Labels live in their own byte buffer, the claim bitmap in
// the R0 slot; both are cleared by the host before the launch.
// ---------------------------------------------------------------------------
constexpr uint8_t FIM_ACTIVE = 1, FIM_SETTLED = 2;  // E/fim.py:29 (FAR = 0)

template <int DIM, int SOL>
__device__ __forceinline__ real_t cell_solve(const KP &p, const real_t *P, uint32_t c, uint32_t x, uint32_t y,
                                             uint32_t z)
{
    Sten t;
    t.c = __ldcg(P + c);
    t.w = x > 0 ? __ldcg(P + c - 1) : INFINITY;
    t.e = x + 1 < (uint32_t)p.nx ? __ldcg(P + c + 1) : INFINITY;
    t.s = y > 0 ? __ldcg(P + c - p.nx32) : INFINITY;
    t.n = y + 1 < (uint32_t)p.ny ? __ldcg(P + c + p.nx32) : INFINITY;
    t.d = t.u = INFINITY;
    if (DIM == 3) {
        t.d = z > 0 ? __ldcg(P + c - p.plane32) : INFINITY;
        t.u = z + 1 < (uint32_t)p.nz ? __ldcg(P + c + p.plane32) : INFINITY;
    }
    t.k = coef<SOL>(p, c);
    return solve<DIM, SOL>(p, t);
}

template <int DIM>
__device__ __forceinline__ void cell_xyz(const KP &p, uint32_t c, uint32_t &x, uint32_t &y, uint32_t &z, uint32_t &row)
{
    row = fdiv(c, p.fnx);
    x = c - row * p.nx32;
    if (DIM == 3) {
        z = fdiv(row, p.fny);
        y = row - z * (uint32_t)p.ny;
    } else {
        z = 0;
        y = row;
    }
}

template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK) k_fim(KP p)
{
    __shared__ unsigned sscan[WPB + 1];
    __shared__ unsigned long long sred[WPB];
    Ctl *ctl = p.ctl;
    real_t *P = p.P0;
    real_t *V = p.P1;       // values per list slot (phases 1 and 4)
    uint8_t *lab = p.lab;  // FIM labels
    uint32_t *claim = p.R0b;
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x, nthr = gridDim.x * blockDim.x;
    const uint32_t bstride = gridDim.x * BLOCK;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    unsigned nA = vload(&ctl->len[0]);  // initial Active (k_init_active, E/fim.py:78-84)
    for (uint32_t i = tid; i < nA; i += nthr) lab[__ldcg(p.L0 + i)] = FIM_ACTIVE;
    if (lead) {
        ctl->peak = nA;
        ctl->sum = 0;
    }
    if (!grid_barrier(ctl)) return;
    for (int64_t it = 0; nA > 0; ++it) {
        if (it >= p.cap) {  // E/fim.py:90-92
            if (lead) ctl->err = EIK_ECAP;
            return;
        }
        const uint32_t *LA = (it & 1) ? p.L1 : p.L0;
        uint32_t *LN = (it & 1) ? p.L0 : p.L1;
        unsigned *lenN = &ctl->len[(it + 1) % 3];
        unsigned *lenC = &ctl->fc[it % 3];
        if (lead) {
            ctl->len[(it + 2) % 3] = 0;
            ctl->fc[(it + 1) % 3] = 0;
            ctl->iters = (unsigned long long)(it + 1);
            ctl->sum += nA;
        }
        // 1: values from the snapshot; clear the claims of last iteration's activations
        for (uint32_t i = tid; i < nA; i += nthr) {
            const uint32_t c = __ldcg(LA + i);
            uint32_t x, y, z, row;
            cell_xyz<DIM>(p, c, x, y, z, row);
            V[i] = cell_solve<DIM, SOL>(p, P, c, x, y, z);
            atomicAnd(claim + row * p.W + (x >> 5), ~(1u << (x & 31)));
        }
        if (!grid_barrier(ctl)) return;
        // 2: settle or write and survive
        unsigned long long wr = 0;
        for (uint32_t base = blockIdx.x * BLOCK; base < nA; base += bstride) {
            const uint32_t i = base + threadIdx.x;
            unsigned stay = 0;
            uint32_t c = 0;
            if (i < nA) {
                c = __ldcg(LA + i);
                const real_t v = V[i], old = __ldcg(P + c);
                if (v == old || fabs(v - old) <= tol_at(p.tol, old)) {
                    lab[c] = FIM_SETTLED;
                } else {
                    P[c] = v;
                    stay = 1;
                    ++wr;
                }
            }
            const unsigned pos = block_reserve(stay, lenN, sscan);
            if (stay) LN[pos] = c;
        }
        if (!grid_barrier(ctl)) return;
        // 3: neighbour examination
        unsigned long long pairs = 0;
        for (uint32_t base = blockIdx.x * BLOCK; base < nA; base += bstride) {
            const uint32_t i = base + threadIdx.x;
            uint32_t act[6], chk[6];
            unsigned na = 0, nc = 0;
            if (i < nA) {
                const uint32_t c = __ldcg(LA + i);
                uint32_t x, y, z, row;
                cell_xyz<DIM>(p, c, x, y, z, row);
#pragma unroll
                for (int k = 0; k < (DIM == 3 ? 6 : 4); ++k) {
                    const bool inb = k == 0 ? x > 0 : k == 1 ? x + 1 < p.nx32 : k == 2 ? y > 0
                                     : k == 3 ? y + 1 < (uint32_t)p.ny : k == 4 ? z > 0 : z + 1 < (uint32_t)p.nz;
                    if (!inb) continue;
                    const uint32_t e = k == 0 ? c - 1 : k == 1 ? c + 1 : k == 2 ? c - p.nx32 : k == 3 ? c + p.nx32
                                       : k == 4 ? c - p.plane32 : c + p.plane32;
                    const uint32_t xe = k == 0 ? x - 1 : k == 1 ? x + 1 : x;
                    const uint32_t re = k == 2 ? row - 1 : k == 3 ? row + 1 : k == 4 ? row - (uint32_t)p.ny
                                        : k == 5 ? row + (uint32_t)p.ny : row;
                    const uint32_t w = re * p.W + (xe >> 5), bit = 1u << (xe & 31);
                    if (__ldg(p.Fb + w) & bit) continue;  // blocked or seed
                    if (*(volatile uint8_t *)(lab + e) == FIM_ACTIVE) continue;
                    const bool unreached = __ldcg(P + e) == INFINITY;
                    if (!unreached) ++pairs;  // one counted call per examination (E/fim.py:124)
                    if (atomicOr(claim + w, bit) & bit) continue;
                    if (unreached) {
                        lab[e] = FIM_ACTIVE;
                        act[na++] = e;
                    } else {
                        chk[nc++] = e;
                    }
                }
            }
            unsigned pos = block_reserve(na, lenN, sscan);
            for (unsigned q = 0; q < na; ++q) LN[pos + q] = act[q];
            pos = block_reserve(nc, lenC, sscan);
            for (unsigned q = 0; q < nc; ++q) p.L2[pos + q] = chk[q];
        }
        {
            const unsigned long long t = block_sum(pairs, sred);
            if (threadIdx.x == 0 && t) atomicAdd(&ctl->sum, t);
        }
        if (!grid_barrier(ctl)) return;
        // 4: values of the distinct checks from the post-phase-2 field
        const unsigned nC = vload(lenC);
        for (uint32_t j = tid; j < nC; j += nthr) {
            const uint32_t c = __ldcg(p.L2 + j);
            uint32_t x, y, z, row;
            cell_xyz<DIM>(p, c, x, y, z, row);
            V[j] = cell_solve<DIM, SOL>(p, P, c, x, y, z);
        }
        if (!grid_barrier(ctl)) return;
        // 5: re-activate checks that dropped by more than tol
        for (uint32_t base = blockIdx.x * BLOCK; base < nC; base += bstride) {
            const uint32_t j = base + threadIdx.x;
            unsigned go = 0;
            uint32_t c = 0;
            if (j < nC) {
                c = __ldcg(p.L2 + j);
                uint32_t x, y, z, row;
                cell_xyz<DIM>(p, c, x, y, z, row);
                atomicAnd(claim + row * p.W + (x >> 5), ~(1u << (x & 31)));
                const real_t v = V[j], old = __ldcg(P + c);
                if (v < old - tol_at(p.tol, old)) {  // E/fim.py:135
                    P[c] = v;
                    lab[c] = FIM_ACTIVE;
                    go = 1;
                    ++wr;
                }
            }
            const unsigned pos = block_reserve(go, lenN, sscan);
            if (go) LN[pos] = c;
        }
        {
            const unsigned long long t = block_sum(wr, sred);
            if (threadIdx.x == 0 && t) atomicAdd(&ctl->writes, t);
        }
        if (!grid_barrier(ctl)) return;
        nA = vload(lenN);
        if (lead && nA > ctl->peak) ctl->peak = nA;
    }
}

// max_residual (E/harness.py:147-162): max |phi - U(phi)| over free cells with
// finite phi; result as IEEE bits in ctl->peak.
template <int DIM, int SOL>
__global__ void __launch_bounds__(BLOCK) k_residual(KP p)
{
    const unsigned lane = lane_id();
    const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const uint32_t GW = (gridDim.x * blockDim.x) >> 5;
    unsigned long long a_max = 0;
    for (uint32_t w = gw; w < p.nwords; w += GW) {
        const WPos q = wpos<DIM>(p, w);
        const uint32_t freem = q.rowm & ~__ldg(p.Fb + w);
        if (freem == 0) continue;
        Sten s;
        gather<DIM, SOL>(p, p.P0, q, freem, s);
        if (((freem >> lane) & 1u) && s.c < INFINITY) {
            const real_t r = fabs(s.c - solve<DIM, SOL>(p, s));
            const unsigned long long b = bits_of(r);
            if (r == r && b > a_max) a_max = b;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(FULL, a_max, o);
        a_max = t > a_max ? t : a_max;
    }
    if (lane == 0 && a_max) atomicMax(&p.ctl->peak, a_max);
}

// Slab mode: activation requests from the neighbour ranks (their ghost-plane
// touched words) for the owned boundary planes; a requested cell is activated
// iff it is still FAR here (blocked cells are pre-touched).  The requester's
// +inf test used the same snapshot value.  Appends to the next list of `it`.
#if !EIK_SINGLE
__global__ void k_apply_requests(KP p, const uint32_t *req_lo, const uint32_t *req_hi, int64_t it)
{
    const uint32_t planeW = (uint32_t)p.ny * p.W;
    uint32_t *Ln = (it & 1) ? p.L0 : p.L1;
    unsigned *lenN = &p.ctl->len[(it + 1) % 3];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < 2 * planeW; i += gridDim.x * blockDim.x) {
        const bool hi = i >= planeW;
        const uint32_t j = hi ? i - planeW : i;
        const uint32_t *req = hi ? req_hi : req_lo;
        if (!req) continue;
        const uint32_t m = req[j];
        if (!m) continue;
        const uint32_t z = hi ? (uint32_t)p.nz - 2 : 1u;
        const uint32_t w = z * planeW + j;
        const uint32_t nb = m & ~atomicOr(p.Bt + w, m);
        if (!nb) continue;
        const uint32_t row = w / p.W, c0 = row * p.nx32 + (w - row * p.W) * 32u;
        for (uint32_t b = nb; b; b &= b - 1) Ln[atomicAdd(lenN, 1u)] = c0 + (uint32_t)(__ffs(b) - 1);
    }
}
#endif

// Element-wise local solver (parity hook).
__global__ void k_local(int kind, const real_t *a, const real_t *b, const real_t *c, const real_t *f, real_t dx,
                        real_t dy, real_t *out, int64_t n)
{
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const real_t h = dx > 0 ? dx : out[i];  // dx <= 0: each element's spacing is passed in out[i]
        if (kind == 0) out[i] = upd2u(a[i], b[i], h / f[i]);
        else if (kind == 1) out[i] = upd2a(a[i], b[i], f[i], h, dy);
        else out[i] = upd3u(a[i], b[i], c[i], h / f[i], h);
    }
}

// ---------------------------------------------------------------------------
// Verification reductions on device fields (E/harness.py:165-179, SURVEY.md
// §8f rank 2): no full-field host copy at 512^3-1024^3.
//   k_max_diff   max |a - b| with equal same-sign infinities counting 0 and NaN
//                propagating (np.where(both_inf, 0, |a - b|).max())
//   k_sha256_chunks  SHA-256 of each `chunk`-byte piece of a byte range (one thread per
//                piece, FIPS 180-4); the host hashes the concatenated piece digests.
// ---------------------------------------------------------------------------
__global__ void k_max_diff(const real_t *__restrict__ a, const real_t *__restrict__ b, int64_t n,
                           unsigned long long *out)
{
    unsigned long long m = 0;
    unsigned nan = 0;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const real_t x = __ldcs(a + i), y = __ldcs(b + i);
        if (isinf(x) && isinf(y) && ((x > R_ZERO) == (y > R_ZERO))) continue;  // both_inf: 0
        const real_t d = fabs(x - y);
        if (!(d == d)) {
            nan = 1;
            continue;
        }
        const unsigned long long bb = bits_of(d);
        m = bb > m ? bb : m;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(FULL, m, o);
        m = t > m ? t : m;
    }
    nan = __any_sync(FULL, nan);
    if (lane_id() == 0) {
        if (m) atomicMax(out, m);
        if (nan) atomicOr(out + 1, 1ull);
    }
}

__constant__ uint32_t kSha256K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u, 0x923f82a4u, 0xab1c5ed5u,
    0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u, 0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u,
    0xe49b69c1u, 0xefbe4786u, 0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u, 0x06ca6351u, 0x14292967u,
    0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u, 0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u,
    0xa2bfe8a1u, 0xa81a664bu, 0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au, 0x5b9cca4fu, 0x682e6ff3u,
    0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u, 0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) { return __funnelshift_r(x, x, n); }

__device__ void sha256_block(uint32_t h[8], uint32_t w[16])
{
    uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5], g = h[6], k = h[7];
#pragma unroll
    for (int i = 0; i < 64; ++i) {
        uint32_t wi;
        if (i < 16) {
            wi = w[i];
        } else {
            const uint32_t w15 = w[(i - 15) & 15], w2 = w[(i - 2) & 15];
            const uint32_t s0 = rotr32(w15, 7) ^ rotr32(w15, 18) ^ (w15 >> 3);
            const uint32_t s1 = rotr32(w2, 17) ^ rotr32(w2, 19) ^ (w2 >> 10);
            wi = w[i & 15] = w[i & 15] + s0 + w[(i - 7) & 15] + s1;
        }
        const uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
        const uint32_t ch = (e & f) ^ (~e & g);
        const uint32_t t1 = k + S1 + ch + kSha256K[i] + wi;
        const uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
        const uint32_t mj = (a & b) ^ (a & c) ^ (b & c);
        const uint32_t t2 = S0 + mj;
        k = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    h[0] += a; h[1] += b; h[2] += c; h[3] += d; h[4] += e; h[5] += f; h[6] += g; h[7] += k;
}

__global__ void k_sha256_chunks(const uint8_t *__restrict__ data, uint64_t nbytes, uint64_t chunk, uint64_t nchunks,
                                uint8_t *__restrict__ dig)
{
    const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
    if (i >= nchunks) return;
    const uint8_t *p = data + i * chunk;
    const uint64_t len = min(chunk, nbytes - i * chunk);
    uint32_t h[8] = {0x6a09e667u, 0xbb67ae85u, 0x3c6ef372u, 0xa54ff53au,
                     0x510e527fu, 0x9b05688cu, 0x1f83d9abu, 0x5be0cd19u};
    uint32_t w[16];
    const uint64_t nfull = len / 64;
    for (uint64_t blk = 0; blk < nfull; ++blk) {
        const uint4 *q = (const uint4 *)(p + blk * 64);  // chunk and base are 16-byte aligned
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const uint4 x = __ldcs(q + v);
            w[4 * v + 0] = __byte_perm(x.x, 0, 0x0123);
            w[4 * v + 1] = __byte_perm(x.y, 0, 0x0123);
            w[4 * v + 2] = __byte_perm(x.z, 0, 0x0123);
            w[4 * v + 3] = __byte_perm(x.w, 0, 0x0123);
        }
        sha256_block(h, w);
    }
    // tail: the remaining bytes, 0x80, zeros, 64-bit big-endian bit length (one or two blocks)
    const uint32_t rem = (uint32_t)(len - nfull * 64);
    const uint8_t *t = p + nfull * 64;
    const uint64_t bits = len * 8;
    const int nblk = rem + 9 <= 64 ? 1 : 2;
    for (int bk = 0; bk < nblk; ++bk) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            uint32_t word = 0;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const uint32_t pos = (uint32_t)(bk * 64 + 4 * j + q);
                uint32_t byte = 0;
                if (pos < rem) byte = t[pos];
                else if (pos == rem) byte = 0x80u;
                else if (bk == nblk - 1 && 4 * j + q >= 56) byte = (uint32_t)(bits >> (8 * (63 - (4 * j + q)))) & 0xffu;
                word = (word << 8) | byte;
            }
            w[j] = word;
        }
        sha256_block(h, w);
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        dig[32 * i + 4 * j + 0] = (uint8_t)(h[j] >> 24);
        dig[32 * i + 4 * j + 1] = (uint8_t)(h[j] >> 16);
        dig[32 * i + 4 * j + 2] = (uint8_t)(h[j] >> 8);
        dig[32 * i + 4 * j + 3] = (uint8_t)h[j];
    }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------

thread_local std::string g_err;
thread_local int g_remedy_engine = 0;  // eik_last_remedy_engine()

// NVTX range over a scope (host side: the enqueue of a phase's kernels; SURVEY.md §5 tracing)
struct Nvtx {
    explicit Nvtx(const char *name) { nvtxRangePushA(name); }
    ~Nvtx() { nvtxRangePop(); }
};

int fail(int code, const char *fmt, ...)
{
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

#define CK(call)                                                                                \
    do {                                                                                        \
        cudaError_t e_ = (call);                                                                \
        if (e_ != cudaSuccess) return fail(EIK_ECUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

struct Layout {
    int64_t N;
    uint32_t W, nwords, npos, nty4, ntt;
    size_t off_phi2, off_dd, off_bt, off_l0, off_l1, off_l2;
    size_t off_r0, off_d0, off_d1, off_f, off_lab;
    size_t off_hist, off_ctl_u, off_ctl_r, off_kps, total;
    size_t off_ft, off_sb, off_dt0, off_dt1, off_st0, off_st1, off_grab;  // remedy tile engine
    uint32_t tnty, tntz, ntiles;
    size_t off_brec0, off_brec1, off_bfix, off_bmask, off_blist0, off_blist1, off_bcnt;  // brick engine
    uint32_t nbx, nby, nbz, nbricks;
    int64_t cap_upd, cap_rem;
};

int make_layout(const eik_geom *g, Layout &L)
{
    if (!g) return fail(EIK_EINVAL, "null geometry");
    if (g->ndim != 2 && g->ndim != 3) return fail(EIK_EINVAL, "ndim must be 2 or 3, got %d", g->ndim);
    if (g->nx < 1 || g->ny < 1 || g->nz < 1) return fail(EIK_EINVAL, "grid must have at least one cell");
    if (g->ndim == 2 && g->nz != 1) return fail(EIK_EINVAL, "2D grid must have nz == 1");
    if (!(g->dx > 0) || !(g->dy > 0) || !(g->dz > 0)) return fail(EIK_EINVAL, "grid spacing must be positive");
    if (g->ndim == 3 && !(g->dx == g->dy && g->dy == g->dz))
        return fail(EIK_EINVAL, "3D grids require dx == dy == dz (no anisotropic 3D solver, SPEC.md:169)");
    if (g->dtype != EIK_DTYPE)
        return fail(EIK_EINVAL, EIK_SINGLE ? "this library is the float32 engine (dtype EIK_SINGLE)" : "this library is the float64 engine (dtype EIK_F64)");
    if ((g->flags & EIK_GEOM_SLAB) && (g->ndim != 3 || g->nz < 3))
        return fail(EIK_EINVAL, "a slab is 3D with at least one owned plane plus two ghost planes");
    L.N = g->nx * g->ny * g->nz;
    if (L.N >= (int64_t)1 << 31)
        return fail(EIK_EINVAL, "grid too large: %lld cells (limit 2^31 per device)", (long long)L.N);
    const int64_t W = (g->nx + 31) / 32;
    const int64_t nw = W * g->ny * g->nz;
    L.W = (uint32_t)W;
    L.nwords = (uint32_t)nw;
    const int64_t s = g->nx + g->ny + (g->ndim == 3 ? g->nz : 0);
    L.cap_upd = 40 * s;  // E/ifim.py:106 (2D: 40*(nx+ny))
    L.cap_rem = 20 * s;  // E/ifim.py:185
    const size_t bm = (size_t)nw * 4;
    size_t o = 0;
    L.off_phi2 = o; o += al((size_t)L.N * sizeof(real_t));
    L.off_dd = o; o += al((size_t)L.N * sizeof(real_t));
    L.off_bt = o; o += al(bm);
    L.off_l0 = o; o += al((size_t)L.N * 4);  // update: active cells; remedy: members
    L.off_l1 = o; o += al((size_t)L.N * 4);
    L.off_l2 = o; o += al((size_t)L.N * 4);  // FIM check list
    L.off_r0 = o; o += al(bm);
    L.off_d0 = o; o += al(bm);
    L.off_d1 = o; o += al(bm);
    L.off_f = o; o += al(bm);
    L.off_lab = o; o += al((size_t)L.N);  // FIM labels
    L.off_hist = o; o += al((size_t)(L.cap_upd + 2) * 8);
    L.off_ctl_u = o; o += al(sizeof(Ctl));
    L.off_ctl_r = o; o += al(sizeof(Ctl));
    L.off_kps = o; o += al(2 * EIK_MAX_RANKS * sizeof(KP));
    // remedy tile engine: 32 x-cells x (8 y x 4 z) rows per tile in 3D, 32 x 32 in 2D
    {
        const int ly = g->ndim == 3 ? 3 : 5, lz = g->ndim == 3 ? 2 : 0;
        L.tnty = (uint32_t)((g->ny + (1 << ly) - 1) >> ly);
        L.tntz = (uint32_t)((g->nz + (1 << lz) - 1) >> lz);
        const int64_t nt = W * (int64_t)L.tnty * L.tntz;
        if (nt * 32 >= ((int64_t)1 << 32)) return fail(EIK_EINVAL, "grid too large for the tile bitmaps");
        L.ntiles = (uint32_t)nt;
        const size_t tb = (size_t)nt * 32 * 4;
        L.off_ft = o; o += al(tb);
        L.off_sb = o; o += al(tb);
        L.off_dt0 = o; o += al(tb);
        L.off_dt1 = o; o += al(tb);
        L.off_st0 = o; o += al((size_t)nt * 4);
        L.off_st1 = o; o += al((size_t)nt * 4);
        L.off_grab = o; o += al((size_t)3 * 32 * RT_GS * 4);
    }
    // remedy brick engine (3D): 32 x 8 x 8 bricks
    {
        L.nbx = (uint32_t)W;
        L.nby = (uint32_t)((g->ny + 7) / 8);
        L.nbz = g->ndim == 3 ? (uint32_t)((g->nz + 7) / 8) : 1u;
        L.nbricks = L.nbx * L.nby * L.nbz;
        const size_t nb = L.nbricks;
        L.off_brec0 = o; o += al(nb * 512);
        L.off_brec1 = o; o += al(nb * 512);
        L.off_bfix = o; o += al(nb * 256);
        L.off_bmask = o; o += al(3 * nb * 4);
        L.off_blist0 = o; o += al(nb * 4);
        L.off_blist1 = o; o += al(nb * 4);
        L.off_bcnt = o; o += al(8 * 128);
    }
    // member-list traversal (word_at): 3D groups of 4x4 rows, 2D groups of 16 rows, per x-word
    if (g->ndim == 3) {
        L.nty4 = (uint32_t)((g->ny + (1 << TILE_LY) - 1) >> TILE_LY);
        L.ntt = (uint32_t)((g->nz + (1 << TILE_LZ) - 1) >> TILE_LZ);
        L.npos = (L.nty4 * L.ntt << (TILE_LY + TILE_LZ)) * L.W;
    } else {
        L.nty4 = 0;
        L.ntt = (uint32_t)((g->ny + (1 << TILE_L2D) - 1) >> TILE_L2D);
        L.npos = (L.ntt << TILE_L2D) * L.W;
    }
    L.total = o;
    return EIK_OK;
}

int solver_kind(const eik_geom *g)
{
    if (g->ndim == 3) return SOL_U3;
    return g->dx == g->dy ? SOL_U2 : SOL_A2;  // E/_kernels.py:41-44
}

KP make_kp(const eik_geom *g, const Layout &L, void *ws, real_t *phi, const real_t *speed, const uint8_t *state,
           double tol, Ctl *ctl, int64_t cap)
{
    char *b = (char *)ws;
    KP p;
    memset(&p, 0, sizeof(p));
    p.nx = g->nx; p.ny = g->ny; p.nz = g->nz; p.plane = g->nx * g->ny;
    p.W = L.W; p.nwords = L.nwords; p.nrows = (uint32_t)(g->ny * g->nz);
    p.nx32 = (uint32_t)g->nx;
    p.plane32 = (uint32_t)(g->nx * g->ny);
    p.ncells = (uint32_t)(g->nx * g->ny * g->nz);
    p.fnx = make_fastdiv((uint32_t)g->nx);
    p.fny = make_fastdiv((uint32_t)g->ny);
    p.fW = make_fastdiv(L.W);
    p.nty4 = L.nty4;
    p.fnty4 = make_fastdiv(L.nty4 ? L.nty4 : 1);
    p.npos = L.npos;
    p.dx = g->dx; p.dy = g->dy; p.delta = g->dx; p.tol = tol;
    p.slab = (g->flags & EIK_GEOM_SLAB) ? 1 : 0;
    p.it0 = 0;
    p.max_it = (int64_t)1 << 40;
    p.P0 = phi;
    p.P1 = (real_t *)(b + L.off_phi2);
    p.F = speed;
    p.dd = (real_t *)(b + L.off_dd);
    p.state = state;
    p.Bt = (uint32_t *)(b + L.off_bt);
    p.L0 = (uint32_t *)(b + L.off_l0);
    p.L1 = (uint32_t *)(b + L.off_l1);
    p.L2 = (uint32_t *)(b + L.off_l2);
    p.ctl = ctl;
    p.hist = (int64_t *)(b + L.off_hist);
    p.hist_cap = L.cap_upd + 2;
    p.cap = cap;
    p.R0b = (uint32_t *)(b + L.off_r0);
    p.D0b = (uint32_t *)(b + L.off_d0);
    p.D1b = (uint32_t *)(b + L.off_d1);
    p.Fb = (uint32_t *)(b + L.off_f);
    p.lab = (uint8_t *)(b + L.off_lab);
    p.nty = L.tnty;
    p.ntz = L.tntz;
    p.ntiles = L.ntiles;
    p.rt_shs = (L.ntiles + RT_SHARDS - 1) / RT_SHARDS;
    p.fnty = make_fastdiv(L.tnty);
    p.Ft = (uint32_t *)(b + L.off_ft);
    p.St = (uint32_t *)(b + L.off_sb);
    p.Dt0 = (uint32_t *)(b + L.off_dt0);
    p.Dt1 = (uint32_t *)(b + L.off_dt1);
    p.stamp0 = (uint32_t *)(b + L.off_st0);
    p.stamp1 = (uint32_t *)(b + L.off_st1);
    p.grab = (unsigned *)(b + L.off_grab);
    p.nbx = L.nbx; p.nby = L.nby; p.nbz = L.nbz; p.nbricks = L.nbricks;
    p.fnbx = make_fastdiv(L.nbx);
    p.fnby = make_fastdiv(L.nby);
    p.brec0 = (uint32_t *)(b + L.off_brec0);
    p.brec1 = (uint32_t *)(b + L.off_brec1);
    p.bfix = (uint32_t *)(b + L.off_bfix);
    p.bmask = (uint32_t *)(b + L.off_bmask);
    p.blist0 = (uint32_t *)(b + L.off_blist0);
    p.blist1 = (uint32_t *)(b + L.off_blist1);
    p.bcnt = (unsigned *)(b + L.off_bcnt);
    p.bsel = p.bcnt + 6 * 32;
    return p;
}

int g_sms = 0;

int num_sms()
{
    if (!g_sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g_sms, cudaDevAttrMultiProcessorCount, dev);
        if (g_sms <= 0) g_sms = 148;
    }
    return g_sms;
}

int stream_grid(int64_t work_warps)
{
    int64_t blocks = (work_warps + WPB - 1) / WPB;
    const int64_t mx = (int64_t)num_sms() * 8;
    if (blocks > mx) blocks = mx;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

template <typename K>
int coop_launch(K kernel, KP &p, const unsigned *skip, bool with_skip, cudaStream_t st, const char *env_name,
                int default_per_sm, int nt = BLOCK)
{
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, nt, 0);
    if (e != cudaSuccess) return fail(EIK_ECUDA, "occupancy: %s", cudaGetErrorString(e));
    int per_sm = (default_per_sm > 0 && default_per_sm < occ) ? default_per_sm : occ;
    if (const char *env = getenv(env_name)) {  // tuning override, bounded only by the occupancy limit
        const int v = atoi(env);
        if (v > 0 && v <= occ) per_sm = v;
        else if (v > occ) fprintf(stderr, "[eik] %s=%d exceeds the occupancy limit %d; using %d\n", env_name, v, occ, per_sm);
    }
    if (per_sm < 1) return fail(EIK_ECUDA, "persistent kernel cannot be resident");
    dim3 grid(per_sm * num_sms()), block(nt);
    void *args2[] = {&p, (void *)&skip};
    void *args1[] = {&p};
    e = cudaLaunchCooperativeKernel((const void *)kernel, grid, block, with_skip ? args2 : args1, 0, st);
    if (e != cudaSuccess) return fail(EIK_ECUDA, "cooperative launch: %s", cudaGetErrorString(e));
    return EIK_OK;
}

// Cooperative launch of a multi-rank kernel: nlocal rank groups, each with the
// same number of CTAs; each CTA finds its rank's KP in kps_dev[blockIdx.x / per_group].
template <typename K>
int coop_launch_groups(K kernel, const KP *kps_dev, int nlocal, cudaStream_t st, int &per_group_out)
{
    int per_sm = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, BLOCK, 0);
    if (e != cudaSuccess) return fail(EIK_ECUDA, "occupancy: %s", cudaGetErrorString(e));
    const int total = per_sm * num_sms();
    uint32_t per_group = (uint32_t)(total / nlocal);
    if (per_group < 1) return fail(EIK_EINVAL, "too many ranks on one device");
    per_group_out = (int)per_group;
    dim3 grid(per_group * nlocal), block(BLOCK);
    void *args[] = {(void *)&kps_dev, &per_group};
    e = cudaLaunchCooperativeKernel((const void *)kernel, grid, block, args, 0, st);
    if (e != cudaSuccess) return fail(EIK_ECUDA, "cooperative launch: %s", cudaGetErrorString(e));
    return EIK_OK;
}

// TMA descriptors (cuTensorMapEncodeTiled through the runtime's driver entry point: no -lcuda)
int encode_3d(CUtensorMap *tm, CUtensorMapDataType dt, size_t esz, const void *base, uint64_t nx, uint64_t ny,
              uint64_t nz, uint32_t bx, uint32_t by, uint32_t bz)
{
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !f)
            return fail(EIK_ECUDA, "cuTensorMapEncodeTiled is not available");
        fn = (PFN_cuTensorMapEncodeTiled_v12000)f;
    }
    const cuuint64_t dims[3] = {nx, ny, nz};
    const cuuint64_t strides[2] = {nx * esz, nx * ny * esz};
    const cuuint32_t box[3] = {bx, by, bz}, es[3] = {1, 1, 1};
    const CUresult r = fn(tm, dt, 3, const_cast<void *>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                          CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(EIK_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return EIK_OK;
}

// |R_0| share of the grid (percent) from which the device picks the brick engine (auto mode).
// Measured (docs/PERF_LOG.md): cfg4 512^3 (|R_0| 4.9 %) member list 268 vs brick 336 ms;
// cfg5 512^3 (53 %) 322 vs 307 ms, cfg5 1024^3 4.60 vs 4.06 s; cfg3 256^3 4.3 vs 4.8 ms.
#ifndef BRK_DENSE_PCT
#define BRK_DENSE_PCT 20
#endif
int brick_dense_pct()
{
    if (const char *e = getenv("EIK_BRICK_DENSE_PCT")) return atoi(e);
    return BRK_DENSE_PCT;
}

// The brick engine needs TMA-legal strides (16-byte multiples), a box no larger than the grid
// and 16-byte-aligned fields.
bool brick_eligible(const KP &p)
{
    const uint64_t rowb = (uint64_t)p.nx32 * sizeof(real_t);
    return !p.mr && !p.slab && p.nz > 1 && rowb % 16 == 0 && p.nx32 >= (uint32_t)brk::HX && p.ny >= brk::HY &&
           p.nz >= brk::HZ && ((uintptr_t)p.P0 & 15) == 0 && ((uintptr_t)p.P1 & 15) == 0 && ((uintptr_t)p.dd & 15) == 0;
}

template <int DIM, int SOL>
struct Engine {
    // phi copy (optional), d = delta/F, touched (optional) and the fixed brick bitmap
    static int prep(KP &p, bool copy_phi, bool touched, cudaStream_t st)
    {
        const int grid = stream_grid(p.nwords);
        if (p.Ft) CK(cudaMemsetAsync(p.Ft, 0xff, (size_t)p.ntiles * 32 * 4, st));  // padding rows: fixed
        if (SOL == SOL_A2) k_prep<DIM, false><<<grid, BLOCK, 0, st>>>(p, copy_phi, touched);
        else k_prep<DIM, true><<<grid, BLOCK, 0, st>>>(p, copy_phi, touched);
        CK(cudaGetLastError());
        return EIK_OK;
    }
    static int init_active(KP &p, const int64_t *seeds, int64_t ns, cudaStream_t st)
    {
        const int grid = (int)std::min<int64_t>((ns + 255) / 256, 1024);
        k_init_active<DIM><<<grid > 0 ? grid : 1, 256, 0, st>>>(p, seeds, ns);
        CK(cudaGetLastError());
        return EIK_OK;
    }
    static int update(KP &p, cudaStream_t st)
    {
        // 2D fronts are O(n) cells: one CTA per SM keeps the per-iteration barrier cheap
        // (cfg2 4096^2: 29 vs 34 ms); 3D fronts are O(n^2) and want the full occupancy
        return coop_launch(k_update<DIM, SOL>, p, nullptr, false, st, "EIK_UPD_BLOCKS_PER_SM", DIM == 2 ? UPD_2D_PER_SM : 0);
    }
    // remedy-set slots: counters (R0 is rewritten word by word)
    static int reset_set(KP &p, cudaStream_t st)
    {
        if (p.mr) {  // keep bar_* / wcount / wgen: peers may already be waiting at the world barrier
            CK(cudaMemsetAsync(&p.ctl->len[0], 0, offsetof(Ctl, nz_sectors) + sizeof(unsigned long long) -
                                                     offsetof(Ctl, len), st));
        } else {
            CK(cudaMemsetAsync(p.ctl, 0, sizeof(Ctl), st));
        }
        return EIK_OK;
    }
    static int build(KP &p, const real_t *Pc, const unsigned *skip, cudaStream_t st)
    {
        int rc = reset_set(p, st);
        if (rc) return rc;
        k_build<DIM, SOL><<<stream_grid(p.nwords), BLOCK, 0, st>>>(p, Pc, skip);
        CK(cudaGetLastError());
        return EIK_OK;
    }
    static int load(KP &p, const uint8_t *cells, const uint8_t *member, cudaStream_t st)
    {
        int rc = reset_set(p, st);
        if (rc) return rc;
        if (member) CK(cudaMemsetAsync(p.St, 0, (size_t)p.ntiles * 32 * 4, st));  // padding rows
        k_remedy_load<DIM><<<stream_grid(p.nwords), BLOCK, 0, st>>>(p, cells, member);
        CK(cudaGetLastError());
        return EIK_OK;
    }
    static int do_export(KP &p, uint8_t *member, cudaStream_t st)
    {
        k_remedy_export<DIM><<<stream_grid(p.nwords), BLOCK, 0, st>>>(p, member);
        CK(cudaGetLastError());
        return EIK_OK;
    }
    static int update_mr(const KP *kps_dev, int nlocal, cudaStream_t st, int &per_group_out)
    {
        return coop_launch_groups(k_update_mr<DIM, SOL>, kps_dev, nlocal, st, per_group_out);
    }
    static int remedy_mr(const KP *kps_dev, int nlocal, cudaStream_t st, int &per_group_out)
    {
        return coop_launch_groups(k_remedy_mr<DIM, SOL>, kps_dev, nlocal, st, per_group_out);
    }
    static int fixpoint(KP &p, cudaStream_t st)
    {
        return coop_launch(k_fixpoint<DIM, SOL>, p, nullptr, false, st, "EIK_FIX_BLOCKS_PER_SM", 0);
    }
    static int fim(KP &p, cudaStream_t st)
    {
        return coop_launch(k_fim<DIM, SOL>, p, nullptr, false, st, "EIK_FIM_BLOCKS_PER_SM", 0);
    }
    static int residual(KP &p, cudaStream_t st)
    {
        k_residual<DIM, SOL><<<stream_grid(p.nwords), BLOCK, 0, st>>>(p);
        CK(cudaGetLastError());
        return EIK_OK;
    }
    static int remedy(KP &p, const unsigned *skip, cudaStream_t st)
    {
        return coop_launch(k_remedy<DIM, SOL>, p, skip, true, st, "EIK_REM_BLOCKS_PER_SM", 0, REM_NT);
    }
    // single device: EIK_REMEDY=list (member-list kernel) or tile (tile engine); hand-built sets
    // with members outside their work list need the tile engine
    // brick engine (eik_remedy_tma.cuh): TMA-staged bricks, 3D single device
    static int remedy_brick(KP &p, const unsigned *skip, cudaStream_t st)
    {
        const CUtensorMapDataType dt = sizeof(real_t) == 8 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32;
        CUtensorMap m0, m1, md;
        int rc = encode_3d(&m0, dt, sizeof(real_t), p.P0, p.nx32, p.ny, p.nz, brk::HX, brk::HY, brk::HZ);
        if (!rc) rc = encode_3d(&m1, dt, sizeof(real_t), p.P1, p.nx32, p.ny, p.nz, brk::HX, brk::HY, brk::HZ);
        if (!rc) rc = encode_3d(&md, dt, sizeof(real_t), p.dd, p.nx32, p.ny, p.nz, brk::BX, brk::BY, brk::BZ);
        if (rc) return rc;
        CK(cudaMemsetAsync(p.bmask, 0, (size_t)3 * p.nbricks * 4, st));
        CK(cudaMemsetAsync(p.bcnt, 0, 6 * 128, st));
        k_brick_prep<<<stream_grid((int64_t)p.nbricks), 256, 0, st>>>(p, skip);
        CK(cudaGetLastError());
        auto kern = k_remedy_b<SOL>;
        CK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)brk::SMEM));
        int occ = 0;
        CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, brk::THREADS, brk::SMEM));
        if (const char *env = getenv("EIK_BRK_BLOCKS_PER_SM")) {
            const int v = atoi(env);
            if (v > 0 && v <= occ) occ = v;
        }
        if (occ < 1) return fail(EIK_ECUDA, "brick remedy kernel cannot be resident");
        dim3 grid(occ * num_sms()), block(brk::THREADS);
        void *args[] = {&p, (void *)&skip, &m0, &m1, &md};
        const cudaError_t e = cudaLaunchCooperativeKernel((const void *)kern, grid, block, args, brk::SMEM, st);
        if (e != cudaSuccess) return fail(EIK_ECUDA, "cooperative launch (brick remedy): %s", cudaGetErrorString(e));
        return EIK_OK;
    }
    static int remedy_single(KP &p, const unsigned *skip, cudaStream_t st, bool need_tile = false)
    {
        const char *mode = getenv("EIK_REMEDY");
        if constexpr (DIM == 3 && SOL == SOL_U3) {
            if (!need_tile && brick_eligible(p)) {
                if (mode && strcmp(mode, "brick") == 0) {
                    g_remedy_engine = 3;
                    return remedy_brick(p, skip, st);
                }
                if (!mode || strcmp(mode, "auto") == 0) {
                    // chosen on the device from |R_0| (no host sync): the brick pipeline for dense
                    // sets, the member list for sparse ones; the other kernel exits at once
                    k_choose_remedy<<<1, 1, 0, st>>>(p.ctl, skip, p.bsel, (unsigned long long)p.ncells,
                                                     (unsigned)brick_dense_pct());
                    CK(cudaGetLastError());
                    int rc = remedy(p, p.bsel, st);
                    if (!rc) rc = remedy_brick(p, p.bsel + 32, st);
                    g_remedy_engine = 4;  // resolved from Ctl::engine after the solve's sync
                    return rc;
                }
            }
        }
        const bool tile = need_tile || (mode ? strcmp(mode, "tile") == 0 : REMEDY_TILE_DEFAULT);
        g_remedy_engine = tile ? 2 : 1;
        if (!tile) return remedy(p, skip, st);
        CK(cudaMemsetAsync(p.stamp0, 0, (size_t)p.ntiles * 4, st));
        CK(cudaMemsetAsync(p.stamp1, 0, (size_t)p.ntiles * 4, st));
        CK(cudaMemsetAsync(p.grab, 0, (size_t)3 * 32 * RT_GS * 4, st));
        return coop_launch(k_remedy_t<DIM, SOL>, p, skip, true, st, "EIK_REM_BLOCKS_PER_SM", 0);
    }
};

template <typename F>
int dispatch(const eik_geom *g, F &&f)
{
    switch (solver_kind(g)) {
        case SOL_U2: return f(Engine<2, SOL_U2>());
        case SOL_A2: return f(Engine<2, SOL_A2>());
        default: return f(Engine<3, SOL_U3>());
    }
}

struct Events {
    cudaEvent_t e[8];
    Events() { for (auto &x : e) cudaEventCreate(&x); }
    ~Events() { for (auto &x : e) cudaEventDestroy(x); }
    void rec(int i, cudaStream_t s) { cudaEventRecord(e[i], s); }
    float ms(int a, int b)
    {
        float t = 0;
        cudaEventElapsedTime(&t, e[a], e[b]);
        return t;
    }
};

int check_ws(const Layout &L, void *ws, size_t bytes)
{
    if (!ws) return fail(EIK_EINVAL, "null workspace");
    if (bytes < L.total) return fail(EIK_EINVAL, "workspace too small: %zu < %zu", bytes, L.total);
    if ((uintptr_t)ws & 255) return fail(EIK_EINVAL, "workspace must be 256-byte aligned");
    return EIK_OK;
}

int run_update(const eik_geom *g, const Layout &L, real_t *phi, const real_t *speed, uint8_t *state,
               const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol, void *ws,
               cudaStream_t st, int64_t &launches)
{
    char *b = (char *)ws;
    Ctl *ctl = (Ctl *)(b + L.off_ctl_u);
    CK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
    if (nseeds > 0) {
        k_seed<<<(int)std::min<int64_t>((nseeds + 255) / 256, 1024), 256, 0, st>>>(phi, state, seed_idx, seed_val,
                                                                                   nseeds);
        CK(cudaGetLastError());
        ++launches;
    }
    KP p = make_kp(g, L, ws, phi, speed, state, tol, ctl, L.cap_upd);
    return dispatch(g, [&](auto E) {
        int rc = E.prep(p, true, true, st);
        if (rc) return rc;
        rc = E.init_active(p, seed_idx, nseeds, st);
        if (rc) return rc;
        rc = E.update(p, st);
        launches += 3;
        return rc;
    });
}

int check_hang(const Ctl &c, const char *what)
{
    if (c.err == EIK_EHANG)
        return fail(EIK_ECUDA, "%s: device watchdog fired at iteration %llu (grid barrier timeout)", what,
                    (unsigned long long)c.iters);
    return EIK_OK;
}

void fill_update_stats(const Ctl &c, eik_stats *o)
{
    o->upd_iterations = (int64_t)c.iters;
    o->upd_calls = (int64_t)c.sum;
    o->peak_active = (int64_t)c.peak;
    o->converged = (int64_t)c.conv;
    o->history_len = (int64_t)c.iters;
}

int expose_latest(const Layout &L, const Ctl &c, real_t *phi, const real_t *phi2, cudaStream_t st)
{
    if (c.iters & 1) {  // the newest values sit in the workspace buffer
        CK(cudaMemcpyAsync(phi, phi2, (size_t)L.N * sizeof(real_t), cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    return EIK_OK;
}

}  // namespace

// ===========================================================================
// C ABI
// ===========================================================================

extern "C" {

const char *EIK_FN(eik_last_error)(void) { return g_err.c_str(); }
int EIK_FN(eik_last_remedy_engine)(void) { return g_remedy_engine; }

const char *EIK_FN(eik_version)(void)
{
#if EIK_SINGLE
    return "eik_ifim 0.4 (sm_100a, float32 perf mode; persistent cell-worklist update + member-list remedy)";
#else
    return "eik_ifim 0.4 (sm_100a, float64 bit-exact; persistent cell-worklist update + member-list remedy)";
#endif
}

int EIK_FN(eik_workspace_size)(const eik_geom *g, size_t *bytes)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if (!bytes) return fail(EIK_EINVAL, "null output");
    *bytes = L.total;
    return EIK_OK;
}

int EIK_FN(eik_ifim_update_step)(const eik_geom *g, real_t *phi, const real_t *speed, uint8_t *state,
                         const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                         void *workspace, size_t workspace_bytes, int64_t *history, int64_t history_cap,
                         eik_stats *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    if (nseeds < 1 || !seed_idx || !seed_val) return fail(EIK_EINVAL, "boundary condition has no seeds");
    cudaStream_t st = (cudaStream_t)stream;
    Nvtx nvtx_range("eik update step (E/ifim.py:75-134)");
    memset(out, 0, sizeof(*out));
    Events ev;
    ev.rec(0, st);
    int64_t launches = 0;
    rc = run_update(g, L, phi, speed, state, seed_idx, seed_val, nseeds, tol, workspace, st, launches);
    if (rc) return rc;
    ev.rec(1, st);
    Ctl c;
    char *b = (char *)workspace;
    CK(cudaMemcpyAsync(&c, b + L.off_ctl_u, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c, "update step"))) return rc;
    fill_update_stats(c, out);
    out->iterations = out->upd_iterations;
    out->solver_calls = out->upd_calls;
    out->phi_writes = (int64_t)c.writes;
    out->gpu_launches = launches;
    out->upd_ms = out->total_ms = ev.ms(0, 1);
    if (history && history_cap > 0 && c.iters > 0) {
        const int64_t n = std::min<int64_t>((int64_t)c.iters, history_cap);
        CK(cudaMemcpy(history, b + L.off_hist, (size_t)n * 8, cudaMemcpyDeviceToHost));
    }
    if (c.err == EIK_ECAP) {
        if ((rc = expose_latest(L, c, phi, (const real_t *)(b + L.off_phi2), st))) return rc;
        return fail(EIK_ECAP, "active list did not drain within %lld iterations", (long long)L.cap_upd);
    }
    return EIK_OK;
}

int EIK_FN(eik_build_remedy)(const eik_geom *g, const real_t *phi, const real_t *speed, const uint8_t *state, double tol,
                     void *workspace, size_t workspace_bytes, eik_stats *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    cudaStream_t st = (cudaStream_t)stream;
    Nvtx nvtx_range("eik build pass (E/ifim.py:137-161)");
    memset(out, 0, sizeof(*out));
    char *b = (char *)workspace;
    Ctl *ctl = (Ctl *)(b + L.off_ctl_r);
    Events ev;
    ev.rec(0, st);
    KP p = make_kp(g, L, workspace, const_cast<real_t *>(phi), speed, state, tol, ctl, L.cap_rem);
    rc = dispatch(g, [&](auto E) {
        int r = E.prep(p, false, false, st);
        if (r) return r;
        return E.build(p, phi, nullptr, st);
    });
    if (rc) return rc;
    ev.rec(1, st);
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    out->build_calls = out->solver_calls = (int64_t)c.free_cells;
    out->remedy_size = (int64_t)c.flagged;
    out->gpu_launches = 2;
    out->build_ms = out->total_ms = ev.ms(0, 1);
    return EIK_OK;
}

int EIK_FN(eik_remedy_load_set)(const eik_geom *g, const uint8_t *cells, const uint8_t *member, const uint8_t *state,
                                void *workspace, size_t workspace_bytes, int64_t *count, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!cells) return fail(EIK_EINVAL, "null work-list mask");
    cudaStream_t st = (cudaStream_t)stream;
    char *b = (char *)workspace;
    Ctl *ctl = (Ctl *)(b + L.off_ctl_r);
    KP p = make_kp(g, L, workspace, nullptr, nullptr, state, 1e-12, ctl, L.cap_rem);
    rc = dispatch(g, [&](auto E) { return E.load(p, cells, member, st); });
    if (rc) return rc;
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (count) *count = (int64_t)c.flagged;
    return EIK_OK;
}

int EIK_FN(eik_remedy_load)(const eik_geom *g, const uint8_t *member, const uint8_t *state, void *workspace,
                    size_t workspace_bytes, int64_t *count, void *stream)
{
    if (!member) return fail(EIK_EINVAL, "null member mask");
    return EIK_FN(eik_remedy_load_set)(g, member, nullptr, state, workspace, workspace_bytes, count, stream);
}

int EIK_FN(eik_remedy_export)(const eik_geom *g, void *workspace, size_t workspace_bytes, uint8_t *member, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!member) return fail(EIK_EINVAL, "null member mask");
    cudaStream_t st = (cudaStream_t)stream;
    char *b = (char *)workspace;
    Ctl c;
    CK(cudaMemcpyAsync(&c, b + L.off_ctl_r, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemsetAsync(member, 0, (size_t)L.N, st));
    KP p = make_kp(g, L, workspace, nullptr, nullptr, nullptr, 1e-12, nullptr, 0);
    rc = dispatch(g, [&](auto E) { return E.do_export(p, member, st); });
    if (rc) return rc;
    CK(cudaStreamSynchronize(st));
    return EIK_OK;
}

int EIK_FN(eik_remedy_step)(const eik_geom *g, real_t *phi, const real_t *speed, const uint8_t *state, double tol,
                    void *workspace, size_t workspace_bytes, eik_stats *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    cudaStream_t st = (cudaStream_t)stream;
    Nvtx nvtx_range("eik remedy step (E/ifim.py:164-218)");
    memset(out, 0, sizeof(*out));
    char *b = (char *)workspace;
    Ctl *ctl = (Ctl *)(b + L.off_ctl_r);
    Events ev;
    ev.rec(0, st);
    KP p = make_kp(g, L, workspace, phi, speed, state, tol, ctl, L.cap_rem);
    unsigned stale = 0;  // a hand-built set with members outside its work list (eik_remedy_load_set)
    CK(cudaMemcpyAsync(&stale, &ctl->stale, sizeof(stale), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    // staged call: the caller may have edited phi since the last call
    rc = dispatch(g, [&](auto E) {
        int r = E.prep(p, true, false, st);
        if (r) return r;
        return E.remedy_single(p, nullptr, st, stale != 0);
    });
    if (rc) return rc;
    ev.rec(1, st);
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c, "remedy step"))) return rc;
    if (g_remedy_engine == 4) g_remedy_engine = c.engine ? (int)c.engine : 1;
    out->rem_iterations = out->iterations = (int64_t)c.iters;
    out->rem_calls = out->solver_calls = (int64_t)c.sum;
    out->peak_remedy = (int64_t)c.peak;
    out->phi_writes = (int64_t)c.writes;
    out->gpu_launches = 2;
    out->rem_ms = out->total_ms = ev.ms(0, 1);
    if (c.err == EIK_ECAP) {
        if ((rc = expose_latest(L, c, phi, p.P1, st))) return rc;
        return fail(EIK_ECAP, "remedy set did not drain within %lld rounds", (long long)L.cap_rem);
    }
    return EIK_OK;
}

int EIK_FN(eik_ifim_solve)(const eik_geom *g, real_t *phi, const real_t *speed, uint8_t *state, const int64_t *seed_idx,
                   const double *seed_val, int64_t nseeds, double tol, void *workspace, size_t workspace_bytes,
                   int64_t *history, int64_t history_cap, eik_stats *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    if (nseeds < 1 || !seed_idx || !seed_val) return fail(EIK_EINVAL, "boundary condition has no seeds");
    cudaStream_t st = (cudaStream_t)stream;
    memset(out, 0, sizeof(*out));
    char *b = (char *)workspace;
    Ctl *cu = (Ctl *)(b + L.off_ctl_u);
    Ctl *cr = (Ctl *)(b + L.off_ctl_r);
    Events ev;
    int64_t launches = 0;
    Nvtx range_solve("eik_ifim_solve");
    ev.rec(0, st);
    {
        Nvtx r("eik update step (E/ifim.py:75-134)");
        rc = run_update(g, L, phi, speed, state, seed_idx, seed_val, nseeds, tol, workspace, st, launches);
    }
    if (rc) return rc;
    ev.rec(1, st);
    KP p = make_kp(g, L, workspace, phi, speed, state, tol, cr, L.cap_rem);
    // After a drained update step both phi buffers are identical (every cell
    // changed in the last-but-one iteration rewrote itself in the last one),
    // so the build reads the caller's buffer and the remedy starts at parity 0.
    const unsigned *skip = &cu->err;
    {
        Nvtx r("eik build pass (E/ifim.py:137-161)");
        rc = dispatch(g, [&](auto E) { return E.build(p, phi, skip, st); });
    }
    if (rc) return rc;
    ev.rec(2, st);
    {
        Nvtx r("eik remedy step (E/ifim.py:164-218)");
        rc = dispatch(g, [&](auto E) { return E.remedy_single(p, skip, st); });
    }
    if (rc) return rc;
    ev.rec(3, st);
    launches += 2;
    Ctl c[2];
    CK(cudaMemcpyAsync(&c[0], cu, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&c[1], cr, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c[0], "update step")) || (rc = check_hang(c[1], "remedy step"))) return rc;
    if (g_remedy_engine == 4) g_remedy_engine = c[1].engine ? (int)c[1].engine : 1;
    if (c[0].err == EIK_ECAP) {
        if ((rc = expose_latest(L, c[0], phi, p.P1, st))) return rc;
        return fail(EIK_ECAP, "active list did not drain within %lld iterations", (long long)L.cap_upd);
    }
    if (c[1].err == EIK_ECAP) {
        if ((rc = expose_latest(L, c[1], phi, p.P1, st))) return rc;
        return fail(EIK_ECAP, "remedy set did not drain within %lld rounds", (long long)L.cap_rem);
    }
    fill_update_stats(c[0], out);
    out->build_calls = (int64_t)c[1].free_cells;
    out->remedy_size = (int64_t)c[1].flagged;
    out->rem_iterations = (int64_t)c[1].iters;
    out->rem_calls = (int64_t)c[1].sum;
    out->peak_remedy = (int64_t)c[1].peak;
    out->iterations = out->upd_iterations + out->rem_iterations;  // E/ifim.py:227-233
    out->solver_calls = out->upd_calls + out->build_calls + out->rem_calls;
    out->phi_writes = (int64_t)(c[0].writes + c[1].writes);
    out->gpu_launches = launches;
    out->upd_ms = ev.ms(0, 1);
    out->build_ms = ev.ms(1, 2);
    out->rem_ms = ev.ms(2, 3);
    out->total_ms = ev.ms(0, 3);
#ifdef EIK_DIAG
    if (getenv("EIK_DIAG_PRINT")) {
        fprintf(stderr, "[eik diag] remedy member words %llu sectors %llu calls %llu\n",
                (unsigned long long)c[1].nz_words, (unsigned long long)c[1].nz_sectors,
                (unsigned long long)c[1].sum);
        for (int k = 0; k < 25; ++k)
            if (c[0].du[0][k])
                fprintf(stderr, "[eik diag] update |A|~2^%2d iterations %6llu cells %12llu  %9.3f ms  (%.2f us per iteration)\n",
                        k, c[0].du[0][k], c[0].du[2][k], c[0].du[1][k] * 1e-6, c[0].du[1][k] * 1e-3 / c[0].du[0][k]);
        for (int k = 0; k < 25; ++k)
            if (c[0].du[0][k])
                fprintf(stderr, "[eik diag] update |A|~2^%2d per iteration: slowest CTA %.2f us, mean CTA %.2f us\n", k,
                        c[0].du2[0][k] * 1e-3 / c[0].du[0][k], c[0].du2[1][k] * 1e-3 / c[0].du[0][k]);
        for (int k = 0; k < 26; ++k)
            if (c[1].dg[0][k])
                fprintf(stderr, "[eik diag] |R|~2^%2d rounds %6llu members %12llu  B %9.3f ms  A %9.3f ms  (%.2f/%.2f us per round)\n",
                        k, c[1].dg[0][k], c[1].dg[3][k], c[1].dg[1][k] * 1e-6, c[1].dg[2][k] * 1e-6,
                        c[1].dg[1][k] * 1e-3 / c[1].dg[0][k], c[1].dg[2][k] * 1e-3 / c[1].dg[0][k]);
        for (int k = 0; k < 26; ++k)
            if (c[1].dg[0][k])
                fprintf(stderr, "[eik diag] |R|~2^%2d phase B per round: slowest CTA %.2f us, mean CTA %.2f us, start skew %.2f us, last arrival -> lead release %.2f us\n",
                        k, c[1].dg2[0][k] * 1e-3 / c[1].dg[0][k], c[1].dg2[1][k] * 1e-3 / c[1].dg[0][k],
                        c[1].dg2[2][k] * 1e-3 / c[1].dg[0][k], c[1].dg2[3][k] * 1e-3 / c[1].dg[0][k]);
        for (int k = 0; k < 26; ++k)
            if (c[1].dg[0][k])
                fprintf(stderr, "[eik diag] |R|~2^%2d slowest CTA: %.0f members (mean %.0f per CTA), CTA 0 in %llu of %llu rounds, mean id %.1f\n",
                        k, (double)c[1].dg2[4][k] / c[1].dg[0][k], (double)c[1].dg[3][k] / c[1].dg[0][k] / 296.0,
                        c[1].dg2[5][k], c[1].dg[0][k], (double)c[1].dg2[6][k] / c[1].dg[0][k]);
    }
#endif
    if (history && history_cap > 0 && c[0].iters > 0) {
        const int64_t n = std::min<int64_t>((int64_t)c[0].iters, history_cap);
        CK(cudaMemcpy(history, b + L.off_hist, (size_t)n * 8, cudaMemcpyDeviceToHost));
    }
    return EIK_OK;
}

int EIK_FN(eik_solve_fixpoint)(const eik_geom *g, real_t *phi, const real_t *speed, uint8_t *state,
                       const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                       int64_t max_passes, void *workspace, size_t workspace_bytes, eik_stats *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    if (nseeds < 1 || !seed_idx || !seed_val) return fail(EIK_EINVAL, "boundary condition has no seeds");
    cudaStream_t st = (cudaStream_t)stream;
    Nvtx nvtx_range("eik fixpoint (E/oracle.py:22-70)");
    memset(out, 0, sizeof(*out));
    char *b = (char *)workspace;
    Ctl *ctl = (Ctl *)(b + L.off_ctl_r);
    const int64_t s3 = g->nx + g->ny + (g->ndim == 3 ? g->nz : 0);
    const int64_t cap = max_passes > 0 ? max_passes : 10 * s3;  // E/oracle.py:40
    Events ev;
    ev.rec(0, st);
    CK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
    k_seed<<<(int)std::min<int64_t>((nseeds + 255) / 256, 1024), 256, 0, st>>>(phi, state, seed_idx, seed_val, nseeds);
    CK(cudaGetLastError());
    KP p = make_kp(g, L, workspace, phi, speed, state, tol, ctl, cap);
    rc = dispatch(g, [&](auto E) {
        int r = E.prep(p, true, false, st);
        if (r) return r;
        return E.fixpoint(p, st);
    });
    if (rc) return rc;
    ev.rec(1, st);
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c, "fixpoint"))) return rc;
    if (c.iters & 1) {  // the last pass wrote the workspace buffer
        CK(cudaMemcpyAsync(phi, p.P1, (size_t)L.N * sizeof(real_t), cudaMemcpyDeviceToDevice, st));
        CK(cudaStreamSynchronize(st));
    }
    int64_t nfree = 0;
    {
        // free cells = N - #(blocked | source): count from the fixed bitmap
        std::vector<uint32_t> fb(L.nwords);
        CK(cudaMemcpy(fb.data(), p.Fb, (size_t)L.nwords * 4, cudaMemcpyDeviceToHost));
        int64_t fixed_in_row = 0;
        for (uint32_t w = 0; w < L.nwords; ++w) fixed_in_row += __builtin_popcount(fb[w]);
        nfree = (int64_t)L.nwords * 32 - fixed_in_row;  // lanes outside rows are marked fixed
    }
    out->iterations = (int64_t)c.iters;
    out->solver_calls = (int64_t)c.iters * nfree;  // E/oracle.py:52
    out->total_ms = ev.ms(0, 1);
    out->gpu_launches = 3;
    if (c.err == EIK_ECAP) return fail(EIK_ECAP, "fixpoint iteration did not converge within %lld passes", (long long)cap);
    return EIK_OK;
}

int EIK_FN(eik_solve_fim)(const eik_geom *g, real_t *phi, const real_t *speed, uint8_t *state,
                          const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                          void *workspace, size_t workspace_bytes, eik_stats *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);  // E/fim.py:64-65
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    if (nseeds < 1 || !seed_idx || !seed_val) return fail(EIK_EINVAL, "boundary condition has no seeds");
    cudaStream_t st = (cudaStream_t)stream;
    Nvtx nvtx_range("eik FIM (E/fim.py:62-144)");
    memset(out, 0, sizeof(*out));
    char *b = (char *)workspace;
    Ctl *ctl = (Ctl *)(b + L.off_ctl_u);
    Events ev;
    ev.rec(0, st);
    CK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
    k_seed<<<(int)std::min<int64_t>((nseeds + 255) / 256, 1024), 256, 0, st>>>(phi, state, seed_idx, seed_val, nseeds);
    CK(cudaGetLastError());
    KP p = make_kp(g, L, workspace, phi, speed, state, tol, ctl, L.cap_upd);
    rc = dispatch(g, [&](auto E) {
        int r = E.prep(p, false, true, st);
        if (r) return r;
        CK(cudaMemsetAsync(p.lab, 0, (size_t)L.N, st));           // labels: FAR
        CK(cudaMemsetAsync(p.R0b, 0, (size_t)L.nwords * 4, st));  // claims
        r = E.init_active(p, seed_idx, nseeds, st);
        if (r) return r;
        return E.fim(p, st);
    });
    if (rc) return rc;
    ev.rec(1, st);
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c, "fim"))) return rc;
    out->iterations = (int64_t)c.iters;
    out->upd_iterations = (int64_t)c.iters;
    out->solver_calls = out->upd_calls = (int64_t)c.sum;
    out->peak_active = (int64_t)c.peak;
    out->phi_writes = (int64_t)c.writes;
    out->total_ms = out->upd_ms = ev.ms(0, 1);
    out->gpu_launches = 5;
    if (c.err == EIK_ECAP)
        return fail(EIK_ECAP, "active list did not drain within %lld iterations", (long long)L.cap_upd);
    return EIK_OK;
}

int EIK_FN(eik_max_residual)(const eik_geom *g, const real_t *phi, const real_t *speed, const uint8_t *state,
                     void *workspace, size_t workspace_bytes, double *out, void *stream)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if ((rc = check_ws(L, workspace, workspace_bytes))) return rc;
    if (!phi || !speed || !state || !out) return fail(EIK_EINVAL, "null array");
    cudaStream_t st = (cudaStream_t)stream;
    Ctl *ctl = (Ctl *)((char *)workspace + L.off_ctl_r);
    CK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
    KP p = make_kp(g, L, workspace, const_cast<real_t *>(phi), speed, state, 1e-12, ctl, 0);
    rc = dispatch(g, [&](auto E) {
        int r = E.prep(p, false, false, st);
        if (r) return r;
        return E.residual(p, st);
    });
    if (rc) return rc;
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    unsigned long long bits = c.peak;
#if EIK_SINGLE
    const unsigned b32 = (unsigned)bits;
    float r;
    memcpy(&r, &b32, 4);
#else
    double r;
    memcpy(&r, &bits, 8);
#endif
    *out = (double)r;  // 0.0 when no free finite cell (E/harness.py:158-159)
    return EIK_OK;
}

#if !EIK_SINGLE  // multi-GPU slabs: float64 engine only
// ---- multi-rank (peer slabs) -----------------------------------------------

static Peer make_peer(const eik_geom *g, const eik_rank &rk, int use_remedy)
{
    Peer pr;
    memset(&pr, 0, sizeof(pr));
    eik_geom gl = *g;
    gl.nz = rk.nz;
    gl.flags = 0;
    Layout L;
    if (make_layout(&gl, L)) return pr;
    char *b = (char *)rk.workspace;
    pr.P0 = rk.phi0;
    pr.P1 = (real_t *)(b + L.off_phi2);
    pr.Bt = (uint32_t *)(b + L.off_bt);
    pr.L0 = (uint32_t *)(b + L.off_l0);
    pr.L1 = (uint32_t *)(b + L.off_l1);
    pr.D0b = (uint32_t *)(b + L.off_d0);
    pr.D1b = (uint32_t *)(b + L.off_d1);
    pr.ctl = (Ctl *)(b + (use_remedy ? L.off_ctl_r : L.off_ctl_u));
    pr.nz = (uint32_t)rk.nz;
    pr.valid = 1;
    return pr;
}

struct MrCtx {
    eik_geom gl;
    Layout L;
    KP kp;
};

static int mr_setup(const eik_geom *g, int32_t R, const eik_rank *ranks, int32_t q, const real_t *speed,
                    uint8_t *state, double tol, int use_remedy, MrCtx &m)
{
    if (!g || g->ndim != 3 || g->flags) return fail(EIK_EINVAL, "multi-rank solves take the global 3D geometry");
    if (R < 1 || R > EIK_MAX_RANKS) return fail(EIK_EINVAL, "1 <= ranks <= %d", EIK_MAX_RANKS);
    int64_t nzsum = 0;
    for (int r = 0; r < R; ++r) {
        if (ranks[r].nz < 1 || !ranks[r].workspace || !ranks[r].phi0) return fail(EIK_EINVAL, "bad rank %d", r);
        nzsum += ranks[r].nz;
    }
    if (nzsum != g->nz) return fail(EIK_EINVAL, "rank slabs cover %lld planes, grid has %lld", (long long)nzsum,
                                    (long long)g->nz);
    int64_t zg0 = 0;
    for (int r = 0; r < q; ++r) zg0 += ranks[r].nz;
    m.gl = *g;
    m.gl.nz = ranks[q].nz;
    int rc = make_layout(&m.gl, m.L);
    if (rc) return rc;
    char *b = (char *)ranks[q].workspace;
    const int64_t s3 = g->nx + g->ny + g->nz;  // caps of the GLOBAL grid
    m.kp = make_kp(&m.gl, m.L, ranks[q].workspace, ranks[q].phi0, speed, state, tol,
                   (Ctl *)(b + (use_remedy ? m.L.off_ctl_r : m.L.off_ctl_u)), use_remedy ? 20 * s3 : 40 * s3);
    m.kp.mr = 1;
    m.kp.q = q;
    m.kp.R = R;
    if (q > 0) m.kp.lo = make_peer(g, ranks[q - 1], use_remedy);
    if (q + 1 < R) m.kp.hi = make_peer(g, ranks[q + 1], use_remedy);
    for (int r = 0; r < R; ++r) m.kp.rank_ctl[r] = make_peer(g, ranks[r], use_remedy).ctl;
    (void)zg0;
    return EIK_OK;
}

int eik_peer_enable(int32_t device, int32_t peer)
{
    if (device == peer) return EIK_OK;
    int can = 0;
    CK(cudaDeviceCanAccessPeer(&can, device, peer));
    if (!can) return fail(EIK_EINVAL, "device %d cannot map device %d's memory (no NVLink/P2P path)", device, peer);
    int cur = 0;
    CK(cudaGetDevice(&cur));
    CK(cudaSetDevice(device));
    cudaError_t e = cudaDeviceEnablePeerAccess(peer, 0);
    if (e == cudaErrorPeerAccessAlreadyEnabled) {
        (void)cudaGetLastError();
        e = cudaSuccess;
    }
    cudaSetDevice(cur);
    if (e != cudaSuccess) return fail(EIK_ECUDA, "enable peer access %d -> %d: %s", device, peer, cudaGetErrorString(e));
    return EIK_OK;
}

int eik_mr_prepare(const eik_geom *g, int32_t R, const eik_rank *ranks, int32_t r_begin, int32_t r_end,
                   const real_t *const *speed, uint8_t *const *state, const int64_t *seeds, const double *seed_val,
                   int64_t nseeds, double tol, void *stream)
{
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (r_begin < 0 || r_end > R || r_begin >= r_end) return fail(EIK_EINVAL, "bad local rank range");
    if (nseeds < 1 || !seeds || !seed_val) return fail(EIK_EINVAL, "boundary condition has no seeds");
    cudaStream_t st = (cudaStream_t)stream;
    for (int q = r_begin; q < r_end; ++q) {
        MrCtx m;
        int rc = mr_setup(g, R, ranks, q, speed[q - r_begin], state[q - r_begin], tol, 0, m);
        if (rc) return rc;
        char *b = (char *)ranks[q].workspace;
        CK(cudaMemsetAsync(b + m.L.off_ctl_u, 0, sizeof(Ctl), st));
        CK(cudaMemsetAsync(b + m.L.off_ctl_r, 0, sizeof(Ctl), st));
        int64_t zg0 = 0;
        for (int r = 0; r < q; ++r) zg0 += ranks[r].nz;
        k_seed_mr<<<(int)std::min<int64_t>((nseeds + 255) / 256, 1024), 256, 0, st>>>(
            ranks[q].phi0, state[q - r_begin], seeds, seed_val, nseeds, zg0, ranks[q].nz, g->nx * g->ny);
        CK(cudaGetLastError());
        KP p = m.kp;
        rc = dispatch(&m.gl, [&](auto E) { return E.prep(p, true, true, st); });
        if (rc) return rc;
        k_init_active_mr<<<(int)std::min<int64_t>((nseeds + 255) / 256, 1024), 256, 0, st>>>(p, seeds, nseeds, zg0,
                                                                                            g->nz);
        CK(cudaGetLastError());
    }
    CK(cudaStreamSynchronize(st));
    return EIK_OK;
}

int eik_mr_run(const eik_geom *g, int32_t R, const eik_rank *ranks, int32_t r_begin, int32_t r_end,
               const real_t *const *speed, uint8_t *const *state, double tol, int64_t *history, int64_t history_cap,
               eik_stats *out, void *stream)
{
    if (r_begin < 0 || r_end > R || r_begin >= r_end) return fail(EIK_EINVAL, "bad local rank range");
    if (!out) return fail(EIK_EINVAL, "null stats");
    cudaStream_t st = (cudaStream_t)stream;
    Nvtx nvtx_range("eik multi-rank solve");
    memset(out, 0, sizeof(*out));
    const int nl = r_end - r_begin;
    Events ev;
    ev.rec(0, st);
    // update step: one cooperative launch over the local ranks
    std::vector<MrCtx> mu(nl), mrm(nl);
    for (int i = 0; i < nl; ++i) {
        int rc = mr_setup(g, R, ranks, r_begin + i, speed[i], state[i], tol, 0, mu[i]);
        if (rc) return rc;
        rc = mr_setup(g, R, ranks, r_begin + i, speed[i], state[i], tol, 1, mrm[i]);
        if (rc) return rc;
        mu[i].kp.gb0 = mrm[i].kp.gb0 = 0;  // set after the group size is known
    }
    char *b0 = (char *)ranks[r_begin].workspace;
    KP *kps_dev = (KP *)(b0 + mu[0].L.off_kps);
    int per_sm = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_update_mr<3, SOL_U3>, BLOCK, 0));
    uint32_t pg = (uint32_t)(per_sm * num_sms() / nl);
    std::vector<KP> host(nl);
    for (int i = 0; i < nl; ++i) {
        host[i] = mu[i].kp;
        host[i].gb0 = pg * i;
        host[i].gnb = pg;
    }
    CK(cudaMemcpyAsync(kps_dev, host.data(), sizeof(KP) * nl, cudaMemcpyHostToDevice, st));
    int pgo = 0;
    int rc;
    if (nl == 1) {  // one rank on this device: parameters by value
        host[0].gb0 = 0;
        host[0].gnb = 0;
        rc = coop_launch(k_update_mr1<3, SOL_U3>, host[0], nullptr, false, st, "EIK_UPD_BLOCKS_PER_SM", 0);
    } else {
        rc = Engine<3, SOL_U3>::update_mr(kps_dev, nl, st, pgo);
        if (!rc && (uint32_t)pgo != pg) return fail(EIK_ECUDA, "group size mismatch");
    }
    if (rc) return rc;
    ev.rec(1, st);
    // build: per local rank (reads the neighbours' final phi; the update's last world barrier ordered it)
    for (int i = 0; i < nl; ++i) {
        KP p = mrm[i].kp;
        rc = Engine<3, SOL_U3>::build(p, p.P0, nullptr, st);
        if (rc) return rc;
    }
    ev.rec(2, st);
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_remedy_mr<3, SOL_U3>, BLOCK, 0));
    pg = (uint32_t)(per_sm * num_sms() / nl);
    for (int i = 0; i < nl; ++i) {
        host[i] = mrm[i].kp;
        host[i].gb0 = pg * i;
        host[i].gnb = pg;
    }
    KP *kps_dev_r = kps_dev + EIK_MAX_RANKS;
    CK(cudaMemcpyAsync(kps_dev_r, host.data(), sizeof(KP) * nl, cudaMemcpyHostToDevice, st));
    if (nl == 1) {
        host[0].gb0 = 0;
        host[0].gnb = 0;
        rc = coop_launch(k_remedy_mr1<3, SOL_U3>, host[0], nullptr, false, st, "EIK_REM_BLOCKS_PER_SM", 0);
    } else {
        rc = Engine<3, SOL_U3>::remedy_mr(kps_dev_r, nl, st, pgo);
    }
    if (rc) return rc;
    ev.rec(3, st);
    // global stats live in rank 0's control blocks; errors in any local rank's
    Ctl cu0, cr0;
    CK(cudaMemcpyAsync(&cu0, mu[0].kp.rank_ctl[0], sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&cr0, mrm[0].kp.rank_ctl[0], sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    unsigned long long writes = 0, conv = 0, freec = 0, flagged = 0, rwrites = 0;
    for (int r = 0; r < R; ++r) {
        Ctl cu, cr;
        CK(cudaMemcpyAsync(&cu, mu[0].kp.rank_ctl[r], sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(&cr, mrm[0].kp.rank_ctl[r], sizeof(Ctl), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if ((rc = check_hang(cu, "multi-rank update step")) || (rc = check_hang(cr, "multi-rank remedy step")))
            return rc;
        if (cu.err == EIK_ECAP) return fail(EIK_ECAP, "active list did not drain");
        if (cr.err == EIK_ECAP) return fail(EIK_ECAP, "remedy set did not drain");
        writes += cu.writes;
        rwrites += cr.writes;
        conv += cu.conv;
        freec += cr.free_cells;
        flagged += cr.flagged;
    }
    fill_update_stats(cu0, out);
    out->converged = (int64_t)conv;
    out->build_calls = (int64_t)freec;
    out->remedy_size = (int64_t)flagged;
    out->rem_iterations = (int64_t)cr0.iters;
    out->rem_calls = (int64_t)cr0.sum;
    out->peak_remedy = (int64_t)cr0.peak;
    out->iterations = out->upd_iterations + out->rem_iterations;
    out->solver_calls = out->upd_calls + out->build_calls + out->rem_calls;
    out->phi_writes = (int64_t)(writes + rwrites);
    out->upd_ms = ev.ms(0, 1);
    out->build_ms = ev.ms(1, 2);
    out->rem_ms = ev.ms(2, 3);
    out->total_ms = ev.ms(0, 3);
    out->gpu_launches = 2 + nl;
    if (history && history_cap > 0 && cu0.iters > 0) {
        eik_geom g0 = *g;
        g0.nz = ranks[0].nz;
        Layout L0;
        if ((rc = make_layout(&g0, L0))) return rc;
        const int64_t n = std::min<int64_t>((int64_t)cu0.iters, history_cap);
        CK(cudaMemcpy(history, (char *)ranks[0].workspace + L0.off_hist, (size_t)n * 8, cudaMemcpyDeviceToHost));
    }
    return EIK_OK;
}

int eik_workspace_offsets(const eik_geom *g, int64_t *off)
{
    Layout L;
    int rc = make_layout(g, L);
    if (rc) return rc;
    if (!off) return fail(EIK_EINVAL, "null output");
    off[0] = (int64_t)L.off_phi2;
    off[1] = (int64_t)L.off_bt;
    off[2] = (int64_t)L.off_d0;
    off[3] = (int64_t)L.off_d1;
    return EIK_OK;
}

static int slab_check(const eik_geom *g, Layout &L, void *ws, size_t wsb)
{
    int rc = make_layout(g, L);
    if (rc) return rc;
    if (!(g->flags & EIK_GEOM_SLAB)) return fail(EIK_EINVAL, "geometry is not a slab (flags)");
    return check_ws(L, ws, wsb);
}

int eik_slab_update_init(const eik_geom *g, real_t *phi, const real_t *speed, uint8_t *state, const int64_t *seed_idx,
                         const double *seed_val, int64_t nseeds, double tol, void *workspace, size_t workspace_bytes,
                         int64_t *n_active, void *stream)
{
    Layout L;
    int rc = slab_check(g, L, workspace, workspace_bytes);
    if (rc) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    if (!phi || !speed || !state) return fail(EIK_EINVAL, "null array");
    cudaStream_t st = (cudaStream_t)stream;
    rc = [&]() {
        char *b = (char *)workspace;
        Ctl *ctl = (Ctl *)(b + L.off_ctl_u);
        CK(cudaMemsetAsync(ctl, 0, sizeof(Ctl), st));
        if (nseeds > 0) {
            k_seed<<<(int)std::min<int64_t>((nseeds + 255) / 256, 1024), 256, 0, st>>>(phi, state, seed_idx, seed_val,
                                                                                       nseeds);
            CK(cudaGetLastError());
        }
        KP p = make_kp(g, L, workspace, phi, speed, state, tol, ctl, L.cap_upd);
        return dispatch(g, [&](auto E) {
            int r2 = E.prep(p, true, true, st);
            if (r2 || nseeds == 0) return r2;
            return E.init_active(p, seed_idx, nseeds, st);
        });
    }();
    if (rc) return rc;
    Ctl c;
    CK(cudaMemcpyAsync(&c, (char *)workspace + L.off_ctl_u, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (n_active) *n_active = c.len[0];
    return EIK_OK;
}

int eik_slab_update_iter(const eik_geom *g, real_t *phi, const real_t *speed, uint8_t *state, double tol, int64_t it,
                         void *workspace, size_t workspace_bytes, void *stream)
{
    Layout L;
    int rc = slab_check(g, L, workspace, workspace_bytes);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Ctl *ctl = (Ctl *)((char *)workspace + L.off_ctl_u);
    KP p = make_kp(g, L, workspace, phi, speed, state, tol, ctl, L.cap_upd);
    p.it0 = it;
    p.max_it = 1;
    return dispatch(g, [&](auto E) { return E.update(p, st); });
}

int eik_slab_apply_requests(const eik_geom *g, const uint32_t *req_lo, const uint32_t *req_hi, int64_t it,
                            void *workspace, size_t workspace_bytes, int64_t *n_active, void *stream)
{
    Layout L;
    int rc = slab_check(g, L, workspace, workspace_bytes);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Ctl *ctl = (Ctl *)((char *)workspace + L.off_ctl_u);
    KP p = make_kp(g, L, workspace, nullptr, nullptr, nullptr, 1e-12, ctl, L.cap_upd);
    const int64_t planeW = (int64_t)L.W * g->ny;
    if (req_lo || req_hi) {
        k_apply_requests<<<(int)std::min<int64_t>((2 * planeW + 255) / 256, 4096), 256, 0, st>>>(p, req_lo, req_hi, it);
        CK(cudaGetLastError());
    }
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c, "slab update step"))) return rc;
    if (n_active) *n_active = c.len[(it + 1) % 3];
    return EIK_OK;
}

int eik_slab_build(const eik_geom *g, const real_t *phi, const real_t *speed, const uint8_t *state, double tol,
                   void *workspace, size_t workspace_bytes, int64_t *free_cells, int64_t *flagged, void *stream)
{
    Layout L;
    int rc = slab_check(g, L, workspace, workspace_bytes);
    if (rc) return rc;
    if (!(tol > 0)) return fail(EIK_EINVAL, "tol must be positive, got %g", tol);
    cudaStream_t st = (cudaStream_t)stream;
    Ctl *ctl = (Ctl *)((char *)workspace + L.off_ctl_r);
    KP p = make_kp(g, L, workspace, const_cast<real_t *>(phi), speed, state, tol, ctl, L.cap_rem);
    rc = dispatch(g, [&](auto E) { return E.build(p, phi, nullptr, st); });
    if (rc) return rc;
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (free_cells) *free_cells = (int64_t)c.free_cells;
    if (flagged) *flagged = (int64_t)c.flagged;
    return EIK_OK;
}

int eik_slab_remedy_round(const eik_geom *g, real_t *phi, const real_t *speed, const uint8_t *state, double tol,
                          int64_t r, void *workspace, size_t workspace_bytes, int64_t *calls, int64_t *decs,
                          void *stream)
{
    Layout L;
    int rc = slab_check(g, L, workspace, workspace_bytes);
    if (rc) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    Ctl *ctl = (Ctl *)((char *)workspace + L.off_ctl_r);
    KP p = make_kp(g, L, workspace, phi, speed, state, tol, ctl, L.cap_rem);
    p.it0 = r;
    p.max_it = 1;
    if (r == 0) {  // round slots start clean (the build left R0 and its counters)
        CK(cudaMemsetAsync(&ctl->len[0], 0, sizeof(ctl->len), st));
        CK(cudaMemsetAsync(&ctl->cnt[0], 0, sizeof(ctl->cnt), st));
        CK(cudaMemsetAsync(&ctl->dsum[0], 0, sizeof(ctl->dsum), st));
    }
    rc = dispatch(g, [&](auto E) { return E.remedy(p, nullptr, st); });
    if (rc) return rc;
    Ctl c;
    CK(cudaMemcpyAsync(&c, ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if ((rc = check_hang(c, "slab remedy step"))) return rc;
    if (calls) *calls = c.len[r % 3];
    if (decs) *decs = (int64_t)c.dsum[r % 3];
    return EIK_OK;
}

#endif  // !EIK_SINGLE

int EIK_FN(eik_field_max_diff)(const real_t *a, const real_t *b, int64_t n, void *scratch, double *out, void *stream)
{
    if (!out) return fail(EIK_EINVAL, "null output");
    if (n < 0 || (n > 0 && (!a || !b || !scratch))) return fail(EIK_EINVAL, "null array");
    if (n == 0) {  // E/harness.py:170-171
        *out = 0.0;
        return EIK_OK;
    }
    cudaStream_t st = (cudaStream_t)stream;
    unsigned long long *acc = (unsigned long long *)scratch;
    CK(cudaMemsetAsync(acc, 0, 16, st));
    k_max_diff<<<stream_grid((n + 31) / 32), BLOCK, 0, st>>>(a, b, n, acc);
    CK(cudaGetLastError());
    unsigned long long h[2];
    CK(cudaMemcpyAsync(h, acc, 16, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (h[1]) {
        *out = NAN;
    } else {
#if EIK_SINGLE
        const unsigned b32 = (unsigned)h[0];
        float f;
        memcpy(&f, &b32, 4);
        *out = (double)f;
#else
        double d;
        memcpy(&d, &h[0], 8);
        *out = d;
#endif
    }
    return EIK_OK;
}

int EIK_FN(eik_chunk_sha256)(const void *data, int64_t nbytes, int64_t chunk, uint8_t *digests, void *stream)
{
    if (nbytes < 0 || chunk < 64 || (chunk & 63)) return fail(EIK_EINVAL, "chunk must be a positive multiple of 64 bytes");
    if (nbytes > 0 && (!data || !digests)) return fail(EIK_EINVAL, "null array");
    if ((uintptr_t)data & 15) return fail(EIK_EINVAL, "data must be 16-byte aligned");
    const uint64_t nch = nbytes ? ((uint64_t)nbytes + chunk - 1) / chunk : 0;
    if (!nch) return EIK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_sha256_chunks<<<(unsigned)((nch + 127) / 128), 128, 0, st>>>((const uint8_t *)data, (uint64_t)nbytes,
                                                                   (uint64_t)chunk, nch, digests);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return EIK_OK;
}

int EIK_FN(eik_local_solve)(int kind, const real_t *a, const real_t *b, const real_t *c, const real_t *f, double dx,
                    double dy, real_t *out, int64_t n, void *stream)
{
    if (kind < 0 || kind > 2) return fail(EIK_EINVAL, "kind must be 0, 1 or 2");
    if (!a || !b || !f || !out || (kind == 2 && !c)) return fail(EIK_EINVAL, "null array");
    if (n <= 0) return EIK_OK;
    cudaStream_t st = (cudaStream_t)stream;
    k_local<<<(int)std::min<int64_t>((n + 255) / 256, 4096), 256, 0, st>>>(kind, a, b, c, f, (real_t)dx, (real_t)dy,
                                                                          out, n);
    CK(cudaGetLastError());
    CK(cudaStreamSynchronize(st));
    return EIK_OK;
}

}  // extern "C"
