// Remedy step, brick engine (single device, 3D; E/ifim.py:164-218).  Included by eik_ifim.cu.
//
// The grid is cut into 32 x 8 x 8 bricks (one bitmap word per x-row).  Every round r processes
// the bricks that R_r can touch, listed during round r - 1.  A persistent CTA runs a TMA
// pipeline over its share of the list:
//
//   * producer warp: grabs the next brick, arms the stage's mbarrier, and issues
//       - cp.async.bulk.tensor (TMA) of the phi box  (32+4) x (8+2) x (8+2) from P[r & 1]
//         (the brick plus its halo; cells outside the grid arrive as 0 and are
//         replaced by +inf on the edge path, E/_kernels.py:21-38),
//       - TMA of the brick's d = delta/F tile (32 x 8 x 8),
//       - cp.async.bulk of the brick's D_{r-1} rows, its fixed rows and the six face
//         summaries of the neighbours whose D_{r-1} touches it (which ones: the brick's mask
//         word, built by atomics in round r - 1);
//   * 8 consumer warps, one z-plane of the brick each: form the plane's R_r rows
//     (R_r = D_{r-1} u (N(D_{r-1}) \ fixed), E/ifim.py:209-214) from the staged bits, expand
//     the members into a warp list, relax 32 at a time from shared memory (7 stencil loads +
//     d), decrease test (E/ifim.py:203), write P[(r + 1) & 1] (decreases; carries of last
//     round's changes keep the Jacobi double buffer exact), collect D_r bits in shared
//     memory; then write the plane's part of the brick's D_r record and flag / enqueue the
//     bricks R_{r+1} touches.
//
// A brick's D_r record (512 B): own rows [64] | x-low bits u64 | x-high bits u64 | y-low rows
// [8 z] | y-high rows [8 z] | z-low rows [8 y] | z-high rows [8 y].  Records are written
// whole by every processed brick and read only where the mask says they are current, so
// nothing is ever cleared.  |R_r| and |D_r| are counted per warp, summed per CTA and added once
// per round; the loop ends when D_r is empty (R_{r+1} = 0).  Round 0 reads R_0 (the build's
// bitmap, converted by k_brick_prep) without dilation.

#ifndef BRK_NST
#define BRK_NST 2  // pipeline stages per CTA
#endif
#ifndef BRK_PSLEEP
#define BRK_PSLEEP 256  // producer back-off (ns) while its next stage is busy
#endif
#ifndef BRK_CSLEEP
#define BRK_CSLEEP 64  // consumer back-off (ns) while the next brick is in flight
#endif
#ifndef BRK_CTAS
#define BRK_CTAS 2  // CTAs per SM the register budget is sized for
#endif

namespace brk {

constexpr int BX = 32, BY = 8, BZ = 8;          // brick (x is one bitmap word)
// phi box with halo.  The box's first x coordinate times the element size must be a multiple of
// 16 bytes (an odd float64 start is an illegal instruction, tools/cuda/tma_probe.cu), so the x
// halo is XP = 16 / sizeof(real) cells wide on each side; y and z have a 1-cell halo.
constexpr int XP = 16 / (int)sizeof(real_t);
constexpr int HX = BX + 2 * XP, HY = BY + 2, HZ = BZ + 2;
constexpr int NCW = 8;                          // consumer warps (one z-plane each)
constexpr int THREADS = (NCW + 1) * 32;         // + the producer warp
constexpr uint32_t BOX_BYTES = HX * HY * HZ * sizeof(real_t);
constexpr uint32_t DT_BYTES = BX * BY * BZ * sizeof(real_t);
constexpr uint32_t a128(uint32_t x) { return (x + 127u) & ~127u; }
constexpr uint32_t OFF_BOX = 0;
constexpr uint32_t OFF_DT = a128(BOX_BYTES);
constexpr uint32_t OFF_OWN = OFF_DT + DT_BYTES;  // 256 B
constexpr uint32_t OFF_FIX = OFF_OWN + 256;      // 256 B
constexpr uint32_t OFF_XW = OFF_FIX + 256;       // 16 B: west neighbour's x words (we use x-high)
constexpr uint32_t OFF_XE = OFF_XW + 16;         // 16 B: east neighbour's x words (x-low)
constexpr uint32_t OFF_YS = OFF_XE + 16;         // 32 B: south's y-high rows
constexpr uint32_t OFF_YN = OFF_YS + 32;         // north's y-low rows
constexpr uint32_t OFF_ZD = OFF_YN + 32;         // down's z-high rows
constexpr uint32_t OFF_ZU = OFF_ZD + 32;         // up's z-low rows
constexpr uint32_t OFF_HDR = OFF_ZU + 32;        // brick id, mask
constexpr uint32_t STAGE = a128(OFF_HDR + 16);
constexpr uint32_t OFF_BARS = BRK_NST * STAGE;                 // full[NST], empty[NST]
constexpr uint32_t OFF_WL = a128(OFF_BARS + 16 * BRK_NST);     // per-warp member lists (uint16)
constexpr uint32_t OFF_WD = OFF_WL + NCW * 256 * 2;             // per-warp D rows [8]
constexpr uint32_t OFF_RED = OFF_WD + NCW * 8 * 4;              // reduction scratch
constexpr uint32_t SMEM = OFF_RED + 2 * 8 * (NCW + 1) + 1024;  // + alignment slack of the base

// record layout (32-bit words)
constexpr int R_OWN = 0, R_XL = 64, R_XH = 66, R_YL = 68, R_YH = 76, R_ZL = 84, R_ZH = 92, R_WORDS = 128;
// mask bits: which records of round r - 1 a brick reads in round r
constexpr uint32_t MK_SELF = 1, MK_W = 2, MK_E = 4, MK_S = 8, MK_N = 16, MK_D = 32, MK_U = 64;
constexpr uint32_t END = 0xffffffffu;

__device__ __forceinline__ unsigned *len_slot(const KP &p, uint32_t k) { return p.bcnt + k * 32u; }
__device__ __forceinline__ unsigned *grab_slot(const KP &p, uint32_t k) { return p.bcnt + (3u + k) * 32u; }

__device__ __forceinline__ uint32_t sa(const void *ptr) { return (uint32_t)__cvta_generic_to_shared(ptr); }

__device__ __forceinline__ void mbar_init(uint64_t *b, unsigned count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(sa(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b)
{
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(sa(b)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t *b, unsigned tx)
{
    asm volatile("mbarrier.arrive.expect_tx.release.cta.shared::cta.b64 _, [%0], %1;" ::"r"(sa(b)), "r"(tx) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t *b, unsigned parity)
{
    uint32_t ok;
    asm volatile(
        "{\n .reg .pred q;\n mbarrier.try_wait.parity.acquire.cta.shared::cta.b64 q, [%1], %2;\n"
        " selp.u32 %0, 1, 0, q;\n}"
        : "=r"(ok)
        : "r"(sa(b)), "r"(parity)
        : "memory");
    return ok != 0;
}
// Wait for a phase; a phase that never completes (a logic error) trips the watchdog instead of
// wedging the GPU.
template <unsigned SLEEP_NS>
__device__ __forceinline__ bool mbar_wait(uint64_t *b, unsigned parity, Ctl *ctl)
{
    if (mbar_try(b, parity)) return true;
    const unsigned long long t0 = globaltimer();
    for (unsigned k = 0;; ++k) {
        if (SLEEP_NS) __nanosleep(SLEEP_NS);  // a waiting warp yields its issue slots to the working ones
        if (mbar_try(b, parity)) return true;
        if ((k & 63u) == 63u &&
            (*(volatile unsigned *)&ctl->err == EIK_EHANG || globaltimer() - t0 > 10000000000ull)) {
            atomicExch(&ctl->err, EIK_EHANG);
            return false;
        }
    }
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *tm, int x, int y, int z, uint64_t *bar)
{
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(sa(dst)), "l"(tm), "r"(x), "r"(y), "r"(z), "r"(sa(bar))
        : "memory");
}
__device__ __forceinline__ void bulk(void *dst, const void *src, unsigned bytes, uint64_t *bar)
{
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(sa(dst)), "l"(src), "r"(bytes), "r"(sa(bar))
                 : "memory");
}
__device__ __forceinline__ void fence_async() { asm volatile("fence.proxy.async;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

}  // namespace brk

// Round 0 set-up: R_0 rows (the build's row-major bitmap) into record buffer 1, fixed rows
// brick-major (rows outside the grid: all fixed), list 0 = the bricks holding R_0 members.
// One warp per brick; lane l handles rows l and l + 32 (row j = plane j / 8, y = j % 8).
__global__ void __launch_bounds__(256) k_brick_prep(KP p, const unsigned *skip)
{
    if (skip && *skip) return;
    const uint32_t warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = lane_id();
    const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
    for (uint32_t b = warp; b < p.nbricks; b += nwarps) {
        const uint32_t t = fdiv(b, p.fnbx), bx = b - t * p.nbx;
        const uint32_t bz = fdiv(t, p.fnby), by = t - bz * p.nby;
        uint32_t any = 0;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t j = lane + 32u * h, y = by * 8u + (j & 7u), z = bz * 8u + (j >> 3);
            uint32_t r0 = 0, fx = FULL;
            if (y < (uint32_t)p.ny && z < (uint32_t)p.nz) {
                const uint32_t w = (z * (uint32_t)p.ny + y) * p.W + bx;
                r0 = __ldcg(p.R0b + w);
                fx = __ldg(p.Fb + w);
            }
            p.brec1[(size_t)b * brk::R_WORDS + j] = r0;
            p.bfix[(size_t)b * 64u + j] = fx;
            any |= r0;
        }
        if (__ballot_sync(FULL, any != 0) && lane == 0) {
            p.bmask[b] = brk::MK_SELF;  // slot 0
            p.blist0[atomicAdd(brk::len_slot(p, 0), 1u)] = b;
        }
    }
}

// Auto mode: the brick pipeline for dense remedy sets (|R_0| >= pct % of the cells), the member
// list otherwise.  Writes each kernel's skip word (an update-step error skips both).
__global__ void k_choose_remedy(Ctl *ctl, const unsigned *skip, unsigned *sel, unsigned long long ncells, unsigned pct)
{
    const bool err = skip && *skip;
    const bool dense = ctl->flagged * 100ull >= (unsigned long long)pct * ncells;
    sel[0] = err || dense;
    sel[32] = err || !dense;
    ctl->engine = dense ? 3u : 1u;
}

template <int SOL>
__global__ void __launch_bounds__(brk::THREADS, BRK_CTAS)
    k_remedy_b(KP p, const unsigned *skip, const __grid_constant__ CUtensorMap tmP0,
               const __grid_constant__ CUtensorMap tmP1, const __grid_constant__ CUtensorMap tmD)
{
    using namespace brk;
    extern __shared__ __align__(1024) unsigned char sm_raw[];
    // TMA destinations need 128-byte-aligned shared addresses: align the base explicitly
    unsigned char *sm = sm_raw + ((1024u - (sa(sm_raw) & 1023u)) & 1023u);
    if (skip && *skip) return;
    Ctl *ctl = p.ctl;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const bool lead = blockIdx.x == 0 && threadIdx.x == 0;
    uint64_t *full = (uint64_t *)(sm + OFF_BARS), *empty = full + BRK_NST;
    unsigned long long *sred = (unsigned long long *)(sm + OFF_RED);
    const unsigned long long r0 = vload(&ctl->flagged);
    if (r0 == 0) return;  // empty remedy set: zero rounds
    if (threadIdx.x == 0) {
        for (int s = 0; s < BRK_NST; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, NCW);
            ((uint32_t *)(sm + s * STAGE + OFF_HDR))[2] = 0;  // per-stage face / arrival word
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        fence_async();
    }
    if (lead) {
        ctl->peak = r0;
        ctl->sum = 0;
    }
    __syncthreads();
    const uint32_t nx = p.nx32, ny = (uint32_t)p.ny, nz = (uint32_t)p.nz;
    const uint32_t nb = p.nbricks, nbx = p.nbx, nby = p.nby, nbz = p.nbz, nbxy = nbx * nby;
    uint32_t it = 0;  // pipeline item counter (stage = it % NST, phase = (it / NST) & 1)
    for (uint32_t r = 0;; ++r) {
        const uint32_t *mask_r = p.bmask + (r % 3u) * nb;
        uint32_t *mask_n = p.bmask + ((r + 1u) % 3u) * nb;
        const uint32_t *list_r = (r & 1u) ? p.blist1 : p.blist0;
        uint32_t *list_n = (r & 1u) ? p.blist0 : p.blist1;
        const uint32_t *recP = (r & 1u) ? p.brec0 : p.brec1;  // D_{r-1} (round 0: R_0)
        uint32_t *recN = (r & 1u) ? p.brec1 : p.brec0;        // D_r
        unsigned long long a_mem = 0, a_dec = 0;
        if (warp == NCW) {
            // ------------------------------ producer ------------------------------
            const CUtensorMap *tmc = (r & 1u) ? &tmP1 : &tmP0;
            const uint32_t len = vload(len_slot(p, r % 3u));
            unsigned *grab = grab_slot(p, r % 3u);
            fence_async();  // last round's generic writes (phi, records) before this round's async reads
            auto fetch = [&](uint32_t &bid, uint32_t &msk) {
                uint32_t i = 0;
                if (lane == 0) i = atomicAdd(grab, 1u);
                i = __shfl_sync(FULL, i, 0);
                bid = END;
                msk = 0;
                if (i < len) {
                    bid = __ldcg(list_r + i);
                    msk = __ldcg(mask_r + bid);
                }
            };
            uint32_t bid, msk;
            fetch(bid, msk);
            for (;;) {
                const uint32_t s = it % BRK_NST, ph = (it / BRK_NST) & 1u;
                unsigned char *st = sm + s * STAGE;
                if (!mbar_wait<BRK_PSLEEP>(empty + s, ph ^ 1u, ctl)) return;
                if (lane == 0) {
                    uint32_t *hdr = (uint32_t *)(st + OFF_HDR);
                    hdr[0] = bid;
                    hdr[1] = msk;
                    if (bid == END) {
                        mbar_arrive(full + s);
                    } else {
                        const uint32_t t = fdiv(bid, p.fnbx), bx = bid - t * nbx;
                        const uint32_t bz = fdiv(t, p.fnby), by = t - bz * nby;
                        const uint32_t *rp = recP + (size_t)bid * R_WORDS;
                        unsigned tx = BOX_BYTES + DT_BYTES + 256u;
                        if (msk & MK_SELF) tx += 256u;
                        if (r > 0) {
                            tx += ((msk & MK_W) ? 16u : 0u) + ((msk & MK_E) ? 16u : 0u) + ((msk & MK_S) ? 32u : 0u) +
                                  ((msk & MK_N) ? 32u : 0u) + ((msk & MK_D) ? 32u : 0u) + ((msk & MK_U) ? 32u : 0u);
                        }
                        mbar_arrive_tx(full + s, tx);
                        const int x0 = (int)bx * BX, y0 = (int)by * BY, z0 = (int)bz * BZ;
                        tma3(st + OFF_BOX, tmc, x0 - XP, y0 - 1, z0 - 1, full + s);
                        tma3(st + OFF_DT, &tmD, x0, y0, z0, full + s);
                        bulk(st + OFF_FIX, p.bfix + (size_t)bid * 64u, 256u, full + s);
                        if (msk & MK_SELF) bulk(st + OFF_OWN, rp + R_OWN, 256u, full + s);
                        if (r > 0) {
                            if (msk & MK_W) bulk(st + OFF_XW, rp - R_WORDS + R_XL, 16u, full + s);
                            if (msk & MK_E) bulk(st + OFF_XE, rp + R_WORDS + R_XL, 16u, full + s);
                            if (msk & MK_S) bulk(st + OFF_YS, rp - (size_t)nbx * R_WORDS + R_YH, 32u, full + s);
                            if (msk & MK_N) bulk(st + OFF_YN, rp + (size_t)nbx * R_WORDS + R_YL, 32u, full + s);
                            if (msk & MK_D) bulk(st + OFF_ZD, rp - (size_t)nbxy * R_WORDS + R_ZH, 32u, full + s);
                            if (msk & MK_U) bulk(st + OFF_ZU, rp + (size_t)nbxy * R_WORDS + R_ZL, 32u, full + s);
                        }
                    }
                }
                __syncwarp();
                ++it;
                if (bid == END) break;
                fetch(bid, msk);
            }
        } else {
            // ------------------------------ consumers ------------------------------
            real_t *__restrict__ Pn = (r & 1u) ? p.P0 : p.P1;
            uint16_t *wl = (uint16_t *)(sm + OFF_WL) + warp * 256;
            uint32_t *wd = (uint32_t *)(sm + OFF_WD) + warp * 8;
            const uint32_t lt = (1u << lane) - 1u;
            unsigned *len_n = len_slot(p, (r + 1u) % 3u);
            // deferred enqueue: p1 = atomicOr results on the next round's masks (a 0 means this
            // warp flagged the brick first), p2 = reserved list slots of the newly flagged bricks
            bool p1v = false, p2v = false;
            uint32_t p1nb = 0, p1old = 0, p2nb = 0, p2rank = 0, p2base = 0;
            auto resolve_pending = [&]() {
                const uint32_t base = __shfl_sync(FULL, p2base, 0);
                if (p2v) list_n[base + p2rank] = p2nb;
                const uint32_t fresh = __ballot_sync(FULL, p1v && p1old == 0u);
                p2v = (fresh >> lane) & 1u;
                p2nb = p1nb;
                p2rank = __popc(fresh & lt);
                if (fresh && lane == 0) p2base = atomicAdd(len_n, (unsigned)__popc(fresh));
                p1v = false;
            };
            // slot upkeep for later rounds: mask / length / grab slot (r + 2) % 3 was last used in
            // round r - 1
            {
                uint32_t *mclr = p.bmask + ((r + 2u) % 3u) * nb;
                for (uint32_t i = blockIdx.x * (NCW * 32) + threadIdx.x; i < nb; i += gridDim.x * (NCW * 32)) mclr[i] = 0;
                if (blockIdx.x == 0 && threadIdx.x == 0) {
                    *len_slot(p, (r + 2u) % 3u) = 0;
                    *grab_slot(p, (r + 2u) % 3u) = 0;
                    ctl->cnt[(r + 1u) % 3u] = 0;
                    ctl->dsum[(r + 1u) % 3u] = 0;
                }
            }
            for (;;) {
                const uint32_t s = it % BRK_NST, ph = (it / BRK_NST) & 1u;
                const unsigned char *st = sm + s * STAGE;
                if (!mbar_wait<BRK_CSLEEP>(full + s, ph, ctl)) return;
                const uint32_t *hdr = (const uint32_t *)(st + OFF_HDR);
                const uint32_t bid = hdr[0], msk = hdr[1];
                if (bid == END) {
                    __syncwarp();
                    if (lane == 0) mbar_arrive(empty + s);
                    ++it;
                    break;
                }
                const uint32_t t = fdiv(bid, p.fnbx), bx = bid - t * nbx;
                const uint32_t bz = fdiv(t, p.fnby), by = t - bz * nby;
                const uint32_t x0 = bx * BX, y0 = by * BY, z0 = bz * BZ, z = z0 + warp;
                real_t *box = (real_t *)(st + OFF_BOX);
                // cells of this warp's box plane outside the grid in x or y are +inf (E/_kernels.py:21-38;
                // the TMA fills them with 0).  A warp's members read x/y neighbours only in its own
                // plane; the z-neighbours outside the grid are handled by warp-uniform tests below.
                const bool xy_edge = x0 == 0 || x0 + BX >= nx || y0 == 0 || y0 + BY >= ny;
                if (xy_edge && z < nz) {
                    real_t *pl = box + (warp + 1u) * (HX * HY);
                    // box columns [0, xl) and [xh, HX), rows [0, yl) and [yh, HY) lie outside the grid
                    const uint32_t xl = x0 == 0 ? (uint32_t)XP : 0u, xh = min((uint32_t)HX, XP + nx - x0);
                    const uint32_t yl = y0 == 0 ? 1u : 0u, yh = min((uint32_t)HY, 1u + ny - y0);
                    for (uint32_t iy = 0; iy < (uint32_t)HY; ++iy)
                        if (iy < yl || iy >= yh)
                            for (uint32_t ix = lane; ix < (uint32_t)HX; ix += 32) pl[iy * HX + ix] = INFINITY;
                    const uint32_t nc = xl + (HX - xh);  // out-of-grid columns per row
                    for (uint32_t k = lane; k < nc * (yh - yl); k += 32) {
                        const uint32_t r = k / nc, cc = k - r * nc;
                        pl[(yl + r) * HX + (cc < xl ? cc : xh + (cc - xl))] = INFINITY;
                    }
                    __syncwarp();
                }
                const uint32_t *own = (const uint32_t *)(st + OFF_OWN);
                const bool self = msk & MK_SELF;
                // ---- R_r rows of this plane (lanes 0..7: row y = lane) ----
                uint32_t R = 0, carry = 0;
                if (lane < 8) {
                    const uint32_t j = warp * 8u + lane;
                    const uint32_t c = self ? own[j] : 0u;
                    if (r == 0) {
                        R = c;  // R_0 exactly (E/ifim.py:184)
                    } else {
                        const uint32_t fx = ((const uint32_t *)(st + OFF_FIX))[j];
                        const uint32_t wv = (msk & MK_W) ? (uint32_t)(((const unsigned long long *)(st + OFF_XW))[1] >> j) & 1u : 0u;
                        const uint32_t ev = (msk & MK_E) ? (uint32_t)(((const unsigned long long *)(st + OFF_XE))[0] >> j) & 1u : 0u;
                        const uint32_t sv = lane > 0 ? (self ? own[j - 1] : 0u) : ((msk & MK_S) ? ((const uint32_t *)(st + OFF_YS))[warp] : 0u);
                        const uint32_t nv = lane < 7 ? (self ? own[j + 1] : 0u) : ((msk & MK_N) ? ((const uint32_t *)(st + OFF_YN))[warp] : 0u);
                        const uint32_t dv = warp > 0 ? (self ? own[j - 8] : 0u) : ((msk & MK_D) ? ((const uint32_t *)(st + OFF_ZD))[lane] : 0u);
                        const uint32_t uv = warp < 7 ? (self ? own[j + 8] : 0u) : ((msk & MK_U) ? ((const uint32_t *)(st + OFF_ZU))[lane] : 0u);
                        const uint32_t dil = (c << 1) | (c >> 1) | wv | (ev << 31) | sv | nv | dv | uv;
                        R = c | (dil & ~fx);
                        carry = c;
                    }
                    wd[lane] = 0;
                }
                // ---- members: warp list (carry << 8 | y << 5 | x); lane l expands byte l & 3 of row l >> 2 ----
                const uint32_t ly = lane >> 2, sh = (lane & 3u) * 8u;
                uint32_t Rb = (__shfl_sync(FULL, R, ly) >> sh) & 0xffu;
                const uint32_t Cb = (__shfl_sync(FULL, carry, ly) >> sh) & 0xffu;
                const uint32_t cnt = __popc(Rb);
                uint32_t inc = cnt;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const uint32_t v = __shfl_up_sync(FULL, inc, o);
                    if (lane >= (unsigned)o) inc += v;
                }
                const uint32_t T = __shfl_sync(FULL, inc, 31);
                uint32_t off = inc - cnt;
                while (Rb) {
                    const uint32_t b = __ffs(Rb) - 1;
                    Rb &= Rb - 1;
                    wl[off++] = (uint16_t)((((Cb >> b) & 1u) << 8) | (ly << 5) | (sh + b));
                }
                __syncwarp();
                const real_t *dt = (const real_t *)(st + OFF_DT);
                const bool zlo = z == 0, zhi = z + 1 >= nz;
                unsigned ndec = 0;
                for (uint32_t b0 = 0; b0 < T; b0 += 64) {
                    uint32_t e[2];
                    bool live[2];
                    Sten sn[2];
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        const uint32_t i = b0 + u * 32 + lane;
                        live[u] = i < T;
                        e[u] = live[u] ? (uint32_t)wl[i] : 0u;
                        const uint32_t y = (e[u] >> 5) & 7u, x = e[u] & 31u;
                        const uint32_t hi = ((warp + 1u) * HY + (y + 1u)) * HX + (x + XP);
                        sn[u].c = box[hi];
                        sn[u].w = box[hi - 1];
                        sn[u].e = box[hi + 1];
                        sn[u].s = box[hi - HX];
                        sn[u].n = box[hi + HX];
                        sn[u].d = zlo ? (real_t)INFINITY : box[hi - HX * HY];
                        sn[u].u = zhi ? (real_t)INFINITY : box[hi + HX * HY];
                        sn[u].k = dt[(warp * 8u + y) * BX + x];
                    }
#pragma unroll
                    for (int u = 0; u < 2; ++u) {
                        bool dec = false;
                        if (live[u]) {
                            const uint32_t y = (e[u] >> 5) & 7u, x = e[u] & 31u;
                            const real_t v = solve<3, SOL>(p, sn[u]);
                            dec = v < sn[u].c - tol_at(p.tol, sn[u].c);  // E/ifim.py:203
                            const uint32_t c = (z * ny + y0 + y) * nx + x0 + x;
                            if (dec) {
                                Pn[c] = v;
                                atomicOr(wd + y, 1u << x);
                            } else if (e[u] >> 8) {
                                Pn[c] = sn[u].c;  // changed last round: carry into the other buffer
                            }
                        }
                        ndec += __popc(__ballot_sync(FULL, dec));
                    }
                }
                __syncwarp();
                if (xy_edge) fence_async_smem();  // generic writes to the stage before its next TMA fill
                // ---- D_r record of this plane ----
                const uint32_t Dw = lane < 8 ? wd[lane] : 0u;
                uint32_t *rn = recN + (size_t)bid * R_WORDS;
                const uint32_t bl = __ballot_sync(FULL, Dw & 1u) & 0xffu, bh = __ballot_sync(FULL, Dw >> 31) & 0xffu;
                const uint32_t any = __ballot_sync(FULL, Dw != 0u);
                const uint32_t d_y0 = __shfl_sync(FULL, Dw, 0), d_y7 = __shfl_sync(FULL, Dw, 7);
                if (lane < 8) {
                    rn[R_OWN + warp * 8u + lane] = Dw;
                    if (warp == 0) rn[R_ZL + lane] = Dw;
                    if (warp == NCW - 1) rn[R_ZH + lane] = Dw;
                }
                if (lane == 0) {
                    ((uint8_t *)(rn + R_XL))[warp] = (uint8_t)bl;
                    ((uint8_t *)(rn + R_XH))[warp] = (uint8_t)bh;
                    rn[R_YL + warp] = d_y0;
                    rn[R_YH + warp] = d_y7;
                }
                // ---- bricks R_{r+1} touches: the brick's faces are OR-ed per stage in shared memory;
                // the last warp to arrive flags them (atomicOr on the next round's masks) and enqueues
                // the newly flagged ones.  The atomics' results are consumed one brick later
                // (pend_*), so no warp waits on their latency. ----
                resolve_pending();
                uint32_t fb = (any ? 1u : 0u) | (bl ? 2u : 0u) | (bh ? 4u : 0u) | (d_y0 ? 8u : 0u) | (d_y7 ? 16u : 0u) |
                              ((warp == 0 && any) ? 32u : 0u) | ((warp == NCW - 1 && any) ? 64u : 0u);
                uint32_t all = 0;
                if (lane == 0) {
                    uint32_t *sfw = (uint32_t *)(st + OFF_HDR) + 2;
                    const uint32_t mine = fb | (0x100u << warp);
                    all = atomicOr(sfw, mine) | mine;
                    if ((all >> 8) == 0xffu) *sfw = 0;  // last of the brick's warps: reset for the stage's next use
                }
                all = __shfl_sync(FULL, all, 0);
                if ((all >> 8) == 0xffu && lane < 7 && ((all >> lane) & 1u)) {
                    uint32_t nbid = bid, flag = MK_SELF;
                    bool ex = true;
                    switch (lane) {
                        case 0: break;
                        case 1: ex = bx > 0; nbid = bid - 1; flag = MK_E; break;
                        case 2: ex = bx + 1 < nbx; nbid = bid + 1; flag = MK_W; break;
                        case 3: ex = by > 0; nbid = bid - nbx; flag = MK_N; break;
                        case 4: ex = by + 1 < nby; nbid = bid + nbx; flag = MK_S; break;
                        case 5: ex = bz > 0; nbid = bid - nbxy; flag = MK_U; break;
                        default: ex = bz + 1 < nbz; nbid = bid + nbxy; flag = MK_D; break;
                    }
                    if (ex) {
                        p1v = true;
                        p1nb = nbid;
                        p1old = atomicOr(mask_n + nbid, flag);
                    }
                }
                if (lane == 0) {
                    a_mem += T;
                    a_dec += ndec;
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(empty + s);
                ++it;
            }
            resolve_pending();  // the last brick's flags
            resolve_pending();
            fence_async();  // this round's generic writes before next round's async (TMA) reads
        }
        // ---- round totals, barrier, termination (as k_remedy_t) ----
        {
            unsigned long long m = warp_sum(a_mem), d = warp_sum(a_dec);
            __syncthreads();
            if (lane == 0) {
                sred[warp] = m;
                sred[NCW + 1 + warp] = d;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                unsigned long long tm = 0, td = 0;
                for (int w = 0; w <= NCW; ++w) {
                    tm += sred[w];
                    td += sred[NCW + 1 + w];
                }
                if (tm) atomicAdd(&ctl->cnt[r % 3u], tm);
                if (td) {
                    atomicAdd(&ctl->dsum[r % 3u], td);
                    atomicAdd(&ctl->writes, td);
                }
            }
        }
        if (!grid_barrier(ctl)) return;
        const unsigned long long mg = vload(&ctl->cnt[r % 3u]);   // |R_r|
        const unsigned long long dg = vload(&ctl->dsum[r % 3u]);  // |D_r|
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
