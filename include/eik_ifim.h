/*
 * eik_ifim.h -- C ABI of the B200 iFIM engine (libeik_ifim.so).
 *
 * Drop-in boundary for the reference's iFIM path.  The reference is a Python
 * package (`eikonal`, /root/reference/pkg/src/eikonal = E/) with no native
 * code; its "operator API" for this path is the Python solver signature
 * family, which paper_2106_15869_b200/ifim.py keeps and binds to these entry
 * points through ctypes (see INTEGRATION.md for the binding a maintainer of
 * the reference would add).
 *
 *   eik_ifim_update_step  replaces ifim_update_step  (E/ifim.py:75-134)
 *   eik_build_remedy      replaces build_remedy_set  (E/ifim.py:137-161)
 *   eik_remedy_step       replaces ifim_remedy_step  (E/ifim.py:164-218)
 *   eik_ifim_solve        replaces solve_ifim        (E/ifim.py:221-235)
 *   eik_remedy_load / eik_remedy_export
 *                         replace RemedySet's member mask (E/ifim.py:64-72)
 *   eik_local_solve       replaces update_batch / update_3d_uniform
 *                         (E/_kernels.py:41-88, E/local_solver.py:91-157)
 *
 * Conventions (E/grid.py:1-8, 21-26): phi float64 with +inf = unreached,
 * speed float64 >= 0 (0 = Blocked), state uint8 CellState codes
 * {FAR 0, ACTIVE 1, SOURCE 2, REMEDY 3, BLOCKED 4}; linear index j*nx+i in 2D
 * and (k*ny+j)*nx+i in 3D.  All array pointers are DEVICE pointers; `stream`
 * is a cudaStream_t passed as void*.  Every function returns an int status
 * (EIK_OK ...); the message of the last failure on the calling thread is
 * available from eik_last_error().  The caller allocates the workspace
 * (eik_workspace_size); the library allocates nothing persistently.  Calls
 * block until their statistics are on the host.
 */
#ifndef EIK_IFIM_H
#define EIK_IFIM_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define EIK_OK 0
#define EIK_EINVAL 1 /* -> ValueError   (E/ifim.py:83-84, E/grid.py:204-211) */
#define EIK_ECAP 2   /* -> RuntimeError (E/ifim.py:109-110, 188-189) */
#define EIK_ECUDA 3
#define EIK_ENCCL 4

#define EIK_F64 0 /* libeik_ifim.so: float64 fields, bit-exact with the reference */
#define EIK_F32 1 /* libeik_ifim_f32.so: float32 fields (perf mode), names suffixed _f32 */

#define EIK_GEOM_SLAB 1 /* flags: local z-slab of a sharded 3D grid, planes 0 and nz-1 are ghosts */

typedef struct eik_geom {
    int64_t nx, ny, nz; /* nz = 1 for 2D */
    double dx, dy, dz;  /* 3D requires dx == dy == dz */
    int32_t ndim;       /* 2 or 3 */
    int32_t dtype;      /* EIK_F64 */
    int32_t flags;      /* EIK_GEOM_SLAB or 0 */
    int32_t reserved;
} eik_geom;

/* RunStats (E/result.py:9-18) plus device-side extras. */
typedef struct eik_stats {
    int64_t iterations;   /* update iterations + remedy rounds */
    int64_t solver_calls; /* local-solver invocations (node updates) */
    int64_t peak_active;
    int64_t peak_remedy;
    int64_t phi_writes;   /* non-converged update writes + remedy decreases */
    int64_t history_len;  /* entries written to the active_history buffer */
    int64_t remedy_size;  /* cells flagged by the build pass */
    int64_t converged;    /* cells labelled CONVERGED by the update step */
    int64_t upd_iterations, upd_calls, build_calls, rem_iterations, rem_calls;
    int64_t gpu_launches; /* kernels launched by this call */
    float upd_ms, build_ms, rem_ms, total_ms; /* device time (CUDA events) */
} eik_stats;

/* Bytes of device workspace needed for a grid. */
int eik_workspace_size(const eik_geom *g, size_t *bytes);

/* Update step (E/ifim.py:75-134).  Applies the seeds first (E/grid.py:212-215:
 * phi[seed] = value, state[seed] = SOURCE); seed_idx/seed_val are device
 * arrays of nseeds linear indices and values, validated by the caller.
 * history (HOST, int64[history_cap]) receives active_history. */
int eik_ifim_update_step(const eik_geom *g, double *phi, const double *speed, uint8_t *state,
                         const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                         void *workspace, size_t workspace_bytes, int64_t *history,
                         int64_t history_cap, eik_stats *out, void *stream);

/* Build pass (E/ifim.py:137-161).  Leaves the remedy set in the workspace;
 * out->remedy_size = |R0|, out->solver_calls = #free cells. */
int eik_build_remedy(const eik_geom *g, const double *phi, const double *speed, const uint8_t *state,
                     double tol, void *workspace, size_t workspace_bytes, eik_stats *out, void *stream);

/* Load a remedy set from a device bool/uint8 mask[N] (a RemedySet built elsewhere). */
int eik_remedy_load(const eik_geom *g, const uint8_t *member, const uint8_t *state, void *workspace,
                    size_t workspace_bytes, int64_t *count, void *stream);

/* Load a hand-built RemedySet (E/ifim.py:64-72): `cells` marks its work list (the cells the first
 * round relaxes), `member` its membership mask (NULL: equal to cells).  Members outside the work
 * list are never relaxed and never enqueued (E/ifim.py:184-213).  *count = |work list|. */
int eik_remedy_load_set(const eik_geom *g, const uint8_t *cells, const uint8_t *member, const uint8_t *state,
                        void *workspace, size_t workspace_bytes, int64_t *count, void *stream);

/* Verification reductions on device fields (E/harness.py:165-179).  eik_field_max_diff: max |a - b|
 * over n values, equal same-sign infinities count 0, NaN propagates, 0.0 for n == 0; `scratch` is
 * 16 bytes of device memory.  eik_chunk_sha256: SHA-256 (FIPS 180-4) of every `chunk`-byte piece of
 * the device byte range (the last one may be short) into digests[32 * pieces] (device); the
 * package's field_digest hashes the concatenated piece digests on the host. */
int eik_field_max_diff(const double *a, const double *b, int64_t n, void *scratch, double *out, void *stream);
int eik_chunk_sha256(const void *data, int64_t nbytes, int64_t chunk, uint8_t *digests, void *stream);

/* Write the workspace remedy set as a device uint8 mask[N]. */
int eik_remedy_export(const eik_geom *g, void *workspace, size_t workspace_bytes, uint8_t *member,
                      void *stream);

/* Remedy step (E/ifim.py:164-218) on the workspace remedy set; drains it. */
int eik_remedy_step(const eik_geom *g, double *phi, const double *speed, const uint8_t *state,
                    double tol, void *workspace, size_t workspace_bytes, eik_stats *out, void *stream);

/* solve_ifim (E/ifim.py:221-235): update step + build + remedy, device-resident,
 * one host synchronisation at the end. */
int eik_ifim_solve(const eik_geom *g, double *phi, const double *speed, uint8_t *state,
                   const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                   void *workspace, size_t workspace_bytes, int64_t *history, int64_t history_cap,
                   eik_stats *out, void *stream);

/* Element-wise local solver on device arrays (parity hook for
 * E/_kernels.py:41-88 and E/local_solver.py:91-157).  kind: 0 = 2D uniform
 * (a, b, f, dx), 1 = 2D anisotropic (a, b, f, dx, dy), 2 = 3D uniform
 * (a, b, c, f, dx).  dx <= 0 (kinds 0 and 2): each element's spacing is read
 * from out[i] before the result overwrites it. */
int eik_local_solve(int kind, const double *a, const double *b, const double *c, const double *f,
                    double dx, double dy, double *out, int64_t n, void *stream);

/* solve_fixpoint (E/oracle.py:22-70): full-grid Jacobi passes, the independent
 * ground truth; max_passes <= 0 selects the reference cap 10*(nx+ny[+nz]).
 * out->iterations = passes, out->solver_calls = passes * free cells. */
int eik_solve_fixpoint(const eik_geom *g, double *phi, const double *speed, uint8_t *state,
                       const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                       int64_t max_passes, void *workspace, size_t workspace_bytes, eik_stats *out, void *stream);

/* solve_fim (E/fim.py:62-144): the FIM baseline with
 * per-iteration neighbour checks.  out: iterations, solver_calls (active
 * recomputations + one per neighbour examination), peak_active, phi_writes. */
int eik_solve_fim(const eik_geom *g, double *phi, const double *speed, uint8_t *state, const int64_t *seed_idx,
                  const double *seed_val, int64_t nseeds, double tol, void *workspace, size_t workspace_bytes,
                  eik_stats *out, void *stream);

/* max_residual (E/harness.py:147-162): largest |phi - U(phi)| over free cells with finite phi. */
int eik_max_residual(const eik_geom *g, const double *phi, const double *speed, const uint8_t *state,
                     void *workspace, size_t workspace_bytes, double *out, void *stream);

/* ---- z-slab sharding (protocol in paper_2106_15869_b200/slab.py) ----
 * The geometry is the rank's local slab with one ghost plane on each side
 * (flags = EIK_GEOM_SLAB, nz = owned planes + 2).  Every call runs one
 * bulk-synchronous step on the given stream and returns the LOCAL counts; the
 * caller exchanges ghost planes / requests / decrease planes and reduces the
 * counts between steps.  Workspace offsets of the buffers the exchange touches
 * come from eik_workspace_offsets: [0] second phi buffer (float64), [1] touched
 * bitmap (update: ghost rows = outgoing activation requests), [2] D0, [3] D1
 * (remedy decrease bitmaps by round parity); bitmaps have ceil(nx/32) uint32
 * words per x-row, rows ordered (z, y). */
int eik_workspace_offsets(const eik_geom *g, int64_t *offsets /* [4] */);
/* Seeds (local linear indices, owned or ghost planes) + initial activation of
 * owned cells (E/ifim.py:97-102); *n_active = local |A_1|. */
int eik_slab_update_init(const eik_geom *g, double *phi, const double *speed, uint8_t *state,
                         const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                         void *workspace, size_t workspace_bytes, int64_t *n_active, void *stream);
/* Update iteration `it` (0-based; reads phi buffer it&1, writes (it+1)&1). */
int eik_slab_update_iter(const eik_geom *g, double *phi, const double *speed, uint8_t *state, double tol,
                         int64_t it, void *workspace, size_t workspace_bytes, void *stream);
/* Apply the neighbours' requests (ghost touched rows of rank-1 / rank+1, or
 * NULL) to the owned boundary planes; *n_active = local |A_{it+2}|. */
int eik_slab_apply_requests(const eik_geom *g, const uint32_t *req_lo, const uint32_t *req_hi, int64_t it,
                            void *workspace, size_t workspace_bytes, int64_t *n_active, void *stream);
/* Build pass on the owned planes: local #free and |R0|. */
int eik_slab_build(const eik_geom *g, const double *phi, const double *speed, const uint8_t *state, double tol,
                   void *workspace, size_t workspace_bytes, int64_t *free_cells, int64_t *flagged, void *stream);
/* Remedy round `r` (0 uses R0); local |R_r| and |D_r|. */
int eik_slab_remedy_round(const eik_geom *g, double *phi, const double *speed, const uint8_t *state, double tol,
                          int64_t r, void *workspace, size_t workspace_bytes, int64_t *calls, int64_t *decs,
                          void *stream);

/* ---- multi-rank peer slabs (B200 path: no host round trips) ----
 * One z-sharded 3D grid over R ranks.  Each rank owns consecutive planes and
 * keeps them in its own phi buffer + workspace; the persistent kernels read the
 * neighbours' boundary planes / decrease rows and activate cells on them
 * through device-visible pointers (NVLink peer mappings on a multi-GPU box, or
 * plain device pointers when R ranks are emulated on one GPU), with a
 * hierarchical grid + cross-rank barrier per iteration.  ranks[] describes all
 * R ranks as seen from this process; this process runs ranks [r_begin, r_end)
 * and passes their speed/state arrays.  Seeds are global linear indices.
 * Multi-process use needs a host barrier between eik_mr_prepare and eik_mr_run
 * on every rank.  Stats are global (identical on every rank). */
typedef struct eik_rank {
    double *phi0;    /* the rank's phi (owned planes), result buffer */
    void *workspace; /* the rank's workspace (eik_workspace_size of its local slab geometry) */
    int64_t nz;      /* owned planes */
} eik_rank;
int eik_mr_prepare(const eik_geom *g, int32_t R, const eik_rank *ranks, int32_t r_begin, int32_t r_end,
                   const double *const *speed, uint8_t *const *state, const int64_t *seeds, const double *seed_val,
                   int64_t nseeds, double tol, void *stream);
int eik_mr_run(const eik_geom *g, int32_t R, const eik_rank *ranks, int32_t r_begin, int32_t r_end,
               const double *const *speed, uint8_t *const *state, double tol, int64_t *history, int64_t history_cap,
               eik_stats *out, void *stream);

/* Let `device` map `peer`'s memory (NVLink / NVSwitch P2P); single-process multi-GPU peer slabs. */
int eik_peer_enable(int32_t device, int32_t peer);

const char *eik_last_error(void);
const char *eik_version(void);
/* Which engine ran the calling thread's last remedy step: 0 none, 1 member list (k_remedy),
 * 2 tile (k_remedy_t), 3 TMA brick pipeline (k_remedy_b).  Selection: EIK_REMEDY=list|tile|brick,
 * else auto (3D single device, brick-eligible geometry: the device picks the brick engine when
 * |R_0| >= 20 % of the cells (EIK_BRICK_DENSE_PCT), the member list otherwise). */
int eik_last_remedy_engine(void);

/* ---- float32 perf mode (libeik_ifim_f32.so) ----
 * Same semantics and statistics definitions with float32 phi / speed (geometry
 * dtype EIK_F32, tol compared in float32).  The float32 solve is a different
 * rounding of the same algorithm: its phi is checked against the float64 solve
 * at max-rel 1e-5, its counts are its own.  Single device. */
int eik_workspace_size_f32(const eik_geom *g, size_t *bytes);
int eik_ifim_update_step_f32(const eik_geom *g, float *phi, const float *speed, uint8_t *state,
                             const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                             void *workspace, size_t workspace_bytes, int64_t *history, int64_t history_cap,
                             eik_stats *out, void *stream);
int eik_build_remedy_f32(const eik_geom *g, const float *phi, const float *speed, const uint8_t *state, double tol,
                         void *workspace, size_t workspace_bytes, eik_stats *out, void *stream);
int eik_remedy_load_f32(const eik_geom *g, const uint8_t *member, const uint8_t *state, void *workspace,
                        size_t workspace_bytes, int64_t *count, void *stream);
int eik_field_max_diff_f32(const float *a, const float *b, int64_t n, void *scratch, double *out, void *stream);
int eik_chunk_sha256_f32(const void *data, int64_t nbytes, int64_t chunk, uint8_t *digests, void *stream);
int eik_remedy_load_set_f32(const eik_geom *g, const uint8_t *cells, const uint8_t *member, const uint8_t *state,
                            void *workspace, size_t workspace_bytes, int64_t *count, void *stream);
int eik_remedy_export_f32(const eik_geom *g, void *workspace, size_t workspace_bytes, uint8_t *member, void *stream);
int eik_remedy_step_f32(const eik_geom *g, float *phi, const float *speed, const uint8_t *state, double tol,
                        void *workspace, size_t workspace_bytes, eik_stats *out, void *stream);
int eik_ifim_solve_f32(const eik_geom *g, float *phi, const float *speed, uint8_t *state, const int64_t *seed_idx,
                       const double *seed_val, int64_t nseeds, double tol, void *workspace, size_t workspace_bytes,
                       int64_t *history, int64_t history_cap, eik_stats *out, void *stream);
int eik_solve_fixpoint_f32(const eik_geom *g, float *phi, const float *speed, uint8_t *state,
                           const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                           int64_t max_passes, void *workspace, size_t workspace_bytes, eik_stats *out, void *stream);
int eik_solve_fim_f32(const eik_geom *g, float *phi, const float *speed, uint8_t *state, const int64_t *seed_idx,
                      const double *seed_val, int64_t nseeds, double tol, void *workspace, size_t workspace_bytes,
                      eik_stats *out, void *stream);
int eik_max_residual_f32(const eik_geom *g, const float *phi, const float *speed, const uint8_t *state,
                         void *workspace, size_t workspace_bytes, double *out, void *stream);
int eik_local_solve_f32(int kind, const float *a, const float *b, const float *c, const float *f, double dx,
                        double dy, float *out, int64_t n, void *stream);
const char *eik_last_error_f32(void);
const char *eik_version_f32(void);
int eik_last_remedy_engine_f32(void);

#ifdef __cplusplus
}
#endif
#endif /* EIK_IFIM_H */
