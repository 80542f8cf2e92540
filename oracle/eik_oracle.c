/*
 * eik_oracle.c -- CPU restatement of the reference iFIM path (TEST INFRASTRUCTURE).
 *
 * This file is the parity oracle for paper_2106_15869_b200.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it; the product path never does.
 *
 * It restates, operation for operation, the reference package
 * `eikonal` (/root/reference/pkg/src/eikonal, abbreviated E/ below):
 *
 *   upd2u     <- E/_kernels.py:47-58   (_update_uniform_batch, numpy semantics)
 *   upd2a     <- E/_kernels.py:61-88   (_update_aniso_batch)
 *   upd3u     <- E/local_solver.py:91-157 (update_3d_uniform, verified branch walk)
 *   values    <- E/_kernels.py:21-38 + E/ifim.py:48-61 (padded snapshot, axis minima)
 *   orc_ifim_update_step <- E/ifim.py:75-134
 *   orc_build_remedy     <- E/ifim.py:137-161
 *   orc_remedy_step      <- E/ifim.py:164-218
 *   orc_solve_fixpoint   <- E/oracle.py:22-70
 *   orc_solve_fim        <- E/fim.py:62-144 (FIM with per-iteration neighbour checks)
 *
 * 3D generalisation (the reference has no 3D engine): the same
 * engine with six axis neighbours, linear index (k*ny+j)*nx+i, local solver
 * update_3d_uniform, caps 40*(nx+ny+nz) / 20*(nx+ny+nz) / 10*(nx+ny+nz).
 * 2D keeps the reference caps 40*(nx+ny) / 20*(nx+ny) / 10*(nx+ny) exactly.
 *
 * Parity pins: tests/golden/ (generated from the live reference by
 * tests/golden/make_golden.py) -- phi sha256 and every RunStats integer.
 *
 * Build: gcc -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC
 * (no FMA contraction: every op is a separately rounded IEEE op like numpy).
 *
 * threads == 1 reproduces the reference's list orders exactly; threads > 1
 * computes the Jacobi batch in parallel and reconciles with atomic label/member
 * updates.  Because every phase reads an immutable snapshot, set membership and
 * all statistics are identical either way.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_OK 0
#define ORC_EINVAL 1
#define ORC_ECAP 2
#define ORC_ENOMEM 3

/* E/grid.py:21-26 */
enum { ST_FAR = 0, ST_ACTIVE = 1, ST_SOURCE = 2, ST_REMEDY = 3, ST_BLOCKED = 4 };
/* E/ifim.py:32 */
enum { L_FAR = 0, L_ACTIVE = 1, L_CONVERGED = 2 };

static const double SQRT2 = 1.4142135623730951; /* math.sqrt(2.0), E/_kernels.py:18 */
static const double DISC_CLAMP = 1e-12;         /* E/local_solver.py:28 */

typedef struct {
    int64_t nx, ny, nz;
    double dx, dy, dz;
    int32_t ndim;
    int32_t pad;
} orc_geom;

typedef struct {
    int64_t iterations;
    int64_t solver_calls;
    int64_t peak_active;
    int64_t peak_remedy;
    int64_t phi_writes;
    int64_t history_len;
    int64_t remedy_size; /* build: number of flagged cells */
    int64_t converged;   /* update: number of cells labelled CONVERGED */
} orc_stats;

/* numpy.minimum / numpy.maximum on non-NaN inputs (NaN propagates). */
static inline double np_min(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a <= b ? a : b); }
static inline double np_max(double a, double b) { return (isnan(a) || isnan(b)) ? NAN : (a >= b ? a : b); }

/* E/_kernels.py:47-58, element-wise numpy evaluation order. */
double orc_update_2d_uniform(double a, double b, double f, double delta)
{
    double d = delta / f;
    double lo = np_min(a, b);
    double hi = np_max(a, b);
    double one = lo + d;
    double diff = hi - lo;
    int take_two = diff <= SQRT2 * d;
    double disc = 2.0 * d * d - diff * diff;
    double root = 0.5 * (a + b + sqrt(np_max(disc, 0.0)));
    int valid = take_two && (disc >= -DISC_CLAMP * (2.0 * d * d)) && (root >= hi);
    return valid ? root : one;
}

/* E/_kernels.py:61-88 */
double orc_update_2d_aniso(double a, double b, double f, double dx, double dy)
{
    double one_x = a + dx / f;
    double one_y = b + dy / f;
    double dx2 = dx * dx;
    double dy2 = dy * dy;
    double s2 = (dx2 + dy2) / (f * f);
    double s = sqrt(s2);
    double diff = a - b;
    double disc = s2 - diff * diff;
    double root = (a * dy2 + b * dx2 + (dx * dy) * sqrt(np_max(disc, 0.0))) / (dx2 + dy2);
    double drop_larger = (a > b) ? one_y : one_x;
    int valid = isfinite(a) && isfinite(b) && !(diff > s) && !(-diff > s) &&
                (disc >= -DISC_CLAMP * s2) && (root >= a) && (root >= b);
    double out = valid ? root : drop_larger;
    if (isinf(a) && isfinite(b)) out = one_y;
    if (isfinite(a) && isinf(b)) out = one_x;
    if (isinf(a) && isinf(b)) out = INFINITY;
    return out;
}

/* E/local_solver.py:91-157 (scalar Python floats; `x if x > 0 else 0`). */
double orc_update_3d_uniform(double px, double py, double pz, double f, double delta)
{
    double a1 = px, a2 = py, a3 = pz, t;
    /* sorted((px, py, pz)) */
    if (a2 < a1) { t = a1; a1 = a2; a2 = t; }
    if (a3 < a2) { t = a2; a2 = a3; a3 = t; }
    if (a2 < a1) { t = a1; a1 = a2; a2 = t; }
    if (a1 == INFINITY) return INFINITY;
    double d = delta / f;
    int k;
    if (a3 - a1 < delta) k = 3;
    else if (a2 - a1 < delta) k = 2;
    else k = 1;
    unsigned visited = 0;
    for (;;) {
        visited |= 1u << k;
        if (k == 3) {
            double b2 = a2 - a1;
            double b3 = a3 - a1;
            double s = b2 + b3;
            double disc = s * s - 3.0 * (b2 * b2 + b3 * b3 - d * d);
            if (disc < -DISC_CLAMP * (3.0 * d * d)) { k = 2; continue; }
            double root = a1 + (s + sqrt(disc > 0.0 ? disc : 0.0)) / 3.0;
            if (root >= a3 || (visited & (1u << 2))) return root;
            k = 2;
        } else if (k == 2) {
            if (a2 == INFINITY) { k = 1; continue; }
            double diff = a2 - a1;
            double disc = 2.0 * d * d - diff * diff;
            if (disc < -DISC_CLAMP * (2.0 * d * d)) { k = 1; continue; }
            double root = 0.5 * (a1 + a2 + sqrt(disc > 0.0 ? disc : 0.0));
            if (root < a2 && !(visited & (1u << 1))) { k = 1; continue; }
            if (root > a3 && !(visited & (1u << 3))) { k = 3; continue; }
            return root;
        } else {
            double root = a1 + d;
            if (root > a2 && !(visited & (1u << 2))) { k = 2; continue; }
            return root;
        }
    }
}

/* ---- grid helpers ------------------------------------------------------ */

static inline int64_t ncells(const orc_geom *g) { return g->nx * g->ny * (g->ndim == 3 ? g->nz : 1); }

/* Snapshot value of cell c through the +inf border (E/_kernels.py:21-38). */
static inline double cell_value(const orc_geom *g, const double *phi, const double *speed, int64_t c)
{
    const int64_t nx = g->nx, ny = g->ny;
    int64_t i = c % nx;
    int64_t r = c / nx;
    int64_t j = r % ny;
    double w = i > 0 ? phi[c - 1] : INFINITY;
    double e = i < nx - 1 ? phi[c + 1] : INFINITY;
    double s = j > 0 ? phi[c - nx] : INFINITY;
    double n = j < ny - 1 ? phi[c + nx] : INFINITY;
    double xmin = np_min(w, e);
    double ymin = np_min(s, n);
    if (g->ndim == 3) {
        int64_t k = r / ny;
        int64_t plane = nx * ny;
        double dn = k > 0 ? phi[c - plane] : INFINITY;
        double up = k < g->nz - 1 ? phi[c + plane] : INFINITY;
        double zmin = np_min(dn, up);
        return orc_update_3d_uniform(xmin, ymin, zmin, speed[c], g->dx);
    }
    if (g->dx == g->dy) return orc_update_2d_uniform(xmin, ymin, speed[c], g->dx); /* E/_kernels.py:41-44 */
    return orc_update_2d_aniso(xmin, ymin, speed[c], g->dx, g->dy);
}

/* Axis neighbours in the reference's W, E, S, N (, D, U) order (E/ifim.py:35-45). */
static inline int neighbors(const orc_geom *g, int64_t c, int64_t out[6])
{
    const int64_t nx = g->nx, ny = g->ny;
    int64_t i = c % nx, r = c / nx, j = r % ny;
    int m = 0;
    if (i > 0) out[m++] = c - 1;
    if (i < nx - 1) out[m++] = c + 1;
    if (j > 0) out[m++] = c - nx;
    if (j < ny - 1) out[m++] = c + nx;
    if (g->ndim == 3) {
        int64_t k = r / ny, plane = nx * ny;
        if (k > 0) out[m++] = c - plane;
        if (k < g->nz - 1) out[m++] = c + plane;
    }
    return m;
}

static int64_t cap_of(const orc_geom *g, int64_t mult)
{
    int64_t s = g->nx + g->ny + (g->ndim == 3 ? g->nz : 0);
    return mult * s;
}

static void set_threads(int threads)
{
#ifdef _OPENMP
    if (threads > 0) omp_set_num_threads(threads);
#else
    (void)threads;
#endif
}

/* Jacobi batch: every value reads the same snapshot (E/ifim.py:113-114). */
static void batch_values(const orc_geom *g, const double *phi, const double *speed,
                         const int64_t *cells, int64_t m, double *out, int threads)
{
    if (threads == 1) {
        for (int64_t p = 0; p < m; ++p) out[p] = cell_value(g, phi, speed, cells[p]);
        return;
    }
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < m; ++p) out[p] = cell_value(g, phi, speed, cells[p]);
}

/* ---- apply_boundary (E/grid.py:199-215); validation done by the caller -- */
int orc_apply_boundary(const orc_geom *g, double *phi, uint8_t *state,
                       const int64_t *seed_idx, const double *seed_val, int64_t nseeds)
{
    int64_t n = ncells(g);
    if (nseeds <= 0) return ORC_EINVAL;
    for (int64_t s = 0; s < nseeds; ++s) {
        if (seed_idx[s] < 0 || seed_idx[s] >= n) return ORC_EINVAL;
        if (state[seed_idx[s]] == ST_BLOCKED) return ORC_EINVAL;
    }
    for (int64_t s = 0; s < nseeds; ++s) {
        phi[seed_idx[s]] = seed_val[s];
        state[seed_idx[s]] = ST_SOURCE;
    }
    return ORC_OK;
}

/* ---- update step: E/ifim.py:75-134 ------------------------------------ */
int orc_ifim_update_step(const orc_geom *g, double *phi, const double *speed, uint8_t *state,
                         const int64_t *seed_idx, const double *seed_val, int64_t nseeds,
                         double tol, int64_t *history, int64_t history_cap,
                         orc_stats *st, int threads)
{
    if (!(tol > 0)) return ORC_EINVAL;
    int rc = orc_apply_boundary(g, phi, state, seed_idx, seed_val, nseeds);
    if (rc) return rc;
    set_threads(threads);
    const int64_t n = ncells(g);
    memset(st, 0, sizeof(*st));

    uint8_t *label = (uint8_t *)calloc((size_t)n, 1);
    int64_t *active = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double *values = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!label || !active || !next || !values) { free(label); free(active); free(next); free(values); return ORC_ENOMEM; }

    /* E/ifim.py:97-102: initial Active = free FAR neighbours of seeds, in bc order. */
    int64_t na = 0, nb[6];
    for (int64_t s = 0; s < nseeds; ++s) {
        int m = neighbors(g, seed_idx[s], nb);
        for (int q = 0; q < m; ++q) {
            int64_t c = nb[q];
            if (state[c] != ST_BLOCKED && state[c] != ST_SOURCE && label[c] == L_FAR) {
                label[c] = L_ACTIVE;
                active[na++] = c;
            }
        }
    }
    st->peak_active = na;
    const int64_t cap = cap_of(g, 40);
    rc = ORC_OK;
    while (na > 0) {
        st->iterations += 1;
        if (st->iterations > cap) { rc = ORC_ECAP; break; }
        if (st->history_len < history_cap) history[st->history_len] = na;
        st->history_len += 1;
        batch_values(g, phi, speed, active, na, values, threads);
        st->solver_calls += na;

        int64_t nn = 0;
        if (threads == 1) {
            for (int64_t p = 0; p < na; ++p) {
                int64_t c = active[p];
                double v = values[p], old = phi[c];
                if (v == old || fabs(v - old) <= tol) {
                    label[c] = L_CONVERGED;
                    st->converged += 1;
                    int m = neighbors(g, c, nb);
                    for (int q = 0; q < m; ++q) {
                        int64_t e = nb[q];
                        if (phi[e] == INFINITY && state[e] != ST_BLOCKED && label[e] == L_FAR) {
                            label[e] = L_ACTIVE;
                            next[nn++] = e;
                        }
                    }
                } else {
                    phi[c] = v;
                    st->phi_writes += 1;
                    next[nn++] = c;
                }
            }
        } else {
            int64_t conv = 0, writes = 0;
#pragma omp parallel reduction(+ : conv, writes)
            {
                int64_t lnb[6];
#pragma omp for schedule(static)
                for (int64_t p = 0; p < na; ++p) {
                    int64_t c = active[p];
                    double v = values[p], old = phi[c];
                    if (v == old || fabs(v - old) <= tol) {
                        __atomic_store_n(&label[c], (uint8_t)L_CONVERGED, __ATOMIC_RELAXED);
                        conv += 1;
                        int m = neighbors(g, c, lnb);
                        for (int q = 0; q < m; ++q) {
                            int64_t e = lnb[q];
                            /* label first: only ACTIVE cells are written, FAR cells never are */
                            uint8_t expect = L_FAR;
                            if (__atomic_load_n(&label[e], __ATOMIC_RELAXED) != L_FAR) continue;
                            if (!(phi[e] == INFINITY) || state[e] == ST_BLOCKED) continue;
                            if (__atomic_compare_exchange_n(&label[e], &expect, (uint8_t)L_ACTIVE, 0,
                                                            __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
                                int64_t slot = __atomic_fetch_add(&nn, 1, __ATOMIC_RELAXED);
                                next[slot] = e;
                            }
                        }
                    } else {
                        phi[c] = v;
                        writes += 1;
                        int64_t slot = __atomic_fetch_add(&nn, 1, __ATOMIC_RELAXED);
                        next[slot] = c;
                    }
                }
            }
            st->converged += conv;
            st->phi_writes += writes;
        }
        int64_t *t = active; active = next; next = t;
        na = nn;
        if (na > st->peak_active) st->peak_active = na;
    }
    free(label); free(active); free(next); free(values);
    return rc;
}

/* ---- build_remedy_set: E/ifim.py:137-161 ------------------------------- */
int orc_build_remedy(const orc_geom *g, const double *phi, const double *speed, const uint8_t *state,
                     double tol, uint8_t *member, orc_stats *st, int threads)
{
    if (!(tol > 0)) return ORC_EINVAL;
    set_threads(threads);
    const int64_t n = ncells(g);
    memset(st, 0, sizeof(*st));
    int64_t calls = 0, flagged = 0;
#pragma omp parallel for schedule(static) reduction(+ : calls, flagged) if (threads != 1)
    for (int64_t c = 0; c < n; ++c) {
        member[c] = 0;
        if (state[c] == ST_BLOCKED || state[c] == ST_SOURCE) continue;
        calls += 1;
        double v = cell_value(g, phi, speed, c);
        /* |v - phi| > tol; NaN (inf - inf) compares false: E/ifim.py:156-157 */
        if (fabs(v - phi[c]) > tol) { member[c] = 1; flagged += 1; }
    }
    st->solver_calls = calls;
    st->remedy_size = flagged;
    return ORC_OK;
}

/* ---- remedy step: E/ifim.py:164-218 ------------------------------------ */
int orc_remedy_step(const orc_geom *g, double *phi, const double *speed, const uint8_t *state,
                    uint8_t *member, double tol, int64_t *history, int64_t history_cap,
                    orc_stats *st, int threads)
{
    if (!(tol > 0)) return ORC_EINVAL;
    set_threads(threads);
    const int64_t n = ncells(g);
    memset(st, 0, sizeof(*st));
    int64_t *cells = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *next = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    int64_t *dec = (int64_t *)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    double *values = (double *)malloc(sizeof(double) * (size_t)(n > 0 ? n : 1));
    if (!cells || !next || !dec || !values) { free(cells); free(next); free(dec); free(values); return ORC_ENOMEM; }
    int64_t nr = 0;
    for (int64_t c = 0; c < n; ++c) if (member[c]) cells[nr++] = c; /* ascending, like cells[moved] */
    st->peak_remedy = nr;
    const int64_t cap = cap_of(g, 20);
    int rc = ORC_OK;
    int64_t nb[6];
    while (nr > 0) {
        st->iterations += 1;
        if (st->iterations > cap) { rc = ORC_ECAP; break; }
        if (st->history_len < history_cap) history[st->history_len] = nr;
        st->history_len += 1;
        batch_values(g, phi, speed, cells, nr, values, threads);
        st->solver_calls += nr;
        int64_t nn = 0, nd = 0;
        if (threads == 1) {
            /* decide every stay/drop first (E/ifim.py:195-208) */
            for (int64_t p = 0; p < nr; ++p) {
                int64_t c = cells[p];
                double v = values[p];
                if (v < phi[c] - tol) {
                    phi[c] = v;
                    dec[nd++] = c;
                    next[nn++] = c;
                } else {
                    member[c] = 0;
                }
            }
            /* then enqueue free non-member neighbours of decreased cells (:209-213) */
            for (int64_t p = 0; p < nd; ++p) {
                int m = neighbors(g, dec[p], nb);
                for (int q = 0; q < m; ++q) {
                    int64_t e = nb[q];
                    if (!member[e] && state[e] != ST_BLOCKED && state[e] != ST_SOURCE) {
                        member[e] = 1;
                        next[nn++] = e;
                    }
                }
            }
        } else {
#pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < nr; ++p) {
                int64_t c = cells[p];
                double v = values[p];
                if (v < phi[c] - tol) {
                    phi[c] = v;
                    int64_t slot = __atomic_fetch_add(&nd, 1, __ATOMIC_RELAXED);
                    dec[slot] = c;
                } else {
                    member[c] = 0;
                }
            }
            memcpy(next, dec, sizeof(int64_t) * (size_t)nd);
            nn = nd;
#pragma omp parallel for schedule(static)
            for (int64_t p = 0; p < nd; ++p) {
                int64_t lnb[6];
                int m = neighbors(g, dec[p], lnb);
                for (int q = 0; q < m; ++q) {
                    int64_t e = lnb[q];
                    if (state[e] == ST_BLOCKED || state[e] == ST_SOURCE) continue;
                    uint8_t expect = 0;
                    if (__atomic_load_n(&member[e], __ATOMIC_RELAXED)) continue;
                    if (__atomic_compare_exchange_n(&member[e], &expect, (uint8_t)1, 0,
                                                    __ATOMIC_RELAXED, __ATOMIC_RELAXED)) {
                        int64_t slot = __atomic_fetch_add(&nn, 1, __ATOMIC_RELAXED);
                        next[slot] = e;
                    }
                }
            }
        }
        st->phi_writes += nd;
        int64_t *t = cells; cells = next; next = t;
        nr = nn;
        if (nr > st->peak_remedy) st->peak_remedy = nr;
    }
    if (rc == ORC_OK) memset(member, 0, (size_t)n); /* drained */
    free(cells); free(next); free(dec); free(values);
    return rc;
}

/* ---- solve_ifim: E/ifim.py:221-235 ------------------------------------- */
int orc_solve_ifim(const orc_geom *g, double *phi, const double *speed, uint8_t *state,
                   const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                   int64_t *history, int64_t history_cap, orc_stats *out, orc_stats *phases,
                   int threads)
{
    orc_stats up, bd, rm;
    int rc = orc_ifim_update_step(g, phi, speed, state, seed_idx, seed_val, nseeds, tol, history,
                                  history_cap, &up, threads);
    if (rc) return rc;
    const int64_t n = ncells(g);
    uint8_t *member = (uint8_t *)malloc((size_t)(n > 0 ? n : 1));
    if (!member) return ORC_ENOMEM;
    rc = orc_build_remedy(g, phi, speed, state, tol, member, &bd, threads);
    if (!rc) rc = orc_remedy_step(g, phi, speed, state, member, tol, NULL, 0, &rm, threads);
    free(member);
    if (rc) return rc;
    memset(out, 0, sizeof(*out));
    out->iterations = up.iterations + rm.iterations;
    out->solver_calls = up.solver_calls + bd.solver_calls + rm.solver_calls;
    out->peak_active = up.peak_active;
    out->peak_remedy = rm.peak_remedy;
    out->phi_writes = up.phi_writes + rm.phi_writes;
    out->history_len = up.history_len;
    out->remedy_size = bd.remedy_size;
    out->converged = up.converged;
    if (phases) { phases[0] = up; phases[1] = bd; phases[2] = rm; }
    return ORC_OK;
}

/* ---- solve_fixpoint: E/oracle.py:22-70 --------------------------------- */
int orc_solve_fixpoint(const orc_geom *g, double *phi, const double *speed, uint8_t *state,
                       const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol,
                       int64_t max_passes, orc_stats *st, int threads)
{
    if (!(tol > 0)) return ORC_EINVAL;
    int rc = orc_apply_boundary(g, phi, state, seed_idx, seed_val, nseeds);
    if (rc) return rc;
    set_threads(threads);
    const int64_t n = ncells(g);
    memset(st, 0, sizeof(*st));
    int64_t nf = 0;
    for (int64_t c = 0; c < n; ++c) if (state[c] != ST_SOURCE && state[c] != ST_BLOCKED) nf++;
    int64_t *cells = (int64_t *)malloc(sizeof(int64_t) * (size_t)(nf > 0 ? nf : 1));
    double *cand = (double *)malloc(sizeof(double) * (size_t)(nf > 0 ? nf : 1));
    if (!cells || !cand) { free(cells); free(cand); return ORC_ENOMEM; }
    nf = 0;
    for (int64_t c = 0; c < n; ++c) if (state[c] != ST_SOURCE && state[c] != ST_BLOCKED) cells[nf++] = c;
    const int64_t cap = max_passes > 0 ? max_passes : cap_of(g, 10);
    rc = ORC_OK;
    for (;;) {
        batch_values(g, phi, speed, cells, nf, cand, threads);
        st->solver_calls += nf;
        st->iterations += 1;
        int any = 0;
        double max_change = 0.0;
        for (int64_t p = 0; p < nf; ++p) {
            double old = phi[cells[p]];
            double nw = np_min(old, cand[p]);
            if (nw < old) {
                any = 1;
                double ch = old - nw;
                if (ch > max_change || isnan(max_change)) max_change = ch;
            }
            phi[cells[p]] = nw;
        }
        if (!any) break;
        if (max_change < tol) break;
        if (st->iterations >= cap) { rc = ORC_ECAP; break; }
    }
    free(cells); free(cand);
    return rc;
}

/* Batch entry points used by the local-solver parity tests (per-element spacing). */
/* ---- solve_fim: E/fim.py:62-144 (serial, the reference's list orders) ----
 * Phase one: Jacobi values of the active list; settle (|v-old| <= tol) or write
 * and survive (:95-108).  Phase two: every cell active this iteration examines
 * its neighbours: skip fixed / ACTIVE, activate +inf ones, queue the others as
 * checks -- one counted call per examination (:110-124).  Checks: Jacobi values
 * from the post-phase-one field; a non-active check cell whose value drops by
 * more than tol is written and re-activated (:126-138). */
enum { F_FAR = 0, F_ACTIVE = 1, F_SETTLED = 2 }; /* E/fim.py:29 */

int orc_solve_fim(const orc_geom *g, double *phi, const double *speed, uint8_t *state,
                  const int64_t *seed_idx, const double *seed_val, int64_t nseeds, double tol, orc_stats *st)
{
    if (!(tol > 0)) return ORC_EINVAL;
    int rc = orc_apply_boundary(g, phi, state, seed_idx, seed_val, nseeds);
    if (rc) return rc;
    const int64_t n = ncells(g);
    memset(st, 0, sizeof(*st));
    const size_t cap_n = (size_t)(n > 0 ? n : 1);
    uint8_t *label = (uint8_t *)calloc(cap_n, 1);
    int64_t *active = (int64_t *)malloc(sizeof(int64_t) * cap_n);
    int64_t *surv = (int64_t *)malloc(sizeof(int64_t) * cap_n);
    int64_t *check = (int64_t *)malloc(sizeof(int64_t) * cap_n * 6);
    double *values = (double *)malloc(sizeof(double) * cap_n * 6);
    if (!label || !active || !surv || !check || !values) {
        free(label); free(active); free(surv); free(check); free(values);
        return ORC_ENOMEM;
    }
    int64_t na = 0, nb[6];
    for (int64_t s = 0; s < nseeds; ++s) { /* :78-84 */
        int m = neighbors(g, seed_idx[s], nb);
        for (int q = 0; q < m; ++q) {
            int64_t c = nb[q];
            if (state[c] != ST_BLOCKED && state[c] != ST_SOURCE && label[c] == F_FAR) {
                label[c] = F_ACTIVE;
                active[na++] = c;
            }
        }
    }
    st->peak_active = na;
    const int64_t cap = cap_of(g, 40);
    rc = ORC_OK;
    while (na > 0) {
        st->iterations += 1;
        if (st->iterations > cap) { rc = ORC_ECAP; break; }
        batch_values(g, phi, speed, active, na, values, 1);
        st->solver_calls += na;
        int64_t ns = 0;
        for (int64_t p = 0; p < na; ++p) {
            int64_t c = active[p];
            double v = values[p], old = phi[c];
            if (v == old || fabs(v - old) <= tol) {
                label[c] = F_SETTLED;
            } else {
                phi[c] = v;
                st->phi_writes += 1;
                surv[ns++] = c;
            }
        }
        int64_t nc = 0;
        for (int64_t p = 0; p < na; ++p) {
            int m = neighbors(g, active[p], nb);
            for (int q = 0; q < m; ++q) {
                int64_t c = nb[q];
                if (state[c] == ST_BLOCKED || state[c] == ST_SOURCE || label[c] == F_ACTIVE) continue;
                if (phi[c] == INFINITY) {
                    label[c] = F_ACTIVE;
                    surv[ns++] = c;
                } else {
                    check[nc++] = c;
                }
            }
        }
        int64_t *t = active; active = surv; surv = t;
        na = ns;
        if (nc > 0) {
            batch_values(g, phi, speed, check, nc, values, 1);
            st->solver_calls += nc;
            for (int64_t p = 0; p < nc; ++p) {
                int64_t c = check[p];
                if (label[c] == F_ACTIVE) continue;
                double v = values[p];
                if (v < phi[c] - tol) {
                    phi[c] = v;
                    st->phi_writes += 1;
                    label[c] = F_ACTIVE;
                    active[na++] = c;
                }
            }
        }
        if (na > st->peak_active) st->peak_active = na;
    }
    free(label); free(active); free(surv); free(check); free(values);
    return rc;
}

void orc_update_2d_uniform_batch(const double *a, const double *b, const double *f, const double *delta,
                                 double *out, int64_t n)
{
    for (int64_t p = 0; p < n; ++p) out[p] = orc_update_2d_uniform(a[p], b[p], f[p], delta[p]);
}
void orc_update_2d_aniso_batch(const double *a, const double *b, const double *f, const double *dx,
                               const double *dy, double *out, int64_t n)
{
    for (int64_t p = 0; p < n; ++p) out[p] = orc_update_2d_aniso(a[p], b[p], f[p], dx[p], dy[p]);
}
void orc_update_3d_uniform_batch(const double *a, const double *b, const double *c, const double *f,
                                 const double *delta, double *out, int64_t n)
{
    for (int64_t p = 0; p < n; ++p) out[p] = orc_update_3d_uniform(a[p], b[p], c[p], f[p], delta[p]);
}
