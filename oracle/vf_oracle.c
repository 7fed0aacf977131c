/*
 * vf_oracle.c -- CPU restatement of the geometry-embedding hot path.
 * TEST INFRASTRUCTURE ONLY (see vf_oracle.h for scope, citations and the
 * parity status).  Every stage is written as the literal sequential / per-cell
 * algorithm of the SPEC / PAPER text; OpenMP only splits independent outer
 * loops (faces, blocks, x-chains), so results never depend on thread count.
 *
 * Compile with -ffp-contract=off: the reference predicate is compiled by numba
 * without FMA contraction (SURVEY finding 7), and this file must evaluate the
 * same IEEE double operations in the same association.
 */
#include "vf_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <time.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORC_ABI 1

/* D3Q27 order of lattice.py:19-39 (rest first, antiparallel pairs (2k-1,2k)) */
static const int C27[27][3] = {
    {0, 0, 0},   {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},   {0, -1, 0},
    {0, 0, 1},   {0, 0, -1},  {1, 1, 0},   {-1, -1, 0}, {1, 0, 1},
    {-1, 0, -1}, {1, 0, -1},  {-1, 0, 1},  {1, -1, 0},  {-1, 1, 0},
    {0, 1, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},  {1, 1, 1},
    {-1, -1, -1}, {1, 1, -1}, {-1, -1, 1}, {1, -1, 1},  {-1, 1, -1},
    {1, -1, -1}, {-1, 1, 1}};

static int slot_of(int dx, int dy, int dz) {
    for (int q = 0; q < 27; ++q)
        if (C27[q][0] == dx && C27[q][1] == dy && C27[q][2] == dz) return q;
    return -1;
}

int orc_abi_version(void) { return ORC_ABI; }

void orc_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int orc_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------------ */
/* SAT predicate: geometry.py:441-500, same operations and association.      */

static inline double mn(double a, double b) { return a < b ? a : b; }
static inline double mx_(double a, double b) { return a > b ? a : b; }

/* geometry.py:441-454 */
static inline int plane_cuts_box(double v1x, double v1y, double v1z,
                                 double v2x, double v2y, double v2z,
                                 double v3x, double v3y, double v3z,
                                 double mx, double my, double mz,
                                 double Mx, double My, double Mz) {
    double nx = (v2y - v1y) * (v3z - v1z) - (v2z - v1z) * (v3y - v1y);
    double ny = (v2z - v1z) * (v3x - v1x) - (v2x - v1x) * (v3z - v1z);
    double nz = (v2x - v1x) * (v3y - v1y) - (v2y - v1y) * (v3x - v1x);
    double cx = (nx > 0.0) ? (Mx - mx) : 0.0;
    double cy = (ny > 0.0) ? (My - my) : 0.0;
    double cz = (nz > 0.0) ? (Mz - mz) : 0.0;
    double d = nx * mx + ny * my + nz * mz;
    double d1 = nx * (cx - v1x) + ny * (cy - v1y) + nz * (cz - v1z);
    double d2 = (nx * ((Mx - mx - cx) - v1x) + ny * ((My - my - cy) - v1y)
                 + nz * ((Mz - mz - cz) - v1z));
    return (d + d1) * (d + d2) <= 0.0;
}

/* geometry.py:457-481; returns 1 when the axis separates */
static inline int axis_gap_2d(int axis, double v1x, double v1y, double v2x,
                              double v2y, double v3x, double v3y, double rmx,
                              double rmy, double rMx, double rMy) {
    double ex, ey;
    if (axis == 0) { ex = 1.0; ey = 0.0; }
    else if (axis == 1) { ex = 0.0; ey = 1.0; }
    else if (axis == 2) { ex = v2y - v1y; ey = v1x - v2x; }
    else if (axis == 3) { ex = v3y - v2y; ey = v2x - v3x; }
    else { ex = v1y - v3y; ey = v3x - v1x; }
    double t1 = v1x * ex + v1y * ey;
    double t2 = v2x * ex + v2y * ey;
    double t3 = v3x * ex + v3y * ey;
    double tmin = mn(mn(t1, t2), t3);
    double tmax = mx_(mx_(t1, t2), t3);
    double r1 = rmx * ex + rmy * ey;
    double r2 = rMx * ex + rmy * ey;
    double r3 = rmx * ex + rMy * ey;
    double r4 = rMx * ex + rMy * ey;
    double rmin = mn(mn(r1, r2), mn(r3, r4));
    double rmax = mx_(mx_(r1, r2), mx_(r3, r4));
    return (tmax < rmin) || (rmax < tmin);
}

/* Algorithmic operation counters (the roofline's ops come
 * from the oracle's branch path).  Per thread, flushed per stage by
 * orc_ops_flush: SAT calls, SAT FP64 ops executed (54 for the plane-cut test
 * + 34 per axis-gap test evaluated, geometry.py:441-500) and the stage's
 * other FP64 ops (distance evaluations). */
static _Thread_local uint64_t t_sat_calls, t_sat_ops, t_eval_ops;
enum { ORC_ST_IND = 0, ORC_ST_PAIRS, ORC_ST_VOX, ORC_ST_MD, ORC_ST_LINKS, ORC_NST };
static uint64_t g_ops[ORC_NST][3];

static void orc_ops_flush(int stage) {
#pragma omp parallel
    {
#pragma omp atomic
        g_ops[stage][0] += t_sat_calls;
#pragma omp atomic
        g_ops[stage][1] += t_sat_ops;
#pragma omp atomic
        g_ops[stage][2] += t_eval_ops;
        t_sat_calls = t_sat_ops = t_eval_ops = 0;
    }
    /* the calling thread too (outside a team it is thread 0 of the region) */
}

/* counters of the stages since the last call, then reset:
 * out[5][3] = {indicators 1D, bin pairs, voxelize, MD bins, link lengths} x
 * {SAT calls, SAT ops, other ops} */
void orc_op_counters(uint64_t *out) {
    memcpy(out, g_ops, sizeof(g_ops));
    memset(g_ops, 0, sizeof(g_ops));
}

/* geometry.py:484-500 */
static inline int sat3(const double *v, double mx, double my, double mz,
                       double Mx, double My, double Mz) {
    const double v1x = v[0], v1y = v[1], v1z = v[2];
    const double v2x = v[3], v2y = v[4], v2z = v[5];
    const double v3x = v[6], v3y = v[7], v3z = v[8];
    ++t_sat_calls;
    t_sat_ops += 54;
    if (!plane_cuts_box(v1x, v1y, v1z, v2x, v2y, v2z, v3x, v3y, v3z, mx, my,
                        mz, Mx, My, Mz))
        return 0;
    for (int k = 0; k < 5; ++k) {
        t_sat_ops += 34;
        if (axis_gap_2d(k, v1x, v1y, v2x, v2y, v3x, v3y, mx, my, Mx, My))
            return 0;
    }
    for (int k = 0; k < 5; ++k) {
        t_sat_ops += 34;
        if (axis_gap_2d(k, v1y, v1z, v2y, v2z, v3y, v3z, my, mz, My, Mz))
            return 0;
    }
    for (int k = 0; k < 5; ++k) {
        t_sat_ops += 34;
        if (axis_gap_2d(k, v1z, v1x, v2z, v2x, v3z, v3x, mz, mx, Mz, Mx))
            return 0;
    }
    return 1;
}

int orc_sat(const double *tri, const double *box) {
    return sat3(tri, box[0], box[1], box[2], box[3], box[4], box[5]);
}

void orc_sat_batch(const double *tri, const double *box, int64_t n,
                   uint8_t *out) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) out[i] = (uint8_t)orc_sat(tri + 9 * i, box + 6 * i);
}

/* ------------------------------------------------------------------------ */
/* shared pins                                           */

static inline double level_dx(const orc_config *c, int L) { return ldexp(c->dx0, -L); }
static inline int cells_axis(const orc_config *c, int d, int L) { return (4 * c->nb[d]) << L; }
static inline int bins_axis(const orc_config *c, int d, int L) { return c->nb[d] << L; }
/* A2: cell / lattice-node centre, one rounding */
static inline double node_c(int gi, double dx) { return ((double)gi + 0.5) * dx; }

/* floor-range of lattice indices [floor(lo/s), floor(hi/s)] widened by w and
 * clamped to [0, n-1].  Returns 0 when empty.  Only a superset matters
 * (rows outside are rejected by the SAT's box axes). */
static int index_range(double lo, double hi, double s, int w, int n, int *a, int *b) {
    double fa = floor(lo / s) - w, fb = floor(hi / s) + w;
    if (fa < 0) fa = 0;
    if (fb > n - 1) fb = n - 1;
    if (fa > fb) return 0;
    *a = (int)fa;
    *b = (int)fb;
    return 1;
}

static inline void face_bounds(const double *v, double *lo, double *hi) {
    for (int d = 0; d < 3; ++d) {
        lo[d] = mn(mn(v[d], v[3 + d]), v[6 + d]);
        hi[d] = mx_(mx_(v[d], v[3 + d]), v[6 + d]);
    }
}

/* A7/A17: plane-distance numerator, fixed association */
static inline double plane_num(const double *v, const double *n, double x,
                               double y, double z) {
    return (v[0] - x) * n[0] + ((v[1] - y) * n[1] + (v[2] - z) * n[2]);
}

/* ------------------------------------------------------------------------ */
/* Alg. 1 ray indicators (pin A6)         */

static int indicator_1d(const double *v, const double *n, const orc_config *c, int L) {
    if (fabs(n[0]) < c->eps_parallel) return 0;
    const double dx = level_dx(c, L), eps = c->eps_slab;
    double lo[3], hi[3];
    face_bounds(v, lo, hi);
    int j0, j1, k0, k1;
    if (!index_range(lo[1], hi[1], dx, 0, cells_axis(c, 1, L), &j0, &j1)) return 0;
    if (!index_range(lo[2], hi[2], dx, 0, cells_axis(c, 2, L), &k0, &k1)) return 0;
    for (int k = k0; k <= k1; ++k) {
        const double z = node_c(k, dx);
        for (int j = j0; j <= j1; ++j) {
            const double y = node_c(j, dx);
            if (sat3(v, 0.0, y - eps, z - eps, c->len[0], y + eps, z + eps)) return 1;
        }
    }
    return 0;
}

static int indicator_md(const double *v, const double *n, const orc_config *c, int L) {
    const double dx = level_dx(c, L), eps = c->eps_slab;
    double lo[3], hi[3];
    face_bounds(v, lo, hi);
    int a[3], b[3];
    for (int d = 0; d < 3; ++d)
        if (!index_range(lo[d], hi[d], dx, 1, cells_axis(c, d, L), &a[d], &b[d])) return 0;
    for (int q = 1; q < 27; q += 2) {
        const double c0 = C27[q][0], c1 = C27[q][1], c2 = C27[q][2];
        const double cn = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
        const double den = (c0 * n[0] + c1 * n[1]) + c2 * n[2];
        if (fabs(den) < c->eps_parallel * cn) continue;
        for (int k = a[2]; k <= b[2]; ++k) {
            const double z = node_c(k, dx);
            for (int j = a[1]; j <= b[1]; ++j) {
                const double y = node_c(j, dx);
                for (int i = a[0]; i <= b[0]; ++i) {
                    const double x = node_c(i, dx);
                    const double d = plane_num(v, n, x, y, z) / den;
                    const double xi = x + d * c0, yi = y + d * c1, zi = z + d * c2;
                    if (sat3(v, xi - eps, yi - eps, zi - eps, xi + eps, yi + eps, zi + eps))
                        return 1;
                }
            }
        }
    }
    return 0;
}

int orc_ray_indicators(const double *fc, const double *nrm, int64_t F,
                       const orc_config *cfg, int L, int mode, uint8_t *out) {
    if (!fc || !nrm || !cfg || !out || F < 0 || L < 0) return ORC_EARG;
#pragma omp parallel for schedule(dynamic, 1024)
    for (int64_t f = 0; f < F; ++f)
        out[f] = (uint8_t)(mode == 0 ? indicator_1d(fc + 9 * f, nrm + 3 * f, cfg, L)
                                     : indicator_md(fc + 9 * f, nrm + 3 * f, cfg, L));
    return ORC_OK;
}

/* ascending original ids of faces with indicator 1 */
int64_t orc_compact(const uint8_t *ind, int64_t F, int32_t *map) {
    int64_t m = 0;
    for (int64_t f = 0; f < F; ++f)
        if (ind[f]) map[m++] = (int32_t)f;
    return m;
}

/* ------------------------------------------------------------------------ */
/* Alg. 2 bin pairs (pin A5)              */

static int face_pairs(const double *v, const orc_config *c, int L, int nlim,
                      int32_t *bins_out) {
    double lo[3], hi[3];
    face_bounds(v, lo, hi);
    for (int d = 0; d < 3; ++d)
        if (hi[d] < 0.0 || lo[d] > c->len[d]) return 0; /* outside domain */
    const double dx = level_dx(c, L), h = 4.0 * dx;
    int B[3], a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        B[d] = bins_axis(c, d, L);
        const double s = (double)B[d] / c->len[d];
        double fa = floor(lo[d] * s) - 1, fb = floor(hi[d] * s) + 1;
        if (fa < 0) fa = 0;
        if (fb > B[d] - 1) fb = B[d] - 1;
        if (fa > fb) return 0;
        a[d] = (int)fa;
        b[d] = (int)fb;
    }
    int cnt = 0;
    for (int bk = a[2]; bk <= b[2]; ++bk)
        for (int bj = a[1]; bj <= b[1]; ++bj)
            for (int bi = a[0]; bi <= b[0]; ++bi) {
                const double mx = (double)bi * h - dx, Mx = (double)(bi + 1) * h + dx;
                const double my = (double)bj * h - dx, My = (double)(bj + 1) * h + dx;
                const double mz = (double)bk * h - dx, Mz = (double)(bk + 1) * h + dx;
                if (sat3(v, mx, my, mz, Mx, My, Mz)) {
                    if (cnt >= nlim) return -1; /* N_lim cap violated */
                    bins_out[cnt++] = bi + B[0] * (bj + B[1] * bk);
                }
            }
    return cnt;
}

int orc_bin_pairs(const double *fc, int64_t F, const int32_t *map, int64_t nmap,
                  const orc_config *cfg, int L, int32_t *pair_bin,
                  int32_t *pair_face, int64_t cap, int64_t *n_pairs) {
    (void)F;
    const int nlim = (2 + cfg->n_spec) * (2 + cfg->n_spec) * (2 + cfg->n_spec);
    int32_t *tmp = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nmap > 0 ? nmap : 1) * nlim);
    int32_t *cnt = (int32_t *)malloc(sizeof(int32_t) * (size_t)(nmap > 0 ? nmap : 1));
    int bad = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : bad)
    for (int64_t m = 0; m < nmap; ++m) {
        const int32_t f = map ? map[m] : (int32_t)m;
        int r = face_pairs(fc + 9 * (int64_t)f, cfg, L, nlim, tmp + m * nlim);
        if (r < 0) { bad = 1; r = 0; }
        cnt[m] = r;
    }
    int64_t p = 0;
    int over = 0;
    for (int64_t m = 0; m < nmap && !bad; ++m) {
        const int32_t f = map ? map[m] : (int32_t)m;
        for (int k = 0; k < cnt[m]; ++k) {
            if (p >= cap) { over = 1; break; }
            pair_bin[p] = tmp[m * nlim + k];
            pair_face[p] = f;
            ++p;
        }
        if (over) break;
    }
    free(tmp);
    free(cnt);
    *n_pairs = p;
    if (bad) return ORC_ECAP_NLIM;
    if (over) return ORC_ECAPACITY;
    return ORC_OK;
}

/* Steps 3-9: stable group-by bin */
void orc_assemble(const int32_t *pair_bin, const int32_t *pair_face, int64_t P,
                  int64_t n_bins, int32_t *counts, int32_t *offsets,
                  int32_t *face_ids) {
    memset(counts, 0, sizeof(int32_t) * (size_t)n_bins);
    for (int64_t p = 0; p < P; ++p) counts[pair_bin[p]]++;
    int64_t run = 0;
    for (int64_t b = 0; b < n_bins; ++b) {
        offsets[b] = (int32_t)run;
        run += counts[b];
    }
    int32_t *cur = (int32_t *)malloc(sizeof(int32_t) * (size_t)(n_bins > 0 ? n_bins : 1));
    memcpy(cur, offsets, sizeof(int32_t) * (size_t)n_bins);
    for (int64_t p = 0; p < P; ++p) face_ids[cur[pair_bin[p]]++] = pair_face[p];
    free(cur);
}

/* ------------------------------------------------------------------------ */
/* forest                                                  */

int orc_init_forest(orc_grid *g, const orc_config *c) {
    const int nx = c->nb[0], ny = c->nb[1], nz = c->nb[2];
    const int64_t n = (int64_t)nx * ny * nz;
    if (n > g->capacity) return ORC_ECAPACITY;
    for (int k = 0; k < nz; ++k)
        for (int j = 0; j < ny; ++j)
            for (int i = 0; i < nx; ++i) {
                const int64_t b = i + (int64_t)nx * (j + (int64_t)ny * k);
                g->coords[4 * b + 0] = i;
                g->coords[4 * b + 1] = j;
                g->coords[4 * b + 2] = k;
                g->coords[4 * b + 3] = 0;
                for (int q = 0; q < 27; ++q) {
                    const int ti = i + C27[q][0], tj = j + C27[q][1], tk = k + C27[q][2];
                    int32_t v;
                    if (ti < 0 || tj < 0 || tk < 0 || ti >= nx || tj >= ny || tk >= nz)
                        v = ORC_NB_OUTSIDE;
                    else
                        v = (int32_t)(ti + nx * (tj + ny * tk));
                    g->nbr[27 * b + q] = v;
                    g->nbr_child[27 * b + q] = -1;
                }
                g->child[b] = -1;
                g->bflags[b] = 0;
                memset(g->masks + 64 * b, ORC_FLUID, 64);
            }
    for (int L = 0; L <= ORC_MAX_LEVELS; ++L) g->level_start[L] = (int32_t)n;
    g->level_start[0] = 0;
    g->level_start[1] = (int32_t)n;
    g->n_levels = 1;
    return ORC_OK;
}

#define CELL(I, J, K) ((I) + 4 * (J) + 16 * (K))

/* ------------------------------------------------------------------------ */
/* Alg. 3 partial surface voxelization (pins A7-A9)                          */

int orc_voxelize_level(orc_grid *g, const orc_config *c, int L,
                       const int32_t *counts, const int32_t *offsets,
                       const int32_t *face_ids, const double *fc,
                       const double *nrm) {
    if (L < 0 || L >= g->n_levels) return ORC_EARG;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1];
    const double dx = level_dx(c, L), eps = c->eps_slab, lx = c->len[0];
    const int Bx = bins_axis(c, 0, L), By = bins_axis(c, 1, L);
#pragma omp parallel for schedule(dynamic, 64)
    for (int32_t b = s; b < e; ++b) {
        const int i = g->coords[4 * (int64_t)b], j = g->coords[4 * (int64_t)b + 1],
                  k = g->coords[4 * (int64_t)b + 2];
        const int64_t bin = i + (int64_t)Bx * (j + (int64_t)By * k);
        const int32_t n_f = counts[bin], off = offsets[bin];
        uint8_t *mk = g->masks + 64 * (int64_t)b;
        uint8_t orig[64], H[64];
        double dmin[64];
        for (int t = 0; t < 64; ++t) { orig[t] = H[t] = mk[t]; dmin[t] = INFINITY; }
        int any = 0;
        for (int K = 0; K < 4; ++K) {
            const double z = node_c(4 * k + K, dx);
            for (int J = 0; J < 4; ++J) {
                const double y = node_c(4 * j + J, dx);
                for (int p = 0; p < n_f; ++p) {
                    const int64_t f = face_ids[off + p];
                    const double *v = fc + 9 * f, *n = nrm + 3 * f;
                    if (fabs(n[0]) < c->eps_parallel) continue; /* A7 */
                    if (!sat3(v, 0.0, y - eps, z - eps, lx, y + eps, z + eps)) continue;
                    t_eval_ops += 4 * 11; /* per cell: num (8), /n_x, |d|, compare */
                    for (int I = 0; I < 4; ++I) {
                        const double x = node_c(4 * i + I, dx);
                        const double d = plane_num(v, n, x, y, z) / n[0];
                        const double ad = fabs(d);
                        const int t = CELL(I, J, K);
                        if (ad < dmin[t]) {
                            dmin[t] = ad;
                            H[t] = (n[0] * d > 0.0) ? ORC_SOLID : ORC_GUARD;
                            any = 1;
                        }
                    }
                }
            }
        }
        if (!any) continue; /* eta reduction */
        /* internal propagation, 3 Jacobi sweeps along +-x;
         * A8: a no-op with block-matched bins, kept literal here. */
        for (int it = 0; it < 3; ++it) {
            uint8_t Hn[64];
            memcpy(Hn, H, 64);
            for (int t = 0; t < 64; ++t) {
                const int I = t & 3;
                for (int sgn = -1; sgn <= 1; sgn += 2) {
                    const int In = I + sgn;
                    if (In < 0 || In > 3) continue;
                    const uint8_t hn = H[t + sgn];
                    if (hn == ORC_GUARD && Hn[t] == ORC_FLUID) Hn[t] = ORC_GUARD;
                    if (hn == ORC_SOLID && Hn[t] != ORC_GUARD) Hn[t] = ORC_SOLID;
                }
            }
            memcpy(H, Hn, 64);
        }
        for (int t = 0; t < 64; ++t) /* A9: write rule */
            if (H[t] == ORC_SOLID || (orig[t] != ORC_GHOST && orig[t] != ORC_INTERFACE))
                mk[t] = H[t];
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* Alg. 5 external propagation, literal chain walk (pin A10)                 */

int orc_propagate(orc_grid *g, const orc_config *c, int L, int dir) {
    (void)c;
    if (L < 0 || L >= g->n_levels) return ORC_EARG;
    const int fwd = dir > 0 ? 1 : 2, back = dir > 0 ? 2 : 1, trail = dir > 0 ? 3 : 0;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1];
#pragma omp parallel for schedule(dynamic, 16)
    for (int32_t b = s; b < e; ++b) {
        const int32_t code = g->nbr[27 * (int64_t)b + back];
        if (code >= 0) continue; /* not a run start */
        uint8_t st[16];
        const uint8_t *m0 = g->masks + 64 * (int64_t)b;
        for (int r = 0; r < 16; ++r) {
            st[r] = m0[trail + 4 * r];
            if (code == ORC_NB_SOLID_NBR && st[r] != ORC_GUARD) st[r] = ORC_SOLID;
        }
        int32_t cur = g->nbr[27 * (int64_t)b + fwd];
        while (cur >= 0) {
            uint8_t *mk = g->masks + 64 * (int64_t)cur;
            uint8_t nst[16];
            for (int r = 0; r < 16; ++r) {
                for (int I = 0; I < 4; ++I) {
                    uint8_t H = mk[I + 4 * r];
                    if (st[r] == ORC_SOLID && H != ORC_GUARD) H = ORC_SOLID;
                    mk[I + 4 * r] = H;
                }
                nst[r] = mk[trail + 4 * r];
                for (int I = 0; I < 4; ++I)
                    if (L == 0 && mk[I + 4 * r] == ORC_GUARD) mk[I + 4 * r] = ORC_FLUID;
            }
            memcpy(st, nst, 16);
            cur = g->nbr[27 * (int64_t)cur + fwd];
        }
    }
    return ORC_OK;
}

/* PAPER.md:832 (pin A11) */
int orc_finalize(orc_grid *g, const orc_config *c, int L) {
    (void)c;
    if (L < 0 || L >= g->n_levels) return ORC_EARG;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1];
#pragma omp parallel for schedule(static)
    for (int32_t b = s; b < e; ++b) {
        uint8_t *mk = g->masks + 64 * (int64_t)b;
        int solid = 0;
        for (int t = 0; t < 64; ++t) {
            if (mk[t] == ORC_GUARD) mk[t] = ORC_FLUID;
            if (mk[t] == ORC_SOLID) solid = 1;
        }
        g->bflags[b] = (uint8_t)((g->bflags[b] & ~ORC_BF_SOLID) | (solid ? ORC_BF_SOLID : 0));
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* near-wall marking (pin A12)                             */

int orc_mark(orc_grid *g, const orc_config *c, int L) {
    if (L < 0 || L >= g->n_levels) return ORC_EARG;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1], n = e - s;
    uint8_t *elig = (uint8_t *)calloc((size_t)n + 1, 1);
    uint8_t *sb = (uint8_t *)calloc((size_t)n + 1, 1);
    uint8_t *src = (uint8_t *)calloc((size_t)n + 1, 1);
    uint8_t *dst = (uint8_t *)calloc((size_t)n + 1, 1);
#define SOLIDB(x) (g->bflags[x] & ORC_BF_SOLID)
    for (int32_t b = s; b < e; ++b) {
        const int32_t *nb = g->nbr + 27 * (int64_t)b;
        int el = 1, sbv = 0;
        for (int q = 1; q < 27; ++q) {
            if (nb[q] == ORC_NB_MISSING || nb[q] == ORC_NB_SOLID_NBR) el = 0;
            if (nb[q] >= 0 && !SOLIDB(nb[q])) sbv = 1;
        }
        elig[b - s] = (uint8_t)el;
        sb[b - s] = (uint8_t)(SOLIDB(b) && sbv);
    }
    /* (i) + (ii) */
    for (int32_t b = s; b < e; ++b) {
        const int32_t *nb = g->nbr + 27 * (int64_t)b;
        int has_sb = 0;
        for (int q = 1; q < 27; ++q)
            if (nb[q] >= 0 && sb[nb[q] - s]) has_sb = 1;
        uint8_t f = (uint8_t)(g->bflags[b] & ~(ORC_BF_SB | ORC_BF_SA | ORC_BF_MARK));
        if (sb[b - s]) f |= ORC_BF_SB;
        if (has_sb && !SOLIDB(b)) f |= ORC_BF_SA;
        src[b - s] = (uint8_t)((sb[b - s] && elig[b - s]) || (has_sb && elig[b - s]));
        g->bflags[b] = f;
    }
    /* (iii) N_prop ping-pong sweeps; solid blocks only in sweep 0 */
    for (int it = 0; it < c->n_prop; ++it) {
        for (int32_t b = s; b < e; ++b) {
            uint8_t m = src[b - s];
            if (!m && elig[b - s] && (!SOLIDB(b) || it == 0)) {
                const int32_t *nb = g->nbr + 27 * (int64_t)b;
                for (int q = 1; q < 27; ++q)
                    if (nb[q] >= 0 && src[nb[q] - s]) { m = 1; break; }
            }
            dst[b - s] = m;
        }
        uint8_t *t = src; src = dst; dst = t;
    }
#undef SOLIDB
    for (int32_t b = s; b < e; ++b)
        if (src[b - s]) g->bflags[b] |= ORC_BF_MARK;
    free(elig); free(sb); free(src); free(dst);
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* adapt, refine-only (pins A13-A14)                       */

int orc_adapt(orc_grid *g, const orc_config *c, int L) {
    if (L < 0 || L != g->n_levels - 1 || L + 1 >= ORC_MAX_LEVELS) return ORC_EARG;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1];
    int64_t nm = 0;
    for (int32_t b = s; b < e; ++b)
        if (g->bflags[b] & ORC_BF_MARK) ++nm;
    if ((int64_t)e + 8 * nm > g->capacity) return ORC_ECAPACITY;
    int64_t r = 0;
    for (int32_t b = s; b < e; ++b) {
        if (g->bflags[b] & ORC_BF_MARK) {
            g->child[b] = (int32_t)(e + 8 * r++);
            g->bflags[b] |= ORC_BF_REFINED;
        } else {
            g->child[b] = -1;
            g->bflags[b] &= (uint8_t)~ORC_BF_REFINED;
        }
    }
    const int nbL1[3] = {bins_axis(c, 0, L + 1), bins_axis(c, 1, L + 1), bins_axis(c, 2, L + 1)};
    int err = 0;
    /* S4/S8: child metadata and neighbour links */
#pragma omp parallel for schedule(dynamic, 64) reduction(| : err)
    for (int32_t b = s; b < e; ++b) {
        if (g->child[b] < 0) continue;
        const int pi = g->coords[4 * (int64_t)b], pj = g->coords[4 * (int64_t)b + 1],
                  pk = g->coords[4 * (int64_t)b + 2];
        for (int cc = 0; cc < 8; ++cc) {
            const int cx = cc & 1, cy = (cc >> 1) & 1, cz = (cc >> 2) & 1;
            const int64_t id = g->child[b] + cc;
            const int ci = 2 * pi + cx, cj = 2 * pj + cy, ck = 2 * pk + cz;
            g->coords[4 * id + 0] = ci;
            g->coords[4 * id + 1] = cj;
            g->coords[4 * id + 2] = ck;
            g->coords[4 * id + 3] = L + 1;
            for (int q = 0; q < 27; ++q) {
                const int ti = ci + C27[q][0], tj = cj + C27[q][1], tk = ck + C27[q][2];
                int32_t v;
                if (ti < 0 || tj < 0 || tk < 0 || ti >= nbL1[0] || tj >= nbL1[1] || tk >= nbL1[2]) {
                    v = ORC_NB_OUTSIDE;
                } else {
                    const int qp = slot_of((ti >> 1) - pi, (tj >> 1) - pj, (tk >> 1) - pk);
                    const int32_t P = (qp == 0) ? b : g->nbr[27 * (int64_t)b + qp];
                    if (P < 0) { err = 1; v = ORC_NB_MISSING; }
                    else if (g->child[P] >= 0)
                        v = g->child[P] + (ti & 1) + 2 * (tj & 1) + 4 * (tk & 1);
                    else
                        v = (g->bflags[P] & ORC_BF_SOLID) ? ORC_NB_SOLID_NBR : ORC_NB_MISSING;
                }
                g->nbr[27 * id + q] = v;
                g->nbr_child[27 * id + q] = -1;
            }
            g->child[id] = -1;
            g->bflags[id] = 0;
            uint8_t *mk = g->masks + 64 * id;
            /* A14 ghost layer: fine cells within Chebyshev distance 2 of an
             * in-domain position without a level-(L+1) block */
            const int32_t *nb = g->nbr + 27 * id;
            for (int t = 0; t < 64; ++t) {
                const int I[3] = {t & 3, (t >> 2) & 3, (t >> 4) & 3};
                int ghost = 0;
                for (int q = 1; q < 27 && !ghost; ++q) {
                    int ok = 1;
                    for (int d = 0; d < 3; ++d) {
                        const int o = C27[q][d];
                        if (o == -1 && I[d] >= 2) ok = 0;
                        if (o == 1 && I[d] < 2) ok = 0;
                    }
                    if (ok && (nb[q] == ORC_NB_MISSING || nb[q] == ORC_NB_SOLID_NBR)) ghost = 1;
                }
                mk[t] = ghost ? ORC_GHOST : ORC_FLUID;
            }
        }
    }
    if (err) return ORC_EARG; /* a marked block had a missing neighbour */
    /* level-L neighbour-child links + interface layer on refined blocks */
#pragma omp parallel for schedule(static)
    for (int32_t b = s; b < e; ++b) {
        const int32_t *nb = g->nbr + 27 * (int64_t)b;
        for (int q = 0; q < 27; ++q) {
            const int32_t n = (q == 0) ? b : nb[q];
            g->nbr_child[27 * (int64_t)b + q] = (n >= 0) ? g->child[n] : -1;
        }
        if (g->child[b] < 0) continue;
        uint8_t *mk = g->masks + 64 * (int64_t)b;
        for (int t = 0; t < 64; ++t) {
            if (mk[t] != ORC_FLUID) continue;
            const int I[3] = {t & 3, (t >> 2) & 3, (t >> 4) & 3};
            int itf = 0;
            for (int q = 1; q < 27 && !itf; ++q) {
                int ok = 1;
                for (int d = 0; d < 3; ++d) {
                    const int o = C27[q][d];
                    if (o == -1 && I[d] != 0) ok = 0;
                    if (o == 1 && I[d] != 3) ok = 0;
                }
                if (ok && nb[q] >= 0 && g->child[nb[q]] < 0) itf = 1;
            }
            if (itf) mk[t] = ORC_INTERFACE;
        }
    }
    g->level_start[L + 2] = (int32_t)(e + 8 * nm);
    for (int k = L + 3; k <= ORC_MAX_LEVELS; ++k) g->level_start[k] = g->level_start[L + 2];
    g->n_levels = L + 2;
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* boundary cells (pins A15, A18)                          */

int orc_boundary(orc_grid *g, const orc_config *c, int32_t *bcount) {
    (void)c;
    const int L = g->n_levels - 1;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1];
    memset(bcount, 0, sizeof(int32_t) * (size_t)g->capacity);
    uint8_t *scratch = (uint8_t *)calloc((size_t)(e - s) * 64 + 1, 1);
#define SOLIDB(x) (g->bflags[x] & ORC_BF_SOLID)
    /* pass 1: candidate flags into scratch */
#pragma omp parallel for schedule(dynamic, 64)
    for (int32_t b = s; b < e; ++b) {
        const int32_t *nb = g->nbr + 27 * (int64_t)b;
        int cand = SOLIDB(b) ? 1 : 0;
        for (int q = 1; q < 27 && !cand; ++q)
            if (nb[q] >= 0 && SOLIDB(nb[q])) cand = 1;
        if (!cand) continue;
        const uint8_t *mk = g->masks + 64 * (int64_t)b;
        int cnt = 0;
        for (int t = 0; t < 64; ++t) {
            if (mk[t] != ORC_FLUID) continue;
            const int I[3] = {t & 3, (t >> 2) & 3, (t >> 4) & 3};
            int bnd = 0;
            for (int q = 1; q < 27 && !bnd; ++q) {
                int w[3], dir[3];
                for (int d = 0; d < 3; ++d) {
                    const int v = I[d] + C27[q][d];
                    /* A15: I' = mod(4 + mod(I + c, 4), 4) */
                    w[d] = ((v % 4) + 4) % 4;
                    dir[d] = (v < 0 || v > 3) ? C27[q][d] : 0;
                }
                const int qs = slot_of(dir[0], dir[1], dir[2]);
                const int32_t nbk = (qs == 0) ? b : nb[qs];
                if (nbk < 0) continue;
                if (g->masks[64 * (int64_t)nbk + CELL(w[0], w[1], w[2])] == ORC_SOLID) bnd = 1;
            }
            if (bnd) { scratch[(int64_t)(b - s) * 64 + t] = 1; ++cnt; }
        }
        bcount[b] = cnt;
    }
#undef SOLIDB
    /* pass 2: commit */
#pragma omp parallel for schedule(static)
    for (int32_t b = s; b < e; ++b) {
        uint8_t *mk = g->masks + 64 * (int64_t)b;
        for (int t = 0; t < 64; ++t)
            if (scratch[(int64_t)(b - s) * 64 + t]) mk[t] = ORC_BOUNDARY;
        if (bcount[b] > 0) g->bflags[b] |= ORC_BF_BOUNDARY;
        else g->bflags[b] &= (uint8_t)~ORC_BF_BOUNDARY;
    }
    free(scratch);
    return ORC_OK;
}

/* PAPER.md:961-969, pin A16: slots ascend by block id */
int64_t orc_tables(const orc_grid *g, const int32_t *bcount, int32_t *cmap) {
    const int32_t n_used = g->level_start[g->n_levels];
    int64_t nb = 0;
    for (int32_t b = 0; b < n_used; ++b) cmap[b] = (bcount[b] > 0) ? (int32_t)nb++ : -1;
    return nb;
}

/* ------------------------------------------------------------------------ */
/* link lengths (pin A17)                                  */

int orc_link_lengths(const orc_grid *g, const orc_config *c, const int32_t *cmap,
                     int64_t n_b, const int32_t *counts, const int32_t *offsets,
                     const int32_t *face_ids, const double *fc, const double *nrm,
                     float *lengths) {
    const int L = g->n_levels - 1;
    const int32_t s = g->level_start[L], e = g->level_start[L + 1];
    const double dx = level_dx(c, L), eps = c->eps_slab;
    const int Bx = bins_axis(c, 0, L), By = bins_axis(c, 1, L);
    for (int64_t i = 0; i < n_b * 27 * 64; ++i) lengths[i] = -1.0f;
    double cn[27];
    for (int q = 0; q < 27; ++q)
        cn[q] = sqrt((double)(C27[q][0] * C27[q][0] + C27[q][1] * C27[q][1] + C27[q][2] * C27[q][2]));
#pragma omp parallel for schedule(dynamic, 16)
    for (int32_t b = s; b < e; ++b) {
        const int32_t slot = cmap[b];
        if (slot < 0) continue;
        const int i = g->coords[4 * (int64_t)b], j = g->coords[4 * (int64_t)b + 1],
                  k = g->coords[4 * (int64_t)b + 2];
        const int64_t bin = i + (int64_t)Bx * (j + (int64_t)By * k);
        const int32_t n_f = counts[bin], off = offsets[bin];
        for (int t = 0; t < 64; ++t) {
            const double x = node_c(4 * i + (t & 3), dx);
            const double y = node_c(4 * j + ((t >> 2) & 3), dx);
            const double z = node_c(4 * k + ((t >> 4) & 3), dx);
            double best[27];
            for (int q = 0; q < 27; ++q) best[q] = INFINITY;
            for (int p = 0; p < n_f; ++p) {
                const int64_t f = face_ids[off + p];
                const double *v = fc + 9 * f, *n = nrm + 3 * f;
                const double num = plane_num(v, n, x, y, z);
                t_eval_ops += 8 + 26 * 9; /* num; per q: den (5), |den| test (2), d, range */
                for (int q = 1; q < 27; ++q) {
                    const double c0 = C27[q][0], c1 = C27[q][1], c2 = C27[q][2];
                    const double den = (c0 * n[0] + c1 * n[1]) + c2 * n[2];
                    if (fabs(den) < c->eps_parallel * cn[q]) continue;
                    const double d = num / den;
                    if (!(d > 0.0 && d <= dx)) continue;
                    t_eval_ops += 6; /* the piercing point */
                    const double xi = x + d * c0, yi = y + d * c1, zi = z + d * c2;
                    if (!sat3(v, xi - eps, yi - eps, zi - eps, xi + eps, yi + eps, zi + eps)) continue;
                    if (d < best[q]) best[q] = d;
                }
            }
            for (int q = 1; q < 27; ++q)
                if (best[q] < INFINITY)
                    lengths[((int64_t)slot * 27 + q) * 64 + t] = (float)(best[q] / dx);
        }
    }
    return ORC_OK;
}

/* ------------------------------------------------------------------------ */
/* embed_geometry driver                                   */

struct orc_links {
    int64_t nb;
    int32_t n_used;
    int32_t *cmap;
    float *lengths;
};

static double now_s(void) {
    struct timespec ts;
    clock_gettime(CLOCK_MONOTONIC, &ts);
    return ts.tv_sec + 1e-9 * ts.tv_nsec;
}

typedef struct {
    int64_t n_bins;
    int32_t *counts, *offsets, *face_ids;
} orc_binlevel;

static int build_bins(const orc_config *c, const double *fc, const double *nrm,
                      int64_t F, int L, int mode, int use_filter, orc_binlevel *out) {
    uint8_t *ind = (uint8_t *)malloc((size_t)F + 1);
    int32_t *map = (int32_t *)malloc(sizeof(int32_t) * ((size_t)F + 1));
    int64_t nmap;
    if (use_filter) {
        orc_ray_indicators(fc, nrm, F, c, L, mode, ind);
        orc_ops_flush(mode == 0 ? ORC_ST_IND : ORC_ST_MD);
        nmap = orc_compact(ind, F, map);
    } else {
        for (int64_t f = 0; f < F; ++f) map[f] = (int32_t)f;
        nmap = F;
    }
    const int nlim = (2 + c->n_spec) * (2 + c->n_spec) * (2 + c->n_spec);
    const int64_t cap = nmap * nlim + 1;
    int32_t *pb = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    int32_t *pf = (int32_t *)malloc(sizeof(int32_t) * (size_t)cap);
    int64_t P = 0;
    int rc = orc_bin_pairs(fc, F, map, nmap, c, L, pb, pf, cap, &P);
    orc_ops_flush(mode == 0 ? ORC_ST_PAIRS : ORC_ST_MD);
    const int64_t nb = (int64_t)bins_axis(c, 0, L) * bins_axis(c, 1, L) * bins_axis(c, 2, L);
    out->n_bins = nb;
    out->counts = (int32_t *)malloc(sizeof(int32_t) * (size_t)nb);
    out->offsets = (int32_t *)malloc(sizeof(int32_t) * (size_t)nb);
    out->face_ids = (int32_t *)malloc(sizeof(int32_t) * (size_t)(P + 1));
    if (rc == ORC_OK) orc_assemble(pb, pf, P, nb, out->counts, out->offsets, out->face_ids);
    free(ind); free(map); free(pb); free(pf);
    return rc;
}

static void free_bins(orc_binlevel *b) {
    free(b->counts); free(b->offsets); free(b->face_ids);
    b->counts = b->offsets = b->face_ids = NULL;
}

/* stage_seconds: [0] binning, [1] voxelize+propagate+finalize, [2] mark,
 * [3] adapt, [4] boundary+tables, [5] MD bins, [6] link lengths, [7] total */
int orc_embed(orc_grid *g, const orc_config *c, const double *fc, const double *nrm,
              int64_t F, int use_filter, orc_links **out, double *st) {
    double acc[8] = {0};
    const double t_start = now_s();
    orc_ops_flush(ORC_ST_IND);          /* drop counts of earlier direct calls */
    memset(g_ops, 0, sizeof(g_ops));
    int rc = orc_init_forest(g, c);
    if (rc) return rc;
    for (int L = 0; L < c->l_max; ++L) {
        double t0 = now_s();
        orc_binlevel bl;
        rc = build_bins(c, fc, nrm, F, L, 0, use_filter, &bl);
        acc[0] += now_s() - t0;
        /* build_bins flushes indicators and pairs separately (below) */
        if (rc) { free_bins(&bl); return rc; }
        t0 = now_s();
        orc_voxelize_level(g, c, L, bl.counts, bl.offsets, bl.face_ids, fc, nrm);
        orc_ops_flush(ORC_ST_VOX);
        free_bins(&bl);
        orc_propagate(g, c, L, +1);
        if (L > 0) orc_propagate(g, c, L, -1);
        orc_finalize(g, c, L);
        acc[1] += now_s() - t0;
        if (L == c->l_max - 1) break;
        t0 = now_s();
        orc_mark(g, c, L);
        acc[2] += now_s() - t0;
        t0 = now_s();
        rc = orc_adapt(g, c, L);
        acc[3] += now_s() - t0;
        if (rc) return rc;
    }
    double t0 = now_s();
    int32_t *bcount = (int32_t *)malloc(sizeof(int32_t) * (size_t)g->capacity);
    orc_boundary(g, c, bcount);
    orc_links *h = (orc_links *)calloc(1, sizeof(orc_links));
    h->n_used = g->level_start[g->n_levels];
    h->cmap = (int32_t *)malloc(sizeof(int32_t) * ((size_t)h->n_used + 1));
    h->nb = orc_tables(g, bcount, h->cmap);
    h->lengths = (float *)malloc(sizeof(float) * (size_t)(h->nb * 27 * 64 + 1));
    free(bcount);
    acc[4] += now_s() - t0;
    t0 = now_s();
    orc_binlevel md;
    rc = build_bins(c, fc, nrm, F, g->n_levels - 1, 1, use_filter, &md);
    acc[5] += now_s() - t0;
    if (rc) { free_bins(&md); orc_links_free(h); return rc; }
    t0 = now_s();
    orc_link_lengths(g, c, h->cmap, h->nb, md.counts, md.offsets, md.face_ids, fc, nrm, h->lengths);
    orc_ops_flush(ORC_ST_LINKS);
    acc[6] += now_s() - t0;
    free_bins(&md);
    acc[7] = now_s() - t_start;
    if (st) memcpy(st, acc, sizeof(acc));
    *out = h;
    return ORC_OK;
}

int64_t orc_links_nb(const orc_links *h) { return h->nb; }

void orc_links_copy(const orc_links *h, int32_t *cmap, float *lengths) {
    if (cmap) memcpy(cmap, h->cmap, sizeof(int32_t) * (size_t)h->n_used);
    if (lengths) memcpy(lengths, h->lengths, sizeof(float) * (size_t)(h->nb * 27 * 64));
}

void orc_links_free(orc_links *h) {
    if (!h) return;
    free(h->cmap);
    free(h->lengths);
    free(h);
}

/* ------------------------------------------------------------------------ */
/* validation: +x ray parity against all faces           */

void orc_parity_inside(const double *fc, int64_t F, const double *pts, int64_t n,
                       double tol, uint8_t *out) {
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; ++i) {
        const double px = pts[3 * i], py = pts[3 * i + 1], pz = pts[3 * i + 2];
        int cnt = 0, amb = 0;
        for (int64_t f = 0; f < F && !amb; ++f) {
            const double *v = fc + 9 * f;
            const double ymin = mn(mn(v[1], v[4]), v[7]), ymax = mx_(mx_(v[1], v[4]), v[7]);
            const double zmin = mn(mn(v[2], v[5]), v[8]), zmax = mx_(mx_(v[2], v[5]), v[8]);
            if (py < ymin - tol || py > ymax + tol || pz < zmin - tol || pz > zmax + tol) continue;
            /* 2D edge functions in the (y,z) projection, long double */
            long double e[3];
            long double len[3];
            for (int a = 0; a < 3; ++a) {
                const double *p0 = v + 3 * a, *p1 = v + 3 * ((a + 1) % 3);
                const long double ey = (long double)p1[1] - p0[1], ez = (long double)p1[2] - p0[2];
                e[a] = ey * ((long double)pz - p0[2]) - ez * ((long double)py - p0[1]);
                len[a] = sqrtl(ey * ey + ez * ez);
            }
            int pos = 0, neg = 0, near = 0;
            for (int a = 0; a < 3; ++a) {
                if (fabsl(e[a]) <= tol * (len[a] > 0 ? len[a] : 1)) near = 1;
                if (e[a] > 0) pos++;
                if (e[a] < 0) neg++;
            }
            if (near) { amb = 1; break; }
            if (pos && neg) continue; /* outside projection */
            if (!pos && !neg) continue; /* degenerate */
            /* plane intersection x along the row */
            const long double ax = (long double)v[3] - v[0], ay = (long double)v[4] - v[1], az = (long double)v[5] - v[2];
            const long double bx = (long double)v[6] - v[0], by = (long double)v[7] - v[1], bz = (long double)v[8] - v[2];
            const long double nx = ay * bz - az * by, ny = az * bx - ax * bz, nz = ax * by - ay * bx;
            if (nx == 0) continue;
            const long double xi = v[0] - (ny * ((long double)py - v[1]) + nz * ((long double)pz - v[2])) / nx;
            const long double nn = sqrtl(nx * nx + ny * ny + nz * nz);
            if (fabsl((xi - px) * nx) <= tol * nn) { amb = 1; break; }
            if (xi > px) cnt++;
        }
        out[i] = amb ? 2 : (uint8_t)(cnt & 1);
    }
}
