/* lbm_oracle.c -- CPU restatement of the LUT consumer: one D3Q27 BGK
 * collide/stream step of one grid level with wall links from the LinkTable
 * (collide_stream_level; equilibrium SPEC.md:392-397;
 * accumulate_forces SPEC.md:436-440).  TEST INFRASTRUCTURE ONLY (see
 * vf_oracle.h): the checker of csrc/vf_lbm.cu, never linked by the product.
 *
 * FP64 throughout, straight per-cell loops.  State = post-collision
 * populations, SoA fin[q][cell], cell = (block - s) * 64 + t over the level's
 * blocks [s, e).  Pull streaming: the population arriving at x along c_o
 * comes from y = x - c_o; when y is
 *   - a level cell that is not SOLID: fin[o](y);
 *   - SOLID (or a missing block, only next to ghost cells): wall link from x
 *     towards y, q = opp(o), q_w from lengths[(cmap[b]*27 + q)*64 + t]:
 *       SBB (or q_w unknown): f_o = fin[q](x)
 *       IBB (Bouzidi linear):
 *         q_w <  1/2: f_o = 2 q_w fin[q](x) + (1 - 2 q_w) fin[q](x + c_o)
 *                     (SBB when x + c_o is not a fluid level cell)
 *         q_w >= 1/2: f_o = fin[q](x) / (2 q_w) + (2 q_w - 1) / (2 q_w) fin[o](x)
 *       momentum exchange F += (fin[q](x) + f_o) c_q (lattice units);
 *   - outside the domain: x = 0 inlet (velocity bounce-back, rho_w = 1:
 *     f_o = fin[q](x) - 6 w_q (c_q . u_in)), x = l_x outlet (anti-bounce-back
 *     at rho_w = 1: f_o = -fin[q](x) + 2 w_q (1 + 4.5 (c_q.u)^2 - 1.5 u.u),
 *     u = velocity of x), other faces SBB (all faces SBB when !open_x).
 * Then BGK: f_o += (feq_o(rho, u) - f_o) / tau.  GHOST cells are held (their
 * values come from the interface exchange), SOLID cells are
 * left untouched. */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "vf_oracle.h"

/* D3Q27 order of lattice.py:19-39 */
static const int LC[27][3] = {{0, 0, 0},   {1, 0, 0},   {-1, 0, 0},  {0, 1, 0},   {0, -1, 0},
                              {0, 0, 1},   {0, 0, -1},  {1, 1, 0},   {-1, -1, 0}, {1, 0, 1},
                              {-1, 0, -1}, {1, 0, -1},  {-1, 0, 1},  {1, -1, 0},  {-1, 1, 0},
                              {0, 1, 1},   {0, -1, -1}, {0, 1, -1},  {0, -1, 1},  {1, 1, 1},
                              {-1, -1, -1}, {1, 1, -1}, {-1, -1, 1}, {1, -1, 1},  {-1, 1, -1},
                              {1, -1, -1}, {-1, 1, 1}};

static double lw(int q) {
    const int s = abs(LC[q][0]) + abs(LC[q][1]) + abs(LC[q][2]);
    return s == 0 ? 8.0 / 27.0 : s == 1 ? 2.0 / 27.0 : s == 2 ? 1.0 / 54.0 : 1.0 / 216.0;
}
static int lopp(int q) { return q == 0 ? 0 : (q & 1 ? q + 1 : q - 1); }
static int lslot(int dx, int dy, int dz) {
    for (int q = 0; q < 27; ++q)
        if (LC[q][0] == dx && LC[q][1] == dy && LC[q][2] == dz) return q;
    return -1;
}

void orc_lbm_equilibrium(double rho, const double *u, double *feq) {
    const double uu = u[0] * u[0] + u[1] * u[1] + u[2] * u[2];
    for (int q = 0; q < 27; ++q) {
        const double cu = LC[q][0] * u[0] + LC[q][1] * u[1] + LC[q][2] * u[2];
        feq[q] = lw(q) * rho * (1.0 + 3.0 * cu + 4.5 * cu * cu - 1.5 * uu);
    }
}

/* level cell of (block b, cell I,J,K shifted by d): returns the block id (or a
 * negative nbr code) and the local cell index through *t */
static int32_t cell_at(const int32_t *nbr, int32_t b, int I, int J, int K, int dx, int dy, int dz,
                       int *t) {
    const int X = I + dx, Y = J + dy, Z = K + dz;
    const int ox = X < 0 ? -1 : (X > 3 ? 1 : 0), oy = Y < 0 ? -1 : (Y > 3 ? 1 : 0),
              oz = Z < 0 ? -1 : (Z > 3 ? 1 : 0);
    *t = (X & 3) + 4 * (Y & 3) + 16 * (Z & 3);
    if (!ox && !oy && !oz) return b;
    return nbr[27 * (int64_t)b + lslot(ox, oy, oz)];
}

int orc_lbm_step(const int32_t *coords, const int32_t *nbr, const uint8_t *masks, int32_t s,
                 int32_t e, int cells_x, const int32_t *cmap, const float *lengths,
                 const float *fin, float *fout, double tau, const double *u_in, int ibb,
                 int open_x, double *force) {
    const int64_t n = (int64_t)(e - s) * 64;
    double F[3] = {0, 0, 0};
#define FIN(q, cell) ((double)fin[(int64_t)(q) * n + (cell)])
    for (int32_t b = s; b < e; ++b) {
        for (int t = 0; t < 64; ++t) {
            const int64_t x = (int64_t)(b - s) * 64 + t;
            const uint8_t m = masks[64 * (int64_t)b + t];
            if (m == ORC_SOLID || m == ORC_GHOST) {
                for (int q = 0; q < 27; ++q) fout[q * n + x] = fin[q * n + x];
                continue;
            }
            const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
            double f[27], rx = 0, ux0 = 0, uy0 = 0, uz0 = 0;
            for (int q = 0; q < 27; ++q) {  /* moments of x (outlet ABB) */
                const double v = FIN(q, x);
                rx += v;
                ux0 += v * LC[q][0];
                uy0 += v * LC[q][1];
                uz0 += v * LC[q][2];
            }
            const double ux[3] = {ux0 / rx, uy0 / rx, uz0 / rx};
            for (int o = 0; o < 27; ++o) {
                const int q = lopp(o);
                int ty;
                const int32_t y = cell_at(nbr, b, I, J, K, -LC[o][0], -LC[o][1], -LC[o][2], &ty);
                if (y >= s && y < e && masks[64 * (int64_t)y + ty] != ORC_SOLID) {
                    f[o] = FIN(o, (int64_t)(y - s) * 64 + ty);
                    continue;
                }
                if (y == ORC_NB_OUTSIDE) {  /* domain face */
                    const int gx = 4 * coords[4 * (int64_t)b] + I - LC[o][0];
                    const double cu = LC[q][0] * u_in[0] + LC[q][1] * u_in[1] + LC[q][2] * u_in[2];
                    if (!open_x) {
                        f[o] = FIN(q, x);
                    } else if (gx < 0) {
                        f[o] = FIN(q, x) - 6.0 * lw(q) * cu;
                    } else if (gx >= cells_x) {
                        const double cq = LC[q][0] * ux[0] + LC[q][1] * ux[1] + LC[q][2] * ux[2];
                        const double uu = ux[0] * ux[0] + ux[1] * ux[1] + ux[2] * ux[2];
                        f[o] = -FIN(q, x) + 2.0 * lw(q) * (1.0 + 4.5 * cq * cq - 1.5 * uu);
                    } else {
                        f[o] = FIN(q, x);
                    }
                    continue;
                }
                /* wall link x -> y (SOLID cell or missing block) */
                double qw = -1.0;
                if (ibb && cmap[b] >= 0) qw = lengths[((int64_t)cmap[b] * 27 + q) * 64 + t];
                const double fq = FIN(q, x);
                double fo;
                if (!(qw > 0.0)) {
                    fo = fq;
                } else if (qw < 0.5) {
                    int tz;
                    const int32_t z = cell_at(nbr, b, I, J, K, LC[o][0], LC[o][1], LC[o][2], &tz);
                    if (z >= s && z < e && masks[64 * (int64_t)z + tz] != ORC_SOLID)
                        fo = 2.0 * qw * fq + (1.0 - 2.0 * qw) * FIN(q, (int64_t)(z - s) * 64 + tz);
                    else
                        fo = fq;
                } else {
                    fo = fq / (2.0 * qw) + (2.0 * qw - 1.0) / (2.0 * qw) * FIN(o, x);
                }
                f[o] = fo;
                for (int d = 0; d < 3; ++d) F[d] += (fq + fo) * LC[q][d];
            }
            double rho = 0, u[3] = {0, 0, 0};
            for (int o = 0; o < 27; ++o) {
                rho += f[o];
                for (int d = 0; d < 3; ++d) u[d] += f[o] * LC[o][d];
            }
            for (int d = 0; d < 3; ++d) u[d] /= rho;
            double feq[27];
            orc_lbm_equilibrium(rho, u, feq);
            for (int o = 0; o < 27; ++o) fout[o * n + x] = (float)(f[o] + (feq[o] - f[o]) / tau);
        }
    }
#undef FIN
    if (force)
        for (int d = 0; d < 3; ++d) force[d] = F[d];
    return 0;
}

/* ---- interface exchange: the rules of csrc/vf_lbm.cu
 * k_lbm_fill_ghosts / k_lbm_restrict, restated in FP64.  Fine global cell g
 * (per axis) sits in coarse cell g >> 1 at offset s/4, s = +1 for odd g, -1
 * for even g.  GHOST fine cells take the tensor-product interpolation of
 * (1 - theta) fc_old + theta fc_new over the coarse cells G + s k:
 * cubic Lagrange at x = 1/4 (k = -1..2, w = (-7, 105, 35, -5)/128) when all
 * 64 stencil cells are level cells that are not SOLID, else linear (k = 0, 1,
 * w = (3, 1)/4) when all 8 are, else the coarse cell G itself, else held;
 * then f = feq(rho, u) + alpha (f - feq(rho, u)) unless alpha == 1.
 * Restriction: coarse cells of refined blocks that are not SOLID, INTERFACE
 * or GHOST and have no GHOST child <- mean of the non-SOLID children, then
 * the beta rescale. */
static void orc_neq_rescale(double *f, double a) {
    if (a == 1.0) return;
    double rho = 0, u[3] = {0, 0, 0};
    for (int o = 0; o < 27; ++o) {
        rho += f[o];
        for (int d = 0; d < 3; ++d) u[d] += f[o] * LC[o][d];
    }
    if (!(rho > 0)) return;
    for (int d = 0; d < 3; ++d) u[d] /= rho;
    double feq[27];
    orc_lbm_equilibrium(rho, u, feq);
    for (int o = 0; o < 27; ++o) f[o] = feq[o] + a * (f[o] - feq[o]);
}

int orc_lbm_fill_ghosts(const int32_t *coords, const int32_t *nbr, const uint8_t *masks,
                        const int32_t *child, int32_t sf, int32_t ef, int32_t sc, int32_t ec,
                        const float *fc_old, const float *fc_new, double theta, double alpha,
                        int order, float *ff) {
    static const double W3[4] = {-7.0 / 128, 105.0 / 128, 35.0 / 128, -5.0 / 128};
    const int64_t nf = (int64_t)(ef - sf) * 64, nc = (int64_t)(ec - sc) * 64;
    int32_t *par = (int32_t *)malloc(sizeof(int32_t) * (size_t)(ef - sf + 1));
    if (!par) return 1;
    for (int32_t b = sf; b < ef; ++b) par[b - sf] = -1;
    for (int32_t P = sc; P < ec; ++P)
        if (child[P] >= 0)
            for (int o = 0; o < 8; ++o)
                if (child[P] + o >= sf && child[P] + o < ef) par[child[P] + o - sf] = P;
    for (int32_t b = sf; b < ef; ++b) {
        const int32_t P = par[b - sf];
        if (P < 0) continue;
        for (int t = 0; t < 64; ++t) {
            if (masks[64 * (int64_t)b + t] != ORC_GHOST) continue;
            const int Il[3] = {t & 3, (t >> 2) & 3, t >> 4};
            int Lc[3], sd[3];
            for (int d = 0; d < 3; ++d) {
                const int g = 4 * coords[4 * (int64_t)b + d] + Il[d];
                Lc[d] = (int)floor(g / 2.0) - 4 * coords[4 * (int64_t)P + d];
                sd[d] = (g % 2 != 0) ? 1 : -1;
            }
            /* stencil cell list for the highest usable order */
            int64_t idx[64];
            int ord = order;
            for (;;) {
                const int kn = ord == 3 ? 4 : (ord == 1 ? 2 : 1), k0 = ord == 3 ? -1 : 0;
                int ok = 1, nk = 0;
                for (int kz = 0; kz < kn && ok; ++kz)
                    for (int ky = 0; ky < kn && ok; ++ky)
                        for (int kx = 0; kx < kn && ok; ++kx) {
                            const int l[3] = {Lc[0] + sd[0] * (kx + k0), Lc[1] + sd[1] * (ky + k0),
                                              Lc[2] + sd[2] * (kz + k0)};
                            int o3[3];
                            for (int d = 0; d < 3; ++d) o3[d] = l[d] < 0 ? -1 : (l[d] > 3 ? 1 : 0);
                            const int32_t Z = (o3[0] || o3[1] || o3[2])
                                                  ? nbr[27 * (int64_t)P + lslot(o3[0], o3[1], o3[2])]
                                                  : P;
                            const int tt = (l[0] & 3) + 4 * (l[1] & 3) + 16 * (l[2] & 3);
                            if (Z < sc || Z >= ec || masks[64 * (int64_t)Z + tt] == ORC_SOLID) ok = 0;
                            else idx[nk++] = (int64_t)(Z - sc) * 64 + tt;
                        }
                if (ok) break;
                if (ord == 0) { ord = -1; break; }
                ord = ord == 3 ? 1 : 0;
            }
            if (ord < 0) continue; /* held */
            const int kn = ord == 3 ? 4 : (ord == 1 ? 2 : 1);
            double f[27];
            for (int q = 0; q < 27; ++q) {
                double acc = 0;
                int k = 0;
                for (int kz = 0; kz < kn; ++kz)
                    for (int ky = 0; ky < kn; ++ky)
                        for (int kx = 0; kx < kn; ++kx, ++k) {
                            const double w =
                                ord == 3 ? W3[kx] * W3[ky] * W3[kz]
                                : ord == 1 ? (kx ? 0.25 : 0.75) * (ky ? 0.25 : 0.75) * (kz ? 0.25 : 0.75)
                                           : 1.0;
                            const int64_t c = (int64_t)q * nc + idx[k];
                            const double v = theta == 0.0 ? (double)fc_old[c]
                                                          : (1.0 - theta) * fc_old[c] + theta * fc_new[c];
                            acc += w * v;
                        }
                f[q] = acc;
            }
            orc_neq_rescale(f, alpha);
            for (int q = 0; q < 27; ++q) ff[(int64_t)q * nf + (int64_t)(b - sf) * 64 + t] = (float)f[q];
        }
    }
    free(par);
    return 0;
}

int orc_lbm_restrict(const uint8_t *masks, const int32_t *child, int32_t sc, int32_t ec, int32_t sf,
                     int32_t ef, const float *ff, double beta, float *fc) {
    const int64_t nf = (int64_t)(ef - sf) * 64, nc = (int64_t)(ec - sc) * 64;
    for (int32_t b = sc; b < ec; ++b) {
        if (child[b] < 0) continue;
        for (int t = 0; t < 64; ++t) {
            const uint8_t m = masks[64 * (int64_t)b + t];
            if (m == ORC_SOLID || m == ORC_INTERFACE || m == ORC_GHOST) continue;
            const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
            const int32_t Cb = child[b] + (I >> 1) + 2 * (J >> 1) + 4 * (K >> 1);
            if (Cb < sf || Cb >= ef) continue;
            int64_t fine[8];
            int n = 0, ghost = 0;
            for (int c = 0; c < 2; ++c)
                for (int bb = 0; bb < 2; ++bb)
                    for (int a = 0; a < 2; ++a) {
                        const int tt = (2 * (I & 1) + a) + 4 * (2 * (J & 1) + bb) + 16 * (2 * (K & 1) + c);
                        const uint8_t mf = masks[64 * (int64_t)Cb + tt];
                        if (mf == ORC_GHOST) ghost = 1;
                        if (mf != ORC_SOLID) fine[n++] = (int64_t)(Cb - sf) * 64 + tt;
                    }
            if (ghost || n == 0) continue;
            double f[27];
            for (int q = 0; q < 27; ++q) {
                double acc = 0;
                for (int k = 0; k < n; ++k) acc += ff[(int64_t)q * nf + fine[k]];
                f[q] = acc / n;
            }
            orc_neq_rescale(f, beta);
            for (int q = 0; q < 27; ++q) fc[(int64_t)q * nc + (int64_t)(b - sc) * 64 + t] = (float)f[q];
        }
    }
    return 0;
}
