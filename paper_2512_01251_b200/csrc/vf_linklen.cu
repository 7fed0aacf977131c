// vf_linklen.cu -- cut-link lengths (pin A17).
//
// FACE-parallel formulation.  A link (lattice node v of a mapped finest-level
// block, direction c_q, 0 < d <= dx) is accepted when the eps-cube around its
// piercing point v + d c_q overlaps the face (exact SAT); the LUT keeps the
// minimum q = d/dx over faces.  Instead of every cell scanning its block's
// all-directions bin (the paper's per-cell loop), every face enumerates the
// lattice LINES that pierce it and min-merges q into the LUT with atomicMin on
// the IEEE bits -- order-free, hence deterministic and equal to the per-cell
// minimum (for q > 0 uint32 order is float order, and the -1.0f initialisation
// 0xBF800000 sorts above every positive float, so "no hit" needs no final
// pass).  A dense block map of the finest level replaces the bin lookup; the
// all-directions binning drops out of the embed path (the result is invariant
// to it; the oracle keeps the per-cell MD-bin formulation).
//
// K-link, thread per face, for each of the 13 antiparallel direction pairs c:
//   - the lattice lines along c cut the coordinate plane x_p = v1_p (p = first
//     axis with c_p != 0) in a square lattice of pitch dx; project the
//     triangle along c onto that plane and enumerate the lattice points of its
//     bounding box that fall inside the projected triangle (FP32, relative to
//     v1, margins >= 10x the FP32 error bound);
//   - a line through the triangle meets the face plane at one point; the
//     (2, rarely 3) lattice nodes within one link of that crossing are the
//     only possible link endpoints, in +c or -c direction.
// Lines are classified with FP32 edge functions and margins far above their
// rounding error:
//   - clearly outside the projected triangle: no link (the exact SAT rejects);
//   - clearly inside, well-conditioned crossing: FAST exact path -- the FP64
//     num/den/d/q of the oracle without the eps-box SAT, which provably
//     accepts an interior piercing point (link_fast);
//   - within the margin band of an edge, or ill-conditioned: the candidate
//     (face, node, pair) goes to a per-warp shared-memory queue drained 32 at
//     a time through the full exact FP64 path with the SAT (link_candidate),
//     so the SAT runs warp-converged.
// Every stored value is the oracle's FP64 value; only the SAT evaluation is
// skipped where its outcome is certain.
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

#ifndef VF_LINK_MINB
#define VF_LINK_MINB 6
#endif

namespace vf {

// exact decision for one (face, node, direction pair) candidate: num and
// d = num/den bit-identical to the oracle (orc_link_lengths), then the
// eps-box SAT at the piercing point
__device__ __noinline__ void link_candidate(const double *__restrict__ faces, int64_t f, int r,
                                            int i, int j, int k, double dx, double eps,
                                            double eps_par, int32_t slot,
                                            float *__restrict__ lengths) {
    double v[9], nn[3];
    load_face(faces, f, v, nn);
    const double x = node_c(i, dx), y = node_c(j, dx), z = node_c(k, dx);
    const double num = plane_num(v, nn, x, y, z);
    const int q1 = 2 * r + 1;
    const double c0 = c27(q1, 0), c1 = c27(q1, 1), c2 = c27(q1, 2);
    const double cn = __dsqrt_rn(VF_DADD(VF_DADD(VF_DMUL(c0, c0), VF_DMUL(c1, c1)), VF_DMUL(c2, c2)));
    const double den = VF_DADD(VF_DADD(VF_DMUL(c0, nn[0]), VF_DMUL(c1, nn[1])), VF_DMUL(c2, nn[2]));
    if (fabs(den) < VF_DMUL(eps_par, cn)) return;  // EPS_PARALLEL (geometry.py:25,435)
    const double d = VF_DDIV(num, den);
    // d > 0: slot q = 2r+1; d < 0: opposite slot with d' = -d exactly
    // (den' = -den bitwise) and v + d'c' == v + d c
    const bool pos = d > 0.0;
    const double dd = pos ? d : -d;
    if (!(dd > 0.0 && dd <= dx)) return;
    const int q = pos ? q1 : q1 + 1;
    const double e0 = c27(q, 0), e1 = c27(q, 1), e2 = c27(q, 2);
    const double xi = VF_DADD(x, VF_DMUL(dd, e0));
    const double yi = VF_DADD(y, VF_DMUL(dd, e1));
    const double zi = VF_DADD(z, VF_DMUL(dd, e2));
    SatFace sf;
    sat_face_init(sf, v);
    if (!sat_exact(sf, VF_DSUB(xi, eps), VF_DSUB(yi, eps), VF_DSUB(zi, eps), VF_DADD(xi, eps),
                   VF_DADD(yi, eps), VF_DADD(zi, eps)))
        return;
    const float qv = __double2float_rn(VF_DDIV(dd, dx));
    const int t = (i & 3) + 4 * (j & 3) + 16 * (k & 3);
    atomicMin(reinterpret_cast<unsigned int *>(lengths) + ((int64_t)slot * 27 + q) * 64 + t,
              __float_as_uint(qv));
}

constexpr int kLinkWarps = 4;

struct LinkCtx {
    const double *faces;
    // finest block of a lattice node -> LUT slot: forest descent + contraction map
    const int32_t *child, *cmap, *level_start;
    LevelInfo li;                    // the finest level (multi-GPU: the rank's rows)
    int64_t lut_cap;                 // slots the LUT holds
    float *lengths;
    int4 *band;        // band candidates (face, slot, i | j<<16, k | r<<16)
    int32_t *n_band;   // [0] count (may exceed cap), [1] overflow flag
    int64_t band_cap;
    double dx, eps, eps_par, inv_dx;
    double len[3];     // domain lengths: faces whose AABB misses [0, l]^3 have no bins, hence no links
    float epsL, dthr;  // eps in cells; the FP32 c.n threshold of the exact parallel test (host-set)
    int bx, by, cells[3];
    int fast;  // eps >> FP64 rounding of the piercing point: fast path allowed
    int pow2;  // dx is a power of two: q = dd * (1/dx) is exactly dd / dx
    // MODE 2 (line enumeration ahead of the grid): piercing-line records
    // (face, R | fast << 4 | (n_nodes - 1) << 5 | ip_lo << 8, m1, m2), and the
    // faces whose lines overflowed the buffer (redone by k_links later)
    int4 *lines;
    int32_t *n_lines;     // may exceed line_cap
    int64_t line_cap;
    int32_t *ovf_list, *n_ovf;
    uint32_t *ovf_bits;   // one bit per face: already listed
    unsigned long long *n_tests;  // lattice lines classified (FP32 intersection tests; roofline ops)
    int32_t *pcnt;                // links per finest parent key (the LUT buckets), counted at conversion
    int3 pdim;                    // parent-key grid
};

// LUT slot of the finest block holding lattice node (i, j, k); -1: not
// mapped (no finest block there, not a boundary block, another rank's row,
// or N_b beyond the LUT capacity).  The forest descent costs L_max dependent
// loads: only the rare exact paths and the SPEC-op / sharded cut links use it.
__device__ __forceinline__ int32_t slot_at(const LinkCtx &c, int i, int j, int k) {
    const int L = c.li.level;
    const int bi = i >> 2, bj = j >> 2, bk = k >> 2;
    if (!owns_row(c.li, bj, bk)) return -1;
    const int3 nb0 = make_int3(c.li.bins[0] >> L, c.li.bins[1] >> L, c.li.bins[2] >> L);
    const int32_t b = block_of_key(L, bi, bj, bk, nb0, c.child, c.level_start[VF_MAX_LEVELS]);
    if (b < 0) return -1;
    const int32_t slot = c.cmap[b];
    return slot < c.lut_cap ? slot : -1;
}

// add a per-thread count to the global test counter, one atomic per warp
__device__ __forceinline__ void add_tests(const LinkCtx &c, unsigned long long n) {
    if (!c.n_tests) return;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if ((threadIdx.x & 31) == 0 && n) atomicAdd(c.n_tests, n);
}

// representative directions q = 2r+1 (lattice.py order) in constant memory
__constant__ int8_t c_rep[13][3] = {
    {1, 0, 0},  {0, 1, 0},  {0, 0, 1},   {1, 1, 0},  {1, 0, 1},  {1, 0, -1}, {1, -1, 0},
    {0, 1, 1},  {0, 1, -1}, {1, 1, 1},   {1, 1, -1}, {1, -1, 1}, {1, -1, -1}};

template <typename T>
__device__ __forceinline__ T pick3(int a, T x, T y, T z) {
    return a == 0 ? x : (a == 1 ? y : z);
}

// Per (face, direction pair) state of the lattice-line enumeration.  Each
// lane builds the state of its own face for the warp-uniform direction pair,
// publishes it in shared memory, and the lattice ROWS of all 32 faces'
// projected bounding boxes are then processed as one flattened work list, 32
// rows per step (per-face loops left 10 of 32 lanes active).
struct LinkDir {
    double off1, off2, vp, den;  // lattice offsets, v1_p, exact c.n
    float P1a, P1b, P2a, P2b;    // projected triangle relative to v1
    float t0, t1, t2, sg;        // edge margins, orientation
    float nq1, nq2, dn, wid0;    // crossing estimate
    int m1a, m1b, m2a, f;        // lattice box, face id
    int lop, hip, fast, pad;     // fallback node range along p, fast path allowed
};

// per-warp shared state: the 32 faces (loaded once, read by every direction
// pair) and their per-pair enumeration state
struct LinkWarp {
    LinkDir d[32];
    double fv[32][6];   // v1 and n of the lane's face (FP64)
    float ff[32][10];   // nf, V1 = v2 - v1, V2 = v3 - v1 (FP32), Ef
    short lohi[32][6];  // fallback node range per axis (cells <= 32767)
    int excl[32];       // exclusive prefix of the per-lane row counts
    int4 lq[96];        // lines that pierce a face: (owner lane | class << 8, m1, m2, Ra bits)
    int lqn;
};
constexpr int kLineQ = 96;

// Exact accept of one node without the eps-box SAT (the FAST path).  Only
// used for lines that pass through the projected triangle with a margin of
// tol (>= 1e-5 (ext + dx), >> the FP32 error of the edge functions) and a
// well-conditioned crossing: the true piercing point is then an interior
// point of the face, its FP64 image lies within ~1e-16 of it, and the
// eps = 1e-9 cube around it overlaps the face on every SAT axis with slack
// eps |axis| >> the FP64 rounding of the test -- the reference SAT
// (geometry.py:441-500) accepts.  num, den, d, the (0, dx] range and q are
// bit-identical to link_candidate / orc_link_lengths.
__device__ __forceinline__ void link_fast(const LinkCtx &c, const double *fv, int r, double den,
                                          int i, int j, int k, int32_t slot) {
    const double dx = c.dx;
    const double x = node_c(i, dx), y = node_c(j, dx), z = node_c(k, dx);
    const double d = VF_DDIV(plane_num(fv, fv + 3, x, y, z), den);
    const bool pos = d > 0.0;
    const double dd = pos ? d : -d;
    if (!(dd > 0.0 && dd <= dx)) return;
    const int q = pos ? 2 * r + 1 : 2 * r + 2;
    // dx = 2^-k: dd * 2^k is exact, hence equal to the correctly rounded dd/dx
    const double qd = c.pow2 ? VF_DMUL(dd, c.inv_dx) : VF_DDIV(dd, dx);
    const float qv = __double2float_rn(qd);
    const int t = (i & 3) + 4 * (j & 3) + 16 * (k & 3);
    atomicMin(reinterpret_cast<unsigned int *>(c.lengths) + ((int64_t)slot * 27 + q) * 64 + t,
              __float_as_uint(qv));
}

// |c| of the 13 representative directions: sqrt(1), sqrt(2), sqrt(3), the
// correctly rounded doubles __dsqrt_rn produces (link_candidate's cn)
__constant__ double c_cn[13] = {1.0, 1.0, 1.0, 1.4142135623730951, 1.4142135623730951,
                                1.4142135623730951, 1.4142135623730951, 1.4142135623730951,
                                1.4142135623730951, 1.7320508075688772, 1.7320508075688772,
                                1.7320508075688772, 1.7320508075688772};

// c_k n_k for c_k in {-1, 0, 1}: exactly DMUL(c_k, n_k) up to the sign of a
// zero product, which cannot change a nonzero sum (a zero den is rejected)
__device__ __forceinline__ double cmul(int ck, double nk) { return ck == 0 ? 0.0 : (ck > 0 ? nk : -nk); }

// state of (lane's face, pair R); returns the number of lattice rows of the
// projected bounding box (0: no link of this face in this pair)
template <int MODE>
__device__ __forceinline__ int link_dir_setup(LinkDir &D, const LinkCtx &c, const double *v,
                                              const float *ff, const short *lohi, int R, int p,
                                              int q1, int q2, int s1, int s2) {
    const double *n = v + 3;
    const float *nf = ff, *V1 = ff + 3, *V2 = ff + 6;
    const int cx = c_rep[R][0], cy = c_rep[R][1], cz = c_rep[R][2];
    const float dn = (float)cx * nf[0] + (float)cy * nf[1] + (float)cz * nf[2];  // c.n in FP32
    // exact den / EPS_PARALLEL (link_candidate): a face parallel to c has no
    // link in this direction pair at all.  The enumeration (MODE 2) never
    // uses den itself: it decides exactly only when the FP32 c.n is near 0.
    double den = 0.0;
    if (MODE != 2 || !(fabsf(dn) > (float)(2.0 * c.eps_par * 1.7320508075688772) + 1e-5f)) {
        den = VF_DADD(VF_DADD(cmul(cx, n[0]), cmul(cy, n[1])), cmul(cz, n[2]));
        if (fabs(den) < VF_DMUL(c.eps_par, c_cn[R])) return 0;
    }
    const double dx = c.dx;
    const float dxf = (float)dx;
    const float V1p = pick3(p, V1[0], V1[1], V1[2]), V2p = pick3(p, V2[0], V2[1], V2[2]);
    const float P1a = pick3(q1, V1[0], V1[1], V1[2]) - (float)s1 * V1p;
    const float P1b = pick3(q2, V1[0], V1[1], V1[2]) - (float)s2 * V1p;
    const float P2a = pick3(q1, V2[0], V2[1], V2[2]) - (float)s1 * V2p;
    const float P2b = pick3(q2, V2[0], V2[1], V2[2]) - (float)s2 * V2p;
    const float ext = fmaxf(fmaxf(fabsf(P1a), fabsf(P1b)), fmaxf(fabsf(P2a), fabsf(P2b)));
    // tolerance: eps-cube acceptance (<= 2 sqrt 6 eps after the oblique
    // projection) + FP32 error of coordinates of magnitude ext + dx, plus an
    // absolute term >= the FP32 rounding of E_k itself (sliver edges)
    const float tol = 1e-5f * (ext + dxf) + 6.0f * (float)c.eps;
    const double vp = pick3(p, v[0], v[1], v[2]);
    // lattice of line traces: coordinate j of the trace of the line through
    // node (i_p, i_q1, i_q2) is ((i_qj - s_j i_p) + delta_j) dx + s_j v1_p,
    // delta_j = (1 - s_j)/2; relative to v1: subtract v1_qj
    const double off1 = (double)s1 * vp - pick3(q1, v[0], v[1], v[2]);
    const double off2 = (double)s2 * vp - pick3(q2, v[0], v[1], v[2]);
    const double d1 = 0.5 * (1 - s1), d2 = 0.5 * (1 - s2);
    const float bmin1 = fminf(fminf(0.0f, P1a), P2a) - tol, bmax1 = fmaxf(fmaxf(0.0f, P1a), P2a) + tol;
    const float bmin2 = fminf(fminf(0.0f, P1b), P2b) - tol, bmax2 = fmaxf(fmaxf(0.0f, P1b), P2b) + tol;
    const double inv = c.inv_dx;
    const int m1a = (int)ceil(((double)bmin1 - off1) * inv - d1 - 1e-6);
    const int m1b = (int)floor(((double)bmax1 - off1) * inv - d1 + 1e-6);
    if (m1b < m1a) return 0;
    const int m2a = (int)ceil(((double)bmin2 - off2) * inv - d2 - 1e-6);
    const int m2b = (int)floor(((double)bmax2 - off2) * inv - d2 + 1e-6);
    if (m2b < m2a) return 0;
    // (a degenerate projection -- face parallel to c -- keeps only lattice
    // points within tol of the projected segment: the edge tests stay valid)
    const float cr = P1a * P2b - P1b * P2a;
    const float ab = 4e-6f * (ext + dxf) * (ext + dxf);
    D.P1a = P1a; D.P1b = P1b; D.P2a = P2a; D.P2b = P2b;
    // edge margins with the L1 length |a| + |b| >= |e| (no square root; a
    // larger margin only moves lines into the exactly-decided band)
    D.t0 = tol * (fabsf(P1a) + fabsf(P1b)) * 1.0001f + ab;
    D.t1 = tol * (fabsf(P2a - P1a) + fabsf(P2b - P1b)) * 1.0001f + ab;
    D.t2 = tol * (fabsf(P2a) + fabsf(P2b)) * 1.0001f + ab;
    D.sg = cr >= 0.0f ? 1.0f : -1.0f;
    const bool steep = fabsf(dn) >= 1e-3f;
    D.off1 = off1; D.off2 = off2; D.vp = vp; D.den = den;
    D.nq1 = pick3(q1, nf[0], nf[1], nf[2]);
    D.nq2 = pick3(q2, nf[0], nf[1], nf[2]);
    D.dn = steep ? dn : 0.0f;  // 0: ill-conditioned crossing, full node range
    D.wid0 = steep ? dxf * (1.0f + 1e-4f) + 1e-5f * dxf + __fdividef(ff[9], fabsf(dn)) * 1.0001f : 0.0f;
    D.m1a = m1a; D.m1b = m1b; D.m2a = m2a;
    D.lop = pick3(p, lohi[0], lohi[1], lohi[2]);
    D.hip = pick3(p, lohi[3], lohi[4], lohi[5]);
    D.fast = steep && c.fast;
    return m2b - m2a + 1;
}

// a candidate the fast path cannot decide: appended to the band list for
// k_links_band (MODE 1: decided inline -- the overflow fallback kernel; MODE 2
// appends with slot -1: the block map does not exist yet, k_links_band looks it up)
template <int MODE>
__device__ __forceinline__ void link_slow(const LinkCtx &c, int f, int slot, int i, int j, int k,
                                          int r) {
    if (MODE == 1) {
        link_candidate(c.faces, f, r, i, j, k, c.dx, c.eps, c.eps_par, slot, c.lengths);
        return;
    }
    const int pos = atomicAdd(&c.n_band[0], 1);
    if (pos < c.band_cap) c.band[pos] = make_int4(f, slot, i | (j << 16), k | (r << 16));
    else c.n_band[1] = 1;  // the fallback kernel redoes every face inline
}

// the (2, rarely 3) nodes of one line that pierces the face: crossing
// estimate, then the fast exact path (interior lines) or link_slow (margin
// band, ill-conditioned crossings)
// node range along p of the line through (Ra, Rb): the nodes within one link
// of its crossing with the face plane (crossing estimate in FP32, widened
// past its error), or the face's full range for ill-conditioned crossings
__device__ __forceinline__ void line_nodes(const LinkCtx &c, const LinkDir &D, float Ra, float Rb,
                                           int cp, int &ip_lo, int &ip_hi) {
    // crossing with the face plane: Q = v1 + Ra e_q1 + Rb e_q2 (+0 e_p),
    // points Q + lam c; n.(Q + lam c - v1) = 0
    ip_lo = D.lop;
    ip_hi = D.hip;
    if (D.dn != 0.0f) {
        const float lam = -__fdividef(D.nq1 * Ra + D.nq2 * Rb, D.dn);
        const float xs = (float)cp * lam;  // x_p* - v1_p
        const float wid = D.wid0 + 1.0001e-6f * __fdividef(fabsf(xs), fabsf(D.dn));
        // node index i_p with |x_p* - (i_p + 0.5) dx| <= dx
        ip_lo = max((int)ceil(((double)(xs - wid) + D.vp) * c.inv_dx - 0.5), ip_lo);
        ip_hi = min((int)floor(((double)(xs + wid) + D.vp) * c.inv_dx - 0.5), ip_hi);
    }
}

template <int MODE>
__device__ __forceinline__ void link_line(const LinkCtx &c, const LinkDir &D, const double *fv,
                                          int m1, int m2, float Ra, float Rb, bool fast, int R,
                                          int p, int cp, int s1, int s2, int n1, int n2) {
    int ip_lo, ip_hi;
    line_nodes(c, D, Ra, Rb, cp, ip_lo, ip_hi);
    if (MODE == 2 && ip_lo <= ip_hi && ip_hi - ip_lo < 8 && fast) {
        // (inline overflow path of the warp queue) record the line
        const int pos = atomicAdd(c.n_lines, 1);
        if (pos < c.line_cap) {
            c.lines[pos] = make_int4(D.f, R | (1 << 4) | ((ip_hi - ip_lo) << 5) | (ip_lo << 8), m1, m2);
        } else {
            const uint32_t bit = 1u << (D.f & 31);
            if (!(atomicOr(&c.ovf_bits[D.f >> 5], bit) & bit)) c.ovf_list[atomicAdd(c.n_ovf, 1)] = D.f;
        }
        return;
    }
    for (int ip = ip_lo; ip <= ip_hi; ++ip) {
        // i_qj = m_j + s_j i_p
        const int a = m1 + s1 * ip, b = m2 + s2 * ip;
        if (a < 0 || a >= n1 || b < 0 || b >= n2) continue;
        const int i = p == 0 ? ip : a;
        const int j = p == 1 ? ip : (p == 0 ? a : b);
        const int k = p == 2 ? ip : b;
        if (MODE == 2) {  // margin band / ill-conditioned lines: exact path later
            link_slow<MODE>(c, D.f, -1, i, j, k, R);
            continue;
        }
        const int32_t slot = slot_at(c, i, j, k);
        if (slot < 0) continue;
        if (fast) link_fast(c, fv, R, D.den, i, j, k, slot);
        else link_slow<MODE>(c, D.f, slot, i, j, k, R);
    }
}

// Lines found by the row scans are queued per warp and resolved 32 at a time
// (one line per lane): the row / point loops leave few lanes active, the node
// work (bmap lookup, FP64 num/den, atomicMin) then runs on full warps.  The
// queue is drained before the next pair overwrites the per-lane LinkDir.
template <int MODE>
__device__ __forceinline__ void line_drain(LinkWarp &W, int lane, const LinkCtx &c, bool all, int R,
                                           int p, int cp, int s1, int s2, int n1, int n2) {
    __syncwarp();
    int n = min(W.lqn, kLineQ);
    while (n >= 32 || (all && n > 0)) {
        const int take = min(n, 32);
        int4 e = make_int4(0, 0, 0, 0);
        if (lane < take) e = W.lq[n - take + lane];
        __syncwarp();
        if (MODE == 2) {
            // enumeration: record the line (warp-aggregated slot in the
            // global line buffer); margin-band / long-range lines go to the
            // band list node by node
            bool want = false;
            int4 rec = make_int4(0, 0, 0, 0);
            if (lane < take) {
                const int o = e.x & 31;
                const LinkDir &D = W.d[o];
                const float Rb = (float)(((double)e.z + 0.5 * (1 - s2)) * c.dx + D.off2);
                const bool fast = (e.x >> 8) & 1;
                int ip_lo, ip_hi;
                line_nodes(c, D, __int_as_float(e.w), Rb, cp, ip_lo, ip_hi);
                if (fast && ip_lo <= ip_hi && ip_hi - ip_lo < 8) {
                    want = true;
                    rec = make_int4(D.f, R | (1 << 4) | ((ip_hi - ip_lo) << 5) | (ip_lo << 8), e.y, e.z);
                } else {
                    link_line<MODE>(c, D, W.fv[o], e.y, e.z, __int_as_float(e.w), Rb, fast, R, p, cp, s1,
                                    s2, n1, n2);
                }
            }
            const uint32_t m = __ballot_sync(0xffffffffu, want);
            int base = 0;
            if (lane == 0 && m) base = atomicAdd(c.n_lines, __popc(m));
            base = __shfl_sync(0xffffffffu, base, 0);
            if (want) {
                const int pos = base + __popc(m & ((1u << lane) - 1u));
                if (pos < c.line_cap) {
                    c.lines[pos] = rec;
                } else {
                    const uint32_t bit = 1u << (rec.x & 31);
                    if (!(atomicOr(&c.ovf_bits[rec.x >> 5], bit) & bit)) c.ovf_list[atomicAdd(c.n_ovf, 1)] = rec.x;
                }
            }
        } else if (lane < take) {
            const int o = e.x & 31;
            const LinkDir &D = W.d[o];
            const float Rb = (float)(((double)e.z + 0.5 * (1 - s2)) * c.dx + D.off2);
            link_line<MODE>(c, D, W.fv[o], e.y, e.z, __int_as_float(e.w), Rb, (e.x >> 8) & 1, R, p, cp,
                            s1, s2, n1, n2);
        }
        n -= take;
    }
    __syncwarp();
    if (lane == 0) W.lqn = n;
    __syncwarp();
}

// inside test of the line through (Ra, Rb): 0 misses the face, 1 interior
// with margin and fast path allowed, 2 undecided (exact path with the SAT)
__device__ __forceinline__ int point_class(const LinkDir &D, float Ra, float Rb) {
    const float sg = D.sg;
    const float E0 = sg * (D.P1a * Rb - D.P1b * Ra);
    const float E1 = sg * ((D.P2a - D.P1a) * (Rb - D.P1b) - (D.P2b - D.P1b) * (Ra - D.P1a));
    const float E2 = sg * (D.P2b * Ra - D.P2a * Rb);
    if (E0 < -D.t0 || E1 < -D.t1 || E2 < -D.t2) return 0;
    return (D.fast && E0 >= D.t0 && E1 >= D.t1 && E2 >= D.t2) ? 1 : 2;
}

// one lattice point (line) of a row: inside test; a piercing line is queued
// (or, when the queue is full, resolved inline)
template <int MODE>
__device__ __forceinline__ void link_point(LinkWarp &W, int o, const LinkCtx &c, const LinkDir &D,
                                           const double *fv, int m1, int m2, float Rb, int R, int p,
                                           int cp, int s1, int s2, int n1, int n2) {
    const float Ra = (float)(((double)m1 + 0.5 * (1 - s1)) * c.dx + D.off1);
    const int cls = point_class(D, Ra, Rb);
    if (cls == 0) return;  // misses the face
    const bool fast = MODE != 1 && cls == 1;
    const int pos = atomicAdd(&W.lqn, 1);
    if (pos < kLineQ) W.lq[pos] = make_int4(o | ((int)fast << 8), m1, m2, __float_as_int(Ra));
    else link_line<MODE>(c, D, fv, m1, m2, Ra, Rb, fast, R, p, cp, s1, s2, n1, n2);
}

// one lattice row m2: the conservative m1 interval of the row inside the
// margin-widened triangle (scanline; each edge function is linear in Ra,
// E_k = alpha_k Ra + beta_k >= -t_k), then its points.  An edge whose bound
// is ill-conditioned (|alpha_k| tiny) does not restrict the row; the interval
// is widened by one lattice point on each side -- a superset of the points
// that pass link_point's own test, which alone decides.
__device__ __forceinline__ bool row_interval(const LinkCtx &c, const LinkDir &D, float Rb, int s1,
                                             int &m1lo, int &m1hi) {
    const float sg = D.sg;
    const float al[3] = {-sg * D.P1b, -sg * (D.P2b - D.P1b), sg * D.P2b};
    const float be[3] = {sg * D.P1a * Rb, sg * ((D.P2a - D.P1a) * (Rb - D.P1b) + (D.P2b - D.P1b) * D.P1a),
                         -sg * D.P2a * Rb};
    const float tk[3] = {D.t0, D.t1, D.t2};
    const float dxf = (float)c.dx;
    // magnitude bound of the products in beta_k (FP32 error <~ 3e-7 M)
    const float sP = fabsf(D.P1a) + fabsf(D.P1b) + fabsf(D.P2a) + fabsf(D.P2b);
    const float M = sP * (fabsf(Rb) + sP);
    float lo = -INFINITY, hi = INFINITY;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const float a = al[k], rhs = -tk[k] - be[k];
        if (1e-5f * (M + tk[k]) >= 0.25f * dxf * fabsf(a)) {
            // (near-)parallel edge: the row is either fully out or unrestricted
            if (a == 0.0f && be[k] < -tk[k] - 1e-5f * (M + tk[k])) return false;
            continue;
        }
        const float b = __fdividef(rhs, a);  // ~2 ulp: the bound is padded by a lattice step
        if (a > 0.0f) lo = fmaxf(lo, b);
        else hi = fminf(hi, b);
    }
    const double d1 = 0.5 * (1 - s1);
    m1lo = D.m1a;
    m1hi = D.m1b;
    if (lo > -INFINITY) m1lo = max(m1lo, (int)ceil(((double)lo - D.off1) * c.inv_dx - d1) - 1);
    if (hi < INFINITY) m1hi = min(m1hi, (int)floor(((double)hi - D.off1) * c.inv_dx - d1) + 1);
    return m1lo <= m1hi;
}

// one lattice row m2: the conservative m1 interval of the row inside the
// margin-widened triangle (scanline; each edge function is linear in Ra,
// E_k = alpha_k Ra + beta_k >= -t_k), then its points.  An edge whose bound
// is ill-conditioned (|alpha_k| tiny) does not restrict the row; the interval
// is widened by one lattice point on each side -- a superset of the points
// that pass point_class, which alone decides.
template <int MODE>
__device__ __forceinline__ int link_row(LinkWarp &W, int o, const LinkCtx &c, const LinkDir &D,
                                         const double *fv, int m2, int R, int p, int cp, int s1,
                                         int s2, int n1, int n2) {
    const float Rb = (float)(((double)m2 + 0.5 * (1 - s2)) * c.dx + D.off2);
    int m1lo, m1hi;
    if (!row_interval(c, D, Rb, s1, m1lo, m1hi)) return 0;
    for (int m1 = m1lo; m1 <= m1hi; ++m1)
        link_point<MODE>(W, o, c, D, fv, m1, m2, Rb, R, p, cp, s1, s2, n1, n2);
    return m1hi - m1lo + 1;
}

constexpr size_t kLinkSmem = kLinkWarps * sizeof(LinkWarp);

// K-link.  MODE 0: the main kernel (fast path + band list); MODE 2: the
// grid-independent line enumeration (k_links_enum, records piercing lines);
// MODE 1:
// the overflow fallback, a no-op unless the band list overflowed, in which
// case it redoes every face with every undecided candidate decided inline
// (atomicMin is idempotent, so re-merging the fast results is harmless).
template <int MODE>
__global__ void __launch_bounds__(kLinkWarps * 32, MODE == 1 ? 1 : VF_LINK_MINB)
    k_links(LinkCtx c, int widen, int64_t F, const int32_t *__restrict__ map,
            const int32_t *__restrict__ d_n_map) {
    if (MODE == 1 && c.n_band[1] == 0) return;
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    LinkWarp &W = reinterpret_cast<LinkWarp *>(s_raw)[w];
    const int64_t n = d_n_map ? (int64_t)*d_n_map : F;
    if (lane == 0) W.lqn = 0;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // all lanes of a warp iterate together (uniform trip count); lanes past
    // the end are inactive
    const int64_t first = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    unsigned long long tests = 0;
    for (int64_t base = first; base < n; base += stride) {
        const int64_t m = base + lane;
        bool active = m < n;
        int f = 0;
        __syncwarp();
        if (active) {
            f = map ? map[m] : (int)m;
            double v[9], nn[3];
            load_face(c.faces, f, v, nn);
            double ext = 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                W.fv[lane][d] = v[d];
                W.fv[lane][3 + d] = nn[d];
                W.ff[lane][d] = (float)nn[d];
                W.ff[lane][3 + d] = (float)(v[3 + d] - v[d]);
                W.ff[lane][6 + d] = (float)(v[6 + d] - v[d]);
                const double flo = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
                const double fhi = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
                ext = fmax(ext, fhi - flo);
                if (fhi < 0.0 || flo > c.len[d]) active = false;  // in no bin (A5), no links
                // nodes within one link of the face AABB (fallback range)
                W.lohi[lane][d] = (short)max((int)floor((flo - c.dx - 2.0 * c.eps) * c.inv_dx - 0.5) - widen, 0);
                W.lohi[lane][3 + d] =
                    (short)min((int)floor((fhi + c.dx + 2.0 * c.eps) * c.inv_dx - 0.5) + 1 + widen, c.cells[d] - 1);
            }
            W.ff[lane][9] = 4e-6f * (float)(ext + 2.0 * c.dx);

        }
        __syncwarp();
#pragma unroll 1
        for (int R = 0; R < 13; ++R) {
            // warp-uniform axis bookkeeping of the pair
            const int cx = c_rep[R][0], cy = c_rep[R][1], cz = c_rep[R][2];
            const int p = cx != 0 ? 0 : (cy != 0 ? 1 : 2);
            const int q1 = p == 0 ? 1 : 0, q2 = p == 2 ? 1 : 2;
            const int cp = pick3(p, cx, cy, cz);
            const int s1 = pick3(q1, cx, cy, cz) * cp, s2 = pick3(q2, cx, cy, cz) * cp;
            const int n1 = pick3(q1, c.cells[0], c.cells[1], c.cells[2]);
            const int n2 = pick3(q2, c.cells[0], c.cells[1], c.cells[2]);
            int cnt = 0;
            if (active) {
                LinkDir D;
                D.f = f;
                cnt = link_dir_setup<MODE>(D, c, W.fv[lane], W.ff[lane], W.lohi[lane], R, p, q1, q2, s1, s2);
                if (cnt) W.d[lane] = D;
            }
            // warp exclusive prefix of the row counts
            int inc = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int t = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += t;
            }
            const int total = __shfl_sync(0xffffffffu, inc, 31);
            W.excl[lane] = inc - cnt;
            __syncwarp();
            for (int b0 = 0; b0 < total; b0 += 32) {
                const int it = b0 + lane;
                if (it < total) {
                    int o = 0;  // owner lane: largest o with excl[o] <= it
#pragma unroll
                    for (int st = 16; st > 0; st >>= 1)
                        if (W.excl[o + st] <= it) o += st;
                    const LinkDir &D = W.d[o];
                    tests += link_row<MODE>(W, o, c, D, W.fv[o], D.m2a + it - W.excl[o], R, p, cp, s1, s2, n1, n2);
                }
                line_drain<MODE>(W, lane, c, false, R, p, cp, s1, s2, n1, n2);
            }
            line_drain<MODE>(W, lane, c, true, R, p, cp, s1, s2, n1, n2);
        }
    }
    if (MODE == 2) add_tests(c, tests);
}

// ---- small faces: thread per face ----------------------------------------
// At the north-star resolution most faces are smaller than a cell (C4: ~1.3
// piercing lines per face over all 13 pairs), so the warp-flattened row lists
// above spend their time on bookkeeping.  Faces whose bounding box spans at
// most g_small_ext cells are enumerated here one per thread, in lattice-local
// FP32: lengths in units of dx, relative to v1, with v1 = (b + w + 1/2) dx for
// the node b = floor(v1/dx - 1/2) and w in [0, 1).  The trace of the line
// through node b + I (pair R: p, q1, q2, s_j = c_qj c_p) in the plane
// x_p = v1_p is then (M1 + o1, M2 + o2), M_j = I_qj - s_j I_p, o_j = s_j w_p -
// w_qj -- the same quantities link_dir_setup / link_point form in absolute
// FP64/FP32 coordinates, scaled by 1/dx, with smaller rounding (magnitudes of
// a few cells); the margins t_k, tol, the crossing estimate and the node range
// are the same formulas in these units, so the accept / undecided / miss
// classes remain conservative and the recorded lines, band candidates and
// hence the LUT are identical.  Larger faces are appended to a list for the
// warp-flattened kernel.
#ifndef VF_SMALL_MINB
#define VF_SMALL_MINB 8
#endif
static float g_small_ext = 1.5f;  // vf_set_link_small_ext (test / tuning hook)

__device__ __forceinline__ void line_store(const LinkCtx &c, int pos, int4 rec) {
    if (pos < c.line_cap) {
        c.lines[pos] = rec;
    } else {  // buffer full: the direct kernel redoes the face after the tables
        const uint32_t bit = 1u << (rec.x & 31);
        if (!(atomicOr(&c.ovf_bits[rec.x >> 5], bit) & bit)) c.ovf_list[atomicAdd(c.n_ovf, 1)] = rec.x;
    }
}

// lines are staged per CTA in shared memory and written with ONE global slot
// reservation per CTA (a per-warp-per-pair atomicAdd on the shared line
// counter was the kernel's top stall); a full stage falls back to direct slots
#ifndef VF_SMALL_THREADS
#define VF_SMALL_THREADS 128
#endif
constexpr int kLineStage = 4 * VF_SMALL_THREADS;

__device__ __forceinline__ void stage_put(const LinkCtx &c, int4 *st, int pos, int4 rec) {
    if (pos < kLineStage) st[pos] = rec;
    else line_store(c, atomicAdd(c.n_lines, 1), rec);
}

__device__ __forceinline__ int4 qrec_convert(const LinkCtx &c, const int4 rec);

__device__ __forceinline__ void qrec_entry(const int4 rec, int k, int &i, int &j, int &kk, int &q, int &t) {
    const int bi = rec.x & 0x7fff, bj = (rec.x >> 15) & 0x7fff, bk = rec.y & 0x7fff, R = (rec.y >> 15) & 15;
    const uint32_t cd = ((uint32_t)rec.y >> (21 + 4 * k)) & 15u;
    const int o = cd & 7;
    i = bi + o * c27(2 * R + 1, 0);
    j = bj + o * c27(2 * R + 1, 1);
    kk = bk + o * c27(2 * R + 1, 2);
    q = (cd >> 3) ? 2 * R + 2 : 2 * R + 1;
    t = (i & 3) + 4 * (j & 3) + 16 * (kk & 3);
}

// a link's parent bucket key and its bucket entry octant << 41 | (q 64 + t)
// << 30 | q bits (q in (0, 1]: 30 bits)
__device__ __forceinline__ int32_t link_bucket_entry(const int4 rec, int k, int3 pdim, unsigned long long &x) {
    int i, j, kk, q, t;
    qrec_entry(rec, k, i, j, kk, q, t);
    const int oct = ((i >> 2) & 1) + 2 * ((j >> 2) & 1) + 4 * ((kk >> 2) & 1);
    x = ((unsigned long long)oct << 41) | ((unsigned long long)(q * 64 + t) << 30) | (uint32_t)(k ? rec.w : rec.z);
    return (i >> 3) + pdim.x * ((j >> 3) + pdim.y * (kk >> 3));
}

// count the links of a q-record into their parent buckets (warp-aggregated
// over the active lanes: neighbouring records mostly share parents)
__device__ __forceinline__ void count_qrec(const LinkCtx &c, const int4 rec) {
    const int ne = (rec.y >> 19) & 3;
#pragma unroll
    for (int k = 0; k < 2; ++k) {
        unsigned long long x;
        const int32_t key = k < ne ? link_bucket_entry(rec, k, c.pdim, x) : -1;
        const uint32_t grp = __match_any_sync(__activemask(), key);
        if (key >= 0 && (threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&c.pcnt[key], __popc(grp));
    }
}

// ---- small faces: thread per face, queued -----------------------------------
// Faces smaller than ~1.5 cells (the north-star resolution: ~1.3 piercing
// lines per face over all 13 pairs) are enumerated in lattice-local FP32:
// lengths in units of dx, relative to v1, with v1 = (b + w + 1/2) dx for the
// node b = floor(v1/dx - 1/2) and w in [0, 1).  The trace of the line through
// node b + I (pair R: p, q1, q2, s_j = c_qj c_p) in the plane x_p = v1_p is
// then (M1 + o1, M2 + o2), M_j = I_qj - s_j I_p, o_j = s_j w_p - w_qj -- the
// quantities link_dir_setup / link_point form in absolute FP64/FP32
// coordinates, scaled by 1/dx, with smaller rounding; the margins t_k, tol,
// the crossing estimate and the node range are the same formulas in these
// units, so the miss / interior / band classes remain conservative and the
// recorded lines, band candidates and hence the LUT are identical.  Larger
// faces go to the warp-flattened kernel.  Two phases per warp, so the
// expensive part runs on full warps:
//   phase 1 (lane = face): the face's lattice-local FP32 frame into shared
//     memory, then the 13 pairs' lattice boxes (the projected triangle
//     widened by tol); the (face, pair) items with a lattice point in their
//     box are appended to the warp's queue (~30% of the items at C4);
//   phase 2 (lane = item): the queued items, 32 at a time: the pair's
//     EPS_PARALLEL test, edge margins, lattice points (miss / interior /
//     band), line records and band candidates.
// With a lane per face (round 1) the point loop ran on the ~30% of lanes
// whose pair had points while the rest idled through it (C4: 0.98 -> 0.81 ms).
struct QFace {                      // one face of the warp, lattice-local
    float V1[3], V2[3], w[3], nf[3];
    int b[3];
    short lo[3], hi[3];
    float ff9;
    int f;
};
struct QWarp {
    QFace fc[32];
    uint16_t q[32 * 13];            // items: lane | idx << 5 (idx = class-major pair index 0..12)
    int qn;
};

// pair index -> (class, s1, s2, R) from packed immediates (2 bits per pair
// for the class, s1 + 1 and s2 + 1; 4 bits for R in lattice.py order):
// idx 0..8 class 0 (s1, s2) = (t / 3 - 1, t % 3 - 1), 9..11 class 1
// (0, t - 1), 12 class 2 (0, 0)
__device__ __forceinline__ void pair_of(int idx, int &cls, int &s1, int &s2, int &R) {
    cls = (int)((0x2540000u >> (2 * idx)) & 3u);
    s1 = (int)((0x156a540u >> (2 * idx)) & 3u) - 1;
    s2 = (int)((0x1924924u >> (2 * idx)) & 3u) - 1;
    R = (int)((0x271893a405b6cull >> (4 * idx)) & 15);
}

// the class projection (p, q1, q2) of a queued face (small_project, from shared memory)
struct QProj {
    float V1p, V1a, V1b, V2p, V2a, V2b, wp, wa, wb, nfp, nfa, nfb;
    int bp, ba, bb, lop, hip, n1, n2;
};
__device__ __forceinline__ void qproject(const LinkCtx &c, const QFace &F, int cls, QProj &P) {
    const int p = cls, q1 = cls == 0 ? 1 : 0, q2 = cls == 2 ? 1 : 2;
    P.V1p = F.V1[p]; P.V1a = F.V1[q1]; P.V1b = F.V1[q2];
    P.V2p = F.V2[p]; P.V2a = F.V2[q1]; P.V2b = F.V2[q2];
    P.wp = F.w[p]; P.wa = F.w[q1]; P.wb = F.w[q2];
    P.nfp = F.nf[p]; P.nfa = F.nf[q1]; P.nfb = F.nf[q2];
    P.bp = F.b[p]; P.ba = F.b[q1]; P.bb = F.b[q2];
    P.lop = F.lo[p]; P.hip = F.hi[p];
    P.n1 = pick3(q1, c.cells[0], c.cells[1], c.cells[2]);
    P.n2 = pick3(q2, c.cells[0], c.cells[1], c.cells[2]);
}

// the pair's lattice box (the projected triangle widened by tol); false: empty
__device__ __forceinline__ bool qbox(const QProj &P, float epsL, int s1, int s2, float &P1a, float &P1b,
                                     float &P2a, float &P2b, float &ext, float &tol, float &o1, float &o2,
                                     int &m1a, int &m1b, int &m2a, int &m2b) {
    P1a = P.V1a - (float)s1 * P.V1p; P1b = P.V1b - (float)s2 * P.V1p;
    P2a = P.V2a - (float)s1 * P.V2p; P2b = P.V2b - (float)s2 * P.V2p;
    ext = fmaxf(fmaxf(fabsf(P1a), fabsf(P1b)), fmaxf(fabsf(P2a), fabsf(P2b)));
    tol = 1e-5f * (ext + 1.0f) + 6.0f * epsL;
    o1 = (float)s1 * P.wp - P.wa;
    o2 = (float)s2 * P.wp - P.wb;
    m1a = (int)ceilf(fminf(fminf(0.0f, P1a), P2a) - tol - o1 - 1e-4f);
    m1b = (int)floorf(fmaxf(fmaxf(0.0f, P1a), P2a) + tol - o1 + 1e-4f);
    m2a = (int)ceilf(fminf(fminf(0.0f, P1b), P2b) - tol - o2 - 1e-4f);
    m2b = (int)floorf(fmaxf(fmaxf(0.0f, P1b), P2b) + tol - o2 + 1e-4f);
    return m1a <= m1b && m2a <= m2b;
}

__global__ void __launch_bounds__(VF_SMALL_THREADS, VF_SMALL_MINB)
    k_links_smallq(LinkCtx c, int widen, int64_t F, float small_ext, int32_t *__restrict__ big,
                   int32_t *__restrict__ n_big, const int32_t *__restrict__ map,
                   const int32_t *__restrict__ d_n_map) {
    __shared__ int4 s_rec[kLineStage];
    __shared__ int s_n, s_base;
    __shared__ QWarp s_w[VF_SMALL_THREADS / 32];
    const int lane = threadIdx.x & 31;
    QWarp &W = s_w[threadIdx.x >> 5];
    if (threadIdx.x == 0) s_n = 0;
    if (lane == 0) W.qn = 0;
    __syncthreads();
    const int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    // (map: a face subset -- the sharded embed's faces near owned rows)
    bool act = m < (d_n_map ? (int64_t)*d_n_map : F);
    const int f = act && map ? map[m] : (int)m;
    bool small = false;
    QFace &Q = W.fc[lane];
    if (act) {
        double v[9], nn[3], flo[3], fhi[3];
        load_face(c.faces, f, v, nn);
        double ext = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            flo[d] = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
            fhi[d] = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
            ext = fmax(ext, fhi[d] - flo[d]);
            // A5 / face_pairs: a face whose AABB misses the domain is in no
            // bin, so the oracle's per-cell MD-bin scan never sees it
            if (fhi[d] < 0.0 || flo[d] > c.len[d]) act = false;
        }
        const float extL = (float)(ext * c.inv_dx);
        small = act && extL <= small_ext;
        if (small) {
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double t = v[d] * c.inv_dx - 0.5, bd = floor(t);
                Q.b[d] = (int)bd;
                Q.w[d] = (float)(t - bd);
                Q.V1[d] = (float)((v[3 + d] - v[d]) * c.inv_dx);
                Q.V2[d] = (float)((v[6 + d] - v[d]) * c.inv_dx);
                Q.nf[d] = (float)nn[d];
                // nodes within one link of the face AABB (k_links' fallback
                // range), from the lattice-local frame in FP32 and widened by
                // 1e-3 cells (a superset only adds exactly-tested nodes)
                const float mn = fminf(0.0f, fminf(Q.V1[d], Q.V2[d])), mx = fmaxf(0.0f, fmaxf(Q.V1[d], Q.V2[d]));
                Q.lo[d] = (short)max(Q.b[d] + (int)floorf(Q.w[d] + mn - 1.0f - 2.0f * c.epsL - 1e-3f) - widen, 0);
                Q.hi[d] = (short)min(Q.b[d] + (int)floorf(Q.w[d] + mx + 1.0f + 2.0f * c.epsL + 1e-3f) + 1 + widen,
                                     c.cells[d] - 1);
            }
            Q.ff9 = 4e-6f * (extL + 2.0f);
            Q.f = f;
        }
    }
    // large faces: warp-aggregated append to the list of the warp-flattened kernel
    const unsigned bm = __ballot_sync(0xffffffffu, act && !small);
    if (bm) {
        int base = 0;
        if (lane == 0) base = atomicAdd(n_big, __popc(bm));
        base = __shfl_sync(0xffffffffu, base, 0);
        if (act && !small) big[base + __popc(bm & ((1u << lane) - 1u))] = f;
    }
    __syncwarp();
    // phase 1: which of the 13 pairs can have a lattice point.  Per class
    // the box range along q1 depends on s1 only and along q2 on s2 only; with
    // the class's largest tolerance (a bound on every pair's ext) the ranges
    // are supersets of the pairs' exact boxes, so a pair is queued iff both
    // of its axis ranges are non-empty (phase 2 re-derives the exact box).
    unsigned long long tests = 0;
    uint32_t cand = 0;  // bit idx: pair idx may have lattice points
    if (small) {
#pragma unroll
        for (int cls = 0; cls < 3; ++cls) {
            const int p = cls, q1 = cls == 0 ? 1 : 0, q2 = cls == 2 ? 1 : 2;
            const float V1p = Q.V1[p], V2p = Q.V2[p], wp = Q.w[p];
            const float V1a = Q.V1[q1], V2a = Q.V2[q1], wa = Q.w[q1];
            const float V1b = Q.V1[q2], V2b = Q.V2[q2], wb = Q.w[q2];
            // |V_q - s V_p| <= |V_q| + |V_p| for every s in {-1, 0, 1}
            const float extc = fmaxf(fmaxf(fabsf(V1a), fabsf(V2a)), fmaxf(fabsf(V1b), fabsf(V2b))) +
                               fmaxf(fabsf(V1p), fabsf(V2p));
            const float tolc = 1e-5f * (extc + 1.0f) + 6.0f * c.epsL;
            uint32_t okA = 0, okB = 0;  // bit s + 1
#pragma unroll
            for (int sg = -1; sg <= 1; ++sg) {
                if (cls != 0 && sg != 0) continue;  // classes 1, 2: s1 = 0
                const float A1 = V1a - (float)sg * V1p, A2 = V2a - (float)sg * V2p, o = (float)sg * wp - wa;
                if ((int)ceilf(fminf(fminf(0.0f, A1), A2) - tolc - o - 1e-4f) <=
                    (int)floorf(fmaxf(fmaxf(0.0f, A1), A2) + tolc - o + 1e-4f))
                    okA |= 1u << (sg + 1);
            }
#pragma unroll
            for (int sg = -1; sg <= 1; ++sg) {
                if (cls == 2 && sg != 0) continue;  // class 2: s2 = 0
                const float B1 = V1b - (float)sg * V1p, B2 = V2b - (float)sg * V2p, o = (float)sg * wp - wb;
                if ((int)ceilf(fminf(fminf(0.0f, B1), B2) - tolc - o - 1e-4f) <=
                    (int)floorf(fmaxf(fmaxf(0.0f, B1), B2) + tolc - o + 1e-4f))
                    okB |= 1u << (sg + 1);
            }
            const int i0 = cls == 0 ? 0 : (cls == 1 ? 9 : 12);
            const int ns = cls == 0 ? 9 : (cls == 1 ? 3 : 1);
#pragma unroll
            for (int t = 0; t < ns; ++t) {
                const int s1 = cls == 0 ? t / 3 - 1 : 0;
                const int s2 = cls == 0 ? t % 3 - 1 : (cls == 1 ? t - 1 : 0);
                cand |= ((okA >> (s1 + 1)) & (okB >> (s2 + 1)) & 1u) << (i0 + t);
            }
        }
    }
    {  // the warp's items: one exclusive scan of the per-lane counts
        const int cnt = __popc(cand);
        int inc = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += y;
        }
        int pos = inc - cnt;
        for (uint32_t mm = cand; mm; mm &= mm - 1) W.q[pos++] = (uint16_t)(lane | ((__ffs(mm) - 1) << 5));
        if (lane == 31) W.qn = inc;
        __syncwarp();
    }
    // phase 2: the queued items on full warps
    const int nq = W.qn;
    for (int i0 = 0; i0 < nq; i0 += 32) {
        if (i0 + lane >= nq) continue;
        const uint32_t it = W.q[i0 + lane];
        const QFace &Fq = W.fc[it & 31];
        int cls, s1, s2, R;
        pair_of((int)(it >> 5), cls, s1, s2, R);
        QProj P;
        qproject(c, Fq, cls, P);
        float P1a, P1b, P2a, P2b, ext, tol, o1, o2;
        int m1a, m1b, m2a, m2b;
        qbox(P, c.epsL, s1, s2, P1a, P1b, P2a, P2b, ext, tol, o1, o2, m1a, m1b, m2a, m2b);
        tests += (unsigned long long)((m2b - m2a + 1) * (m1b - m1a + 1));
        // exact den / EPS_PARALLEL (link_dir_setup): only where the FP32 c.n is near 0
        const float dn = P.nfp + (float)s1 * P.nfa + (float)s2 * P.nfb;
        if (!(fabsf(dn) > c.dthr)) {
            const double *nr = c.faces + (int64_t)Fq.f * kFaceStride + 9;  // the face's FP64 normal
            const int p = cls, q1 = cls == 0 ? 1 : 0, q2 = cls == 2 ? 1 : 2;
            const double den = VF_DADD(VF_DADD(nr[p], cmul(s1, nr[q1])), cmul(s2, nr[q2]));
            const int nz = (s1 != 0) + (s2 != 0);
            const double cn = nz == 0 ? 1.0 : (nz == 1 ? 1.4142135623730951 : 1.7320508075688772);
            if (fabs(den) < VF_DMUL(c.eps_par, cn)) continue;
        }
        const float cr = P1a * P2b - P1b * P2a;
        const float ab = 4e-6f * (ext + 1.0f) * (ext + 1.0f);
        const float t0 = tol * (fabsf(P1a) + fabsf(P1b)) * 1.0001f + ab;
        const float t1 = tol * (fabsf(P2a - P1a) + fabsf(P2b - P1b)) * 1.0001f + ab;
        const float t2 = tol * (fabsf(P2a) + fabsf(P2b)) * 1.0001f + ab;
        const float sg = cr >= 0.0f ? 1.0f : -1.0f;
        const bool steep = fabsf(dn) >= 1e-3f;
        const bool fast = steep && c.fast;
        const int gm1 = P.ba - s1 * P.bp, gm2 = P.bb - s2 * P.bp;
        for (int M2 = m2a; M2 <= m2b; ++M2) {
            const float Rb = (float)M2 + o2;
            for (int M1 = m1a; M1 <= m1b; ++M1) {
                const float Ra = (float)M1 + o1;
                const float E0 = sg * (P1a * Rb - P1b * Ra);
                const float E1 = sg * ((P2a - P1a) * (Rb - P1b) - (P2b - P1b) * (Ra - P1a));
                const float E2 = sg * (P2b * Ra - P2a * Rb);
                if (E0 < -t0 || E1 < -t1 || E2 < -t2) continue;  // misses the face
                const bool inner = fast && E0 >= t0 && E1 >= t1 && E2 >= t2;
                // node range along p (line_nodes in lattice units; c_p = 1)
                int ip_lo = P.lop, ip_hi = P.hip;
                if (steep) {
                    const float xs = -__fdividef(P.nfa * Ra + P.nfb * Rb, dn);
                    const float wid0 = 1.0f + 1e-4f + 1e-5f + __fdividef(Fq.ff9, fabsf(dn)) * 1.0001f;
                    const float wid = wid0 + 1.0001e-6f * __fdividef(fabsf(xs), fabsf(dn));
                    ip_lo = max(P.bp + (int)ceilf(xs + P.wp - wid), ip_lo);
                    ip_hi = min(P.bp + (int)floorf(xs + P.wp + wid), ip_hi);
                }
                const int mg1 = M1 + gm1, mg2 = M2 + gm2;
                if (inner && ip_lo <= ip_hi && ip_hi - ip_lo < 8) {
                    const int4 rec = make_int4(Fq.f, R | (1 << 4) | ((ip_hi - ip_lo) << 5) | (ip_lo << 8), mg1, mg2);
                    stage_put(c, s_rec, atomicAdd(&s_n, 1), rec);  // CTA stage slot (shared atomic)
                    continue;
                }
                // margin band / ill-conditioned / long range: exact path later
                for (int ip = ip_lo; ip <= ip_hi; ++ip) {
                    const int a = mg1 + s1 * ip, bq = mg2 + s2 * ip;
                    if (a < 0 || a >= P.n1 || bq < 0 || bq >= P.n2) continue;
                    const int i = cls == 0 ? ip : a;
                    const int j = cls == 1 ? ip : (cls == 0 ? a : bq);
                    const int k = cls == 2 ? ip : bq;
                    link_slow<2>(c, Fq.f, -1, i, j, k, R);
                }
            }
        }
    }
    add_tests(c, tests);
    __syncthreads();
    const int n = min(s_n, kLineStage);
    if (threadIdx.x == 0) s_base = n ? atomicAdd(c.n_lines, n) : 0;
    __syncthreads();
    // the staged lines leave as q-records: their faces were just read by
    // this CTA (L1 / L2), so the exact q costs no extra DRAM pass
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        int4 r = s_rec[i];
        if (s_base + i < c.line_cap) {
            r = qrec_convert(c, r);
            count_qrec(c, r);
        }
        line_store(c, s_base + i, r);
    }
}

// The recorded lines (fast class) get their exact q values right after the
// enumeration, still in phase 1 on the enumeration's side stream (the face
// records are re-read while the latency-bound level pipeline leaves HBM
// idle): k_links_q evaluates the oracle's FP64 num/den/d/q on the line's
// (2, rarely 3) candidate nodes and rewrites the record in place as a
// q-record -- base node, direction pair, and up to two accepted links
// (node offset along c, direction sign, q).  Phase 2 (k_links_resolve) then
// only maps nodes to LUT slots and min-merges q: no face access after the
// tables.  A line with more than two accepted nodes (FP64 rounding at the
// d = 0 / d = dx boundaries) sends its nodes to the band list instead.
//   q-record: x = i | j << 15 (base node = the first accepted one),
//             y = k | R << 15 | n << 19 | (o0 | s0 << 3) << 21 | (o1 | s1 << 3) << 25,
//             z, w = q0, q1 bits  (o: node offset along c, s: 1 = the -c link)
constexpr uint32_t kQRec = 1u << 31;  // y flag: the record is a q-record

// raw line record -> q-record (see above)
__device__ __forceinline__ int4 qrec_convert(const LinkCtx &c, const int4 rec) {
    const int f = rec.x, R = rec.y & 15, cnt = (rec.y >> 5) & 7, ip_lo = (rec.y >> 8) & 0x7fff;
    const int m1 = rec.z, m2 = rec.w;
    const int cx = c27(2 * R + 1, 0), cy = c27(2 * R + 1, 1), cz = c27(2 * R + 1, 2);  // c_rep[R], per-thread R
    const int p = cx != 0 ? 0 : (cy != 0 ? 1 : 2);
    const int q1 = p == 0 ? 1 : 0, q2 = p == 2 ? 1 : 2;
    const int cp = pick3(p, cx, cy, cz);
    const int s1 = pick3(q1, cx, cy, cz) * cp, s2 = pick3(q2, cx, cy, cz) * cp;
    const int n1 = pick3(q1, c.cells[0], c.cells[1], c.cells[2]);
    const int n2 = pick3(q2, c.cells[0], c.cells[1], c.cells[2]);
    const double2 *fp = reinterpret_cast<const double2 *>(c.faces + (int64_t)f * kFaceStride);
    const double2 a0 = __ldg(fp), a1 = __ldg(fp + 1), a4 = __ldg(fp + 4), a5 = __ldg(fp + 5);
    const double fv[6] = {a0.x, a0.y, a1.x, a4.y, a5.x, a5.y};  // v1, n
    // exact c.n (link_dir_setup / link_candidate; nonzero: the pair passed EPS_PARALLEL)
    const double den = VF_DADD(VF_DADD(cmul(cx, fv[3]), cmul(cy, fv[4])), cmul(cz, fv[5]));
    const double dx = c.dx;
    int ne = 0, bi = 0, bj = 0, bk = 0, ip0 = 0;
    uint32_t code[2] = {0, 0};
    float qv[2] = {0.0f, 0.0f};
    for (int ip = ip_lo; ip <= ip_lo + cnt; ++ip) {
        const int a = m1 + s1 * ip, b = m2 + s2 * ip;
        if (a < 0 || a >= n1 || b < 0 || b >= n2) continue;
        const int i = p == 0 ? ip : a;
        const int j = p == 1 ? ip : (p == 0 ? a : b);
        const int k = p == 2 ? ip : b;
        // = link_fast: d, the (0, dx] range and q bit-identical to the oracle
        const double d = VF_DDIV(plane_num(fv, fv + 3, node_c(i, dx), node_c(j, dx), node_c(k, dx)), den);
        const bool pos = d > 0.0;
        const double dd = pos ? d : -d;
        if (!(dd > 0.0 && dd <= dx)) continue;
        const double qd = c.pow2 ? VF_DMUL(dd, c.inv_dx) : VF_DDIV(dd, dx);
        if (ne == 0) {  // base node: the first accepted one
            bi = i; bj = j; bk = k; ip0 = ip;
        }
        if (ne < 2) {
            code[ne] = (uint32_t)(ip - ip0) | ((pos ? 0u : 1u) << 3);
            qv[ne] = __double2float_rn(qd);
        }
        ++ne;
    }
    if (ne > 2) {  // rounding at the range ends: node by node through the exact band path
        for (int ip = ip_lo; ip <= ip_lo + cnt; ++ip) {
            const int a = m1 + s1 * ip, b = m2 + s2 * ip;
            if (a < 0 || a >= n1 || b < 0 || b >= n2) continue;
            link_slow<2>(c, f, -1, p == 0 ? ip : a, p == 1 ? ip : (p == 0 ? a : b), p == 2 ? ip : b, R);
        }
        ne = 0;
    }
    return make_int4(bi | (bj << 15), (int)(kQRec | bk | (R << 15) | (ne << 19) | (code[0] << 21) | (code[1] << 25)),
                     __float_as_int(qv[0]), __float_as_int(qv[1]));
}

#ifndef VF_RESOLVE_MINB
#define VF_RESOLVE_MINB 4
#endif
// records the enumeration kernels did not convert themselves (stage overflow,
// large faces)
__global__ void __launch_bounds__(256, VF_RESOLVE_MINB)
    k_links_q(LinkCtx c) {
    const int64_t n = min((int64_t)*c.n_lines, c.line_cap);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int4 rec = c.lines[e];
        if (!((uint32_t)rec.y & kQRec)) {
            const int4 q = qrec_convert(c, rec);
            c.lines[e] = q;
            count_qrec(c, q);
        }
    }
}

// The q-records' links reach the LUT without global atomics on it:
//   phase 1, right after the enumeration (grid-independent, on the
//   enumeration's side stream): (1) every link -> the key of its finest
//   cell's PARENT block P (level L_max - 2 coordinates = node >> 3);
//   per-parent link counts (warp-aggregated atomics), (2) scan over the
//   parent keys (B_P^3 = B_L^3 / 8 counters), (3) scatter the links into
//   parent order;
//   phase 2, after the tables: ONE kernel, a warp per LUT slot (the
//   contraction map's inverse): the slot's 27 x 64 lengths initialised to -1
//   in shared memory, the links of its parent's bucket that fall in this
//   block (octant) min-merged there (shared atomicMin on the IEEE bits:
//   order-free, deterministic), the slot written once with 16-B stores.
//   No separate -1 fill, no LUT sector read back, no block map or hash
//   lookup per link.

// (3) links into parent order (the records are re-read; the cursor atomics'
// returns are the latency: two records per thread in flight)
__global__ void __launch_bounds__(256)
    k_block_scatter(LinkCtx c, int3 pdim, int32_t *__restrict__ bcur, unsigned long long *__restrict__ ent) {
    const int64_t n = min((int64_t)*c.n_lines, c.line_cap);
    const int lane = threadIdx.x & 31;
    const int64_t step = (int64_t)gridDim.x * blockDim.x * 2;
    for (int64_t e0 = (blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31)) * 2; e0 < n; e0 += step) {
        unsigned long long x[4];
        int32_t g[4], base[4];
        uint32_t grp[4];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const int64_t e = e0 + 32 * u + lane;
            const int4 rec = e < n ? c.lines[e] : make_int4(0, 0, 0, 0);
            const int ne = (rec.y >> 19) & 3;
#pragma unroll
            for (int k = 0; k < 2; ++k) g[2 * u + k] = k < ne ? link_bucket_entry(rec, k, pdim, x[2 * u + k]) : -1;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            grp[u] = __match_any_sync(0xffffffffu, g[u]);
            base[u] = 0;
            if (g[u] >= 0 && lane == __ffs(grp[u]) - 1) base[u] = atomicAdd(&bcur[g[u]], __popc(grp[u]));
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t bs = __shfl_sync(0xffffffffu, base[u], __ffs(grp[u]) - 1);
            if (g[u] >= 0) ent[bs + __popc(grp[u] & ((1u << lane) - 1u))] = x[u];
        }
    }
}

struct LoadBlk {
    const int32_t *p;
    __device__ int operator()(int64_t i) const { return p[i]; }
};
struct EmitBlk {
    int32_t *off, *cur;
    __device__ void operator()(int64_t i, int, int ex) const {
        off[i] = ex;
        cur[i] = ex;
    }
};

// phase 2: warp per LUT slot; N_b > cap latches VF_ECAPACITY with the count
// (the LUT stays unwritten), as the -1 fill did
constexpr int kLutWarps = 6;  // 6 x 6912 B of static shared memory
__global__ void __launch_bounds__(kLutWarps * 32)
    k_lut_blocks(LevelInfo li, int3 pdim, const int32_t *__restrict__ coords, const int32_t *__restrict__ inv,
                 const int32_t *__restrict__ d_n_b, int64_t cap, const int32_t *__restrict__ boff,
                 const int32_t *__restrict__ bcnt, const unsigned long long *__restrict__ ent,
                 float *__restrict__ lengths, int32_t *__restrict__ status) {
    __shared__ __align__(16) uint32_t s_lut[kLutWarps][27 * 64];
    const int64_t nb = *d_n_b;
    if (nb > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            atomicMax(status, VF_ECAPACITY);
            status[2] = (int32_t)nb;
        }
        return;
    }
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    uint32_t *S = s_lut[w];
    uint4 *S4 = reinterpret_cast<uint4 *>(S);
    const int64_t stride = (int64_t)gridDim.x * kLutWarps;
    // the warp's slots in batches of 32: lane k resolves slot k's block ->
    // parent bucket chain (inv -> coords -> key -> offsets) for the batch
    // at once, then the warp writes the 32 slots one after another
    for (int64_t sbase = (int64_t)blockIdx.x * kLutWarps + w; sbase < nb; sbase += 32 * stride) {
        uint32_t m_oct = 0;
        int32_t m_e0 = 0, m_ne = -1;  // -1: not this rank's slot / past the end
        {
            const int64_t my = sbase + lane * stride;
            if (my < nb) {
                const int4 co = reinterpret_cast<const int4 *>(coords)[inv[my]];
                const int32_t key = (co.x >> 1) + pdim.x * ((co.y >> 1) + pdim.y * (co.z >> 1));
                m_oct = (uint32_t)((co.x & 1) + 2 * (co.y & 1) + 4 * (co.z & 1));
                // multi-GPU: the LUT is distributed -- a rank writes the slots
                // of the blocks it owns (another rank's are left to their owner)
                if (owns_row(li, co.y, co.z)) {
                    m_e0 = boff[key];
                    m_ne = bcnt[key];
                }
            }
        }
        for (int k = 0; k < 32; ++k) {
            const int64_t slot = sbase + k * stride;
            if (slot >= nb) break;
            const int32_t ne = __shfl_sync(0xffffffffu, m_ne, k);
            if (ne < 0) continue;
            const int32_t e0 = __shfl_sync(0xffffffffu, m_e0, k);
            const uint32_t oct = __shfl_sync(0xffffffffu, m_oct, k);
            // the previous slot's bulk store has read the buffer
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
            for (int i = lane; i < 27 * 64 / 4; i += 32)
                S4[i] = make_uint4(0xBF800000u, 0xBF800000u, 0xBF800000u, 0xBF800000u);  // -1.0f
            __syncwarp();
            for (int i = lane; i < ne; i += 32) {
                const unsigned long long x = ent[e0 + i];
                // the parent's links in this block; q > 0: uint order is float order, below -1's bits
                if ((uint32_t)(x >> 41) == oct) atomicMin(&S[(uint32_t)(x >> 30) & 0x7ffu], (uint32_t)x & 0x3fffffffu);
            }
            // the slot (6,912 contiguous bytes) leaves through one TMA bulk
            // store: shared-memory writes made visible to the async proxy first
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
                const unsigned src = (unsigned)__cvta_generic_to_shared(S);
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(lengths + slot * (27 * 64)),
                             "r"(src), "r"(27 * 64 * 4)
                             : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
        }
    }
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

// the band candidates: full exact path (num, den, d, eps-box SAT), one per
// thread -- all threads take the same path, so the SAT runs converged
__global__ void __launch_bounds__(256)
    k_links_band(LinkCtx c) {
    const int64_t n = min((int64_t)c.n_band[0], c.band_cap);
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int4 x = c.band[e];
        const int i = x.z & 0xffff, j = x.z >> 16, k = x.w & 0xffff;
        int32_t slot = x.y;
        if (slot < 0) {  // queued by the line enumeration before the block map existed
            slot = slot_at(c, i, j, k);
            if (slot < 0) continue;
        }
        link_candidate(c.faces, x.x, x.w >> 16, i, j, k, c.dx, c.eps, c.eps_par, slot, c.lengths);
    }
}

// workspace: dense block map of the finest level | band counters | band list
static int64_t g_band_cap = -1;  // vf_set_link_band_cap (test hook: a smaller cap; -1 none)

static int64_t line_cap_of(const vf_config &cfg, int64_t F) {
    if (cfg.line_cap > 0) return cfg.line_cap;
    return F * 2 > (1 << 22) ? F * 2 : (1 << 22);
}
// band list: overflow only costs the fallback pass
static int64_t band_cap_of(const vf_config &cfg, int64_t F) {
    const int64_t b = line_cap_of(cfg, F) / 16;
    return b > (1 << 20) ? b : (1 << 20);
}

// workspace: band counters | band list
size_t link_workspace_size(const vf_config &cfg, int, int32_t, int64_t F) {
    return 512 + (size_t)band_cap_of(cfg, F) * sizeof(int4);
}

// LUT initialisation to -1 for the device-resident N_b slots (graph-safe:
// no host knowledge of N_b); N_b > cap latches VF_ECAPACITY with the count
__global__ void k_fill_lut(const int32_t *__restrict__ d_n_b, float *__restrict__ lengths, int64_t cap,
                           int32_t *__restrict__ status) {
    const int64_t nb = *d_n_b;
    if (nb > cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) {
            atomicMax(status, VF_ECAPACITY);
            status[2] = (int32_t)nb;
        }
        return;
    }
    const int64_t n4 = nb * 27 * 64 / 4;
    float4 *p = reinterpret_cast<float4 *>(lengths);
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
         i += (int64_t)gridDim.x * blockDim.x)
        p[i] = make_float4(-1.0f, -1.0f, -1.0f, -1.0f);
}

int fill_lut_impl(const int32_t *d_n_b, float *lengths, int64_t cap, int32_t *d_status,
                  cudaStream_t st) {
    k_fill_lut<<<max_ctas(4), 256, 0, st>>>(d_n_b, lengths, cap, d_status);
    return check_launch("k_fill_lut");
}

static int make_link_ctx(const vf_config &cfg, int L, int64_t F_band, const double *faces, float *lengths, void *ws,
                         LinkCtx &c, int &widen, LevelInfo &li) {
    li = make_level(cfg, L);
    if (li.cells[0] > 32767 || li.cells[1] > 32767 || li.cells[2] > 32767)
        return set_error(VF_EARG, "link lengths: > 32767 cells per axis");
    memset(&c, 0, sizeof(c));
    c.faces = faces;
    c.lengths = lengths;
    c.n_band = (int32_t *)ws;
    c.band = (int4 *)((char *)ws + 512);
    c.li = li;
    c.lut_cap = INT64_MAX;
    c.band_cap = band_cap_of(cfg, F_band);  // (F_band = 0: the SPEC-op workspace's list)
    if (g_band_cap >= 0 && g_band_cap < c.band_cap) c.band_cap = g_band_cap;
    c.dx = li.dx;
    c.eps = li.eps;
    c.eps_par = li.eps_par;
    c.bx = li.bins[0];
    c.by = li.bins[1];
    for (int d = 0; d < 3; ++d) c.len[d] = li.len[d];
    c.fast = li.eps >= 1e-12 * fmax(fmax(li.len[0], li.len[1]), li.len[2]);
    for (int d = 0; d < 3; ++d) c.cells[d] = li.cells[d];
    // 1/dx is exact when dx is a power of two; otherwise widen the ranges by one
    int ex = 0;
    const double mant = frexp(li.dx, &ex);
    c.pow2 = mant == 0.5;
    widen = c.pow2 ? 0 : 1;
    c.inv_dx = 1.0 / li.dx;
    c.epsL = (float)(li.eps * c.inv_dx);
    c.dthr = (float)(2.0 * li.eps_par * 1.7320508075688772) + 1e-5f;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_links<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLinkSmem);
        cudaFuncSetAttribute(k_links<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLinkSmem);
        cudaFuncSetAttribute(k_links<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kLinkSmem);
        attr = true;
    }
    return VF_OK;
}

static int link_grid(int64_t F) {
    int64_t grid = (F + 32 * kLinkWarps - 1) / (32 * kLinkWarps);
    if (grid > max_ctas(6)) grid = max_ctas(6);
    return grid < 1 ? 1 : (int)grid;
}

// the slot lookup of the finest level (slot_at): grid + contraction map,
// slots bounded by the LUT capacity (N_b > cap is latched as VF_ECAPACITY by
// the LUT kernels)
static void link_lookup(vf_grid *g, const int32_t *cmap, LinkCtx &c, int64_t lengths_cap) {
    c.child = g->d_child;
    c.cmap = cmap;
    c.level_start = g->d_level_start;
    c.lut_cap = lengths_cap > 0 ? lengths_cap : INT64_MAX;
}

int link_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
              int64_t F, const int32_t *map, const int32_t *d_n_map, float *lengths, void *ws,
              size_t ws_bytes, cudaStream_t st, void **events, const int32_t *d_n_b,
              int64_t lengths_cap) {
    const int L = g->n_levels - 1;
    if (ws_bytes < link_workspace_size(cfg, L, g->capacity, 0)) return set_error(VF_EARG, "link workspace too small");
    LinkCtx c;
    int widen;
    LevelInfo li;
    int rc = make_link_ctx(cfg, L, 0, faces, lengths, ws, c, widen, li);
    if (rc) return rc;
    cudaMemsetAsync(c.n_band, 0, 2 * sizeof(int32_t), st);
    link_lookup(g, cmap, c, lengths_cap);
    const int grid = link_grid(F);
    if (events) cudaEventRecord((cudaEvent_t)events[0], st);
    k_links<0><<<grid, kLinkWarps * 32, kLinkSmem, st>>>(c, widen, F, map, d_n_map);
    if ((rc = check_launch("k_links"))) return rc;
    k_links_band<<<max_ctas(2), 256, 0, st>>>(c);
    if ((rc = check_launch("k_links_band"))) return rc;
    k_links<1><<<grid, kLinkWarps * 32, kLinkSmem, st>>>(c, widen, F, map, d_n_map);
    rc = check_launch("k_links_full");
    if (events) cudaEventRecord((cudaEvent_t)events[1], st);
    return rc;
}

// ---- embed split: the line enumeration does not depend on the grid, so the
// embed launches it on a side stream at the start of phase 1 (overlapping the
// whole level pipeline) and resolves the recorded lines in phase 2.
// lines workspace: counters (n_lines, n_ovf, n_big) | lines | overflow face
// list | overflow bits | big-face list (the warp-flattened enumeration)
static size_t list_bytes(int64_t F) { return (((size_t)(F + 1) * sizeof(int32_t) + 255) & ~(size_t)255); }
static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }
// parent buckets: level L_max - 2 coordinates of the finest level (B_L^3 / 8)
static int3 parent_dims(const vf_config &cfg) {
    const int Lf = cfg.l_max - 1;
    return make_int3((cfg.nb[0] << Lf) / 2, (cfg.nb[1] << Lf) / 2, (cfg.nb[2] << Lf) / 2);
}
static int64_t parents_of(const vf_config &cfg) {
    const int3 p = parent_dims(cfg);
    return (int64_t)p.x * p.y * p.z + 1;
}

// ... | parent counts | parent offsets | parent cursors | slot -> block | scan |
// parent-ordered links (<= 2 links per q-record)
size_t link_lines_bytes(const vf_config &cfg, int64_t F, int32_t capacity) {
    const int64_t cap = line_cap_of(cfg, F), nt = parents_of(cfg);
    return 256 + (size_t)cap * sizeof(int4) + 2 * list_bytes(F) +
           al256(((size_t)F + 32) / 32 * sizeof(uint32_t)) + 3 * al256((size_t)nt * sizeof(int32_t)) +
           al256((size_t)capacity * sizeof(int32_t)) +
           al256(scan_workspace_bytes(nt)) + (size_t)(2 * cap) * sizeof(unsigned long long);
}

struct BlockLinkBufs {
    int32_t *bcnt, *boff, *bcur, *inv;  // per parent bucket: links, first, cursor; slot -> block
    void *scan_ws;
    unsigned long long *ent;  // parent-ordered links
    int64_t n_max;
};

static int32_t *line_bufs(LinkCtx &c, const vf_config &cfg, int64_t F, void *lines_ws, int32_t capacity = 0,
                          BlockLinkBufs *tb = nullptr) {
    c.line_cap = line_cap_of(cfg, F);
    c.n_lines = (int32_t *)lines_ws;
    c.n_ovf = c.n_lines + 1;
    c.n_tests = (unsigned long long *)((char *)lines_ws + 16);
    c.lines = (int4 *)((char *)lines_ws + 256);
    c.ovf_list = (int32_t *)((char *)c.lines + (size_t)c.line_cap * sizeof(int4));
    c.ovf_bits = (uint32_t *)((char *)c.ovf_list + list_bytes(F));
    int32_t *big = (int32_t *)((char *)c.ovf_bits + al256(((size_t)F + 32) / 32 * sizeof(uint32_t)));
    if (tb) {
        const int64_t nt = parents_of(cfg);
        char *p = (char *)big + list_bytes(F);
        tb->n_max = nt;
        tb->bcnt = (int32_t *)p;
        tb->boff = (int32_t *)(p + al256((size_t)nt * sizeof(int32_t)));
        tb->bcur = (int32_t *)(p + 2 * al256((size_t)nt * sizeof(int32_t)));
        tb->inv = (int32_t *)(p + 3 * al256((size_t)nt * sizeof(int32_t)));
        tb->scan_ws = p + 3 * al256((size_t)nt * sizeof(int32_t)) + al256((size_t)capacity * sizeof(int32_t));
        tb->ent = (unsigned long long *)((char *)tb->scan_ws + al256(scan_workspace_bytes(nt)));
    }
    return big;
}

static int link_bucket(const vf_config &cfg, LinkCtx &c, int64_t F, void *lines_ws, int32_t capacity,
                       cudaStream_t st);

int link_enum_impl(const vf_config &cfg, const double *faces, int64_t F, void *ws, void *lines_ws,
                   int32_t capacity, cudaStream_t st, void **events, const int32_t *map,
                   const int32_t *d_n_map) {
    LinkCtx c;
    int widen;
    LevelInfo li;
    int rc = make_link_ctx(cfg, cfg.l_max - 1, F, faces, nullptr, ws, c, widen, li);
    if (rc) return rc;
    BlockLinkBufs tb;
    int32_t *big = line_bufs(c, cfg, F, lines_ws, capacity, &tb);
    c.pcnt = tb.bcnt;
    c.pdim = parent_dims(cfg);
    cudaMemsetAsync(c.n_band, 0, 2 * sizeof(int32_t), st);
    cudaMemsetAsync(c.n_lines, 0, 24, st);  // n_lines, n_ovf, n_big, (pad), n_tests
    cudaMemsetAsync(tb.bcnt, 0, sizeof(int32_t) * (size_t)tb.n_max, st);
    cudaMemsetAsync(c.ovf_bits, 0, ((size_t)F + 32) / 32 * sizeof(uint32_t), st);
    kt_point("memset:link_counters");
    if (events) cudaEventRecord((cudaEvent_t)events[0], st);
    // small faces thread per face; the rest through the warp-flattened
    // kernel.  Short CTAs (no grid-stride loop in the small pass): they
    // retire quickly, so the higher-priority level pipeline takes SMs
    // between them.
    int32_t *n_big = c.n_lines + 2;
    const int64_t gs = (F + VF_SMALL_THREADS - 1) / VF_SMALL_THREADS;
    k_links_smallq<<<(unsigned)gs, VF_SMALL_THREADS, 0, st>>>(c, widen, F, g_small_ext, big, n_big, map, d_n_map);
    if ((rc = check_launch("k_links_small"))) return rc;
    int64_t g2 = (F + 32 * kLinkWarps - 1) / (32 * kLinkWarps);
    if (g2 > 4 * (int64_t)max_ctas(VF_LINK_MINB)) g2 = 4 * (int64_t)max_ctas(VF_LINK_MINB);
    k_links<2><<<(unsigned)(g2 < 1 ? 1 : g2), kLinkWarps * 32, kLinkSmem, st>>>(c, widen, F, big, n_big);
    if ((rc = check_launch("k_links_enum"))) return rc;
    // exact q of the recorded lines (records rewritten in place as q-records)
    k_links_q<<<max_ctas(VF_GRID_RESOLVE), 256, 0, st>>>(c);
    if ((rc = check_launch("k_links_q"))) return rc;
    rc = link_bucket(cfg, c, F, lines_ws, capacity, st);
    if (events) cudaEventRecord((cudaEvent_t)events[1], st);
    return rc;
}

const void *link_enum_kernel(int small) { return small ? (const void *)k_links_smallq : (const void *)k_links<2>; }

// counters of the last embed's cut-link pass (synchronous read):
// {lines recorded, line capacity, overflow faces, band candidates, band capacity,
//  faces of the warp-flattened (large-face) enumeration}
int link_stats(const vf_config &cfg, int64_t F, void *ws, void *lines_ws, int64_t out[7]) {
    LinkCtx c;
    int widen;
    LevelInfo li;
    int rc = make_link_ctx(cfg, cfg.l_max - 1, F, nullptr, nullptr, ws, c, widen, li);
    if (rc) return rc;
    line_bufs(c, cfg, F, lines_ws);
    int32_t a[3] = {0, 0, 0}, b[2] = {0, 0};
    cudaError_t e = cudaMemcpy(a, c.n_lines, sizeof(a), cudaMemcpyDeviceToHost);
    if (e == cudaSuccess) e = cudaMemcpy(b, c.n_band, sizeof(b), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) return set_cuda_error(e, "link stats");
    out[0] = a[0];
    out[1] = c.line_cap;
    out[2] = a[1];
    out[3] = b[0];
    out[4] = c.band_cap;
    out[5] = a[2];
    unsigned long long t = 0;
    if (cudaMemcpy(&t, c.n_tests, sizeof(t), cudaMemcpyDeviceToHost) != cudaSuccess)
        return set_cuda_error(cudaGetLastError(), "link stats");
    out[6] = (int64_t)t;
    return VF_OK;
}

// phase 1, right after the enumeration: the links of the q-records bucketed
// by finest-level parent key (see k_lut_blocks)
static int link_bucket(const vf_config &cfg, LinkCtx &c, int64_t F, void *lines_ws, int32_t capacity,
                       cudaStream_t st) {
    BlockLinkBufs tb;
    line_bufs(c, cfg, F, lines_ws, capacity, &tb);
    // (the counts were made as the records became q-records: count_qrec)
    cudaError_t e = scan_launch(LoadBlk{tb.bcnt}, EmitBlk{tb.boff, tb.bcur}, tb.n_max, nullptr, nullptr, tb.scan_ws, st);
    kt_point("scan_kernel");
    if (e != cudaSuccess) return set_cuda_error(e, "parent link scan");
    k_block_scatter<<<wave_ctas(k_block_scatter, 256), 256, 0, st>>>(c, parent_dims(cfg), tb.bcur, tb.ent);
    return check_launch("k_block_scatter");
}

// slot -> block from a contraction map (for tables computed without the
// inverse output: the sharded stage calls)
__global__ void k_cmap_inverse(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ cmap,
                               const int32_t *__restrict__ d_n_b, int64_t cap, int32_t *__restrict__ inv) {
    if (*d_n_b > cap) return;
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e; b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t slot = cmap[b];
        if (slot >= 0) inv[slot] = (int32_t)b;
    }
}

int link_inverse_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const int32_t *d_n_b, int64_t cap,
                      int64_t F, void *lines_ws, cudaStream_t st) {
    k_cmap_inverse<<<max_ctas(8), 256, 0, st>>>(g->n_levels - 1, g->d_level_start, cmap, d_n_b, cap,
                                                link_slot_inverse(cfg, F, lines_ws, g->capacity));
    return check_launch("k_cmap_inverse");
}

// the slot -> block inverse of the contraction map lives in the lines workspace
int32_t *link_slot_inverse(const vf_config &cfg, int64_t F, void *lines_ws, int32_t capacity) {
    LinkCtx c;
    memset(&c, 0, sizeof(c));
    BlockLinkBufs tb;
    line_bufs(c, cfg, F, lines_ws, capacity, &tb);
    return tb.inv;
}

int link_resolve_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
                      int64_t F, float *lengths, void *ws, void *lines_ws, cudaStream_t st,
                      void **events, const int32_t *d_n_b, int64_t lengths_cap, const int32_t *inv) {
    LinkCtx c;
    int widen;
    LevelInfo li;
    if (g->n_levels != cfg.l_max) return set_error(VF_EARG, "link resolve: the grid must reach L_max");
    int rc = make_link_ctx(cfg, cfg.l_max - 1, F, faces, lengths, ws, c, widen, li);
    if (rc) return rc;
    BlockLinkBufs tb;
    line_bufs(c, cfg, F, lines_ws, g->capacity, &tb);
    // slot hash for the rare paths (overflowed faces, band candidates)
    link_lookup(g, cmap, c, lengths_cap);
    if (events && events[0]) cudaEventRecord((cudaEvent_t)events[0], st);
    k_lut_blocks<<<max_ctas(5), kLutWarps * 32, 0, st>>>(li, parent_dims(cfg), g->d_coords, inv ? inv : tb.inv, d_n_b,
                                                         lengths_cap, tb.boff, tb.bcnt, tb.ent, lengths, g->d_status);
    if ((rc = check_launch("k_lut_blocks"))) return rc;
    // faces whose lines overflowed the record buffer: the direct kernel
    k_links<0><<<link_grid(F), kLinkWarps * 32, kLinkSmem, st>>>(c, widen, F, c.ovf_list, c.n_ovf);
    if ((rc = check_launch("k_links_ovf"))) return rc;
    k_links_band<<<max_ctas(2), 256, 0, st>>>(c);
    if ((rc = check_launch("k_links_band"))) return rc;
    k_links<1><<<link_grid(F), kLinkWarps * 32, kLinkSmem, st>>>(c, widen, F, nullptr, nullptr);
    rc = check_launch("k_links_full");
    if (events && events[1]) cudaEventRecord((cudaEvent_t)events[1], st);
    return rc;
}

}  // namespace vf

extern "C" float vf_set_link_small_ext(float e) {
    const float old = vf::g_small_ext;
    if (e == e) vf::g_small_ext = e;  // NaN only queries
    return old;
}

extern "C" int64_t vf_set_link_band_cap(int64_t n) {
    const int64_t old = vf::g_band_cap;
    if (n >= -1) vf::g_band_cap = n;
    return old;
}
