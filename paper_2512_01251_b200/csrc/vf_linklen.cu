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
// Candidates (face, node, pair) go to a per-warp shared-memory queue drained
// 32 at a time through the exact FP64 path (bit-identical to the oracle), so
// the SAT runs warp-converged.  The pre-filter passes a superset of the exact
// decisions; every stored value comes from the exact path.
#include <math.h>

#include "vf_common.cuh"
#include "vf_internal.h"

namespace vf {

// dense finest-level block -> LUT slot map; nothing is mapped when the
// device-resident N_b exceeds the LUT capacity (error latched by k_fill_lut)
// (multi-GPU: only this rank's blocks are mapped, so every rank fills the
// LUT slots of the blocks it owns)
__global__ void k_blockmap(LevelInfo li, int L, const int32_t *__restrict__ level_start,
                           const int32_t *__restrict__ coords, const int32_t *__restrict__ cmap,
                           int32_t *__restrict__ bmap, const int32_t *__restrict__ d_n_b,
                           int64_t cap) {
    if (d_n_b && *d_n_b > cap) return;
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t slot = cmap[b];
        if (slot < 0) continue;
        const int4 c = reinterpret_cast<const int4 *>(coords)[b];
        if (!owns_row(li, c.y, c.z)) continue;
        bmap[c.x + (int64_t)li.bins[0] * (c.y + (int64_t)li.bins[1] * c.z)] = slot;
    }
}

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
constexpr int kQueue = 640;

struct LinkQueue {
    int4 e[kLinkWarps][kQueue];  // (face, slot, i | j<<16, k | r<<16)
    int n[kLinkWarps];
};

struct LinkCtx {
    const double *faces;
    const int32_t *bmap;
    float *lengths;
    double dx, eps, eps_par;
    int bx, by, cells[3];
};

__device__ __forceinline__ void push_candidate(LinkQueue &Q, int w, const LinkCtx &c, int f, int slot,
                                               int i, int j, int k, int r) {
    const int pos = atomicAdd(&Q.n[w], 1);
    if (pos < kQueue) {
        Q.e[w][pos] = make_int4(f, slot, i | (j << 16), k | (r << 16));
    } else {  // overflow (pathological face): decide inline, same exact path
        link_candidate(c.faces, f, r, i, j, k, c.dx, c.eps, c.eps_par, slot, c.lengths);
    }
}

// drain the queue in full warps (all = drain the remainder too); warp-uniform
__device__ __forceinline__ void drain(LinkQueue &Q, int w, int lane, const LinkCtx &c, bool all) {
    __syncwarp();
    int n = min(Q.n[w], kQueue);
    while (n >= 32 || (all && n > 0)) {
        const int take = min(n, 32);
        int4 e = make_int4(0, -1, 0, 0);
        if (lane < take) e = Q.e[w][n - take + lane];
        __syncwarp();
        if (lane < take)
            link_candidate(c.faces, e.x, e.w >> 16, e.z & 0xffff, e.z >> 16, e.w & 0xffff, c.dx,
                           c.eps, c.eps_par, e.y, c.lengths);
        n -= take;
    }
    __syncwarp();
    if (lane == 0) Q.n[w] = n;
    __syncwarp();
}

// representative directions q = 2r+1 (lattice.py order) in constant memory
__constant__ int8_t c_rep[13][3] = {
    {1, 0, 0},  {0, 1, 0},  {0, 0, 1},   {1, 1, 0},  {1, 0, 1},  {1, 0, -1}, {1, -1, 0},
    {0, 1, 1},  {0, 1, -1}, {1, 1, 1},   {1, 1, -1}, {1, -1, 1}, {1, -1, -1}};

// one direction pair r: enumerate lattice lines along c that pierce the face,
// push the nodes within one link of each crossing.  A runtime loop over r
// (not 13 unrolled copies): the unrolled kernel was 12k SASS instructions and
// stalled 89% on instruction fetch.
__device__ __noinline__ void face_direction(LinkQueue &Q, int w, const LinkCtx &c, int f, int R,
                                            const double *v, const float *nf, const float *V1,
                                            const float *V2, float Ef, const int *lo_p,
                                            const int *hi_p) {
    const int cc[3] = {c_rep[R][0], c_rep[R][1], c_rep[R][2]};
    const int p = cc[0] != 0 ? 0 : (cc[1] != 0 ? 1 : 2);
    const int q1 = p == 0 ? 1 : 0, q2 = p == 2 ? 1 : 2;
    const int s1 = cc[q1] * cc[p], s2 = cc[q2] * cc[p];  // c_q / c_p (c_p = +-1)
    const float dn = (float)cc[0] * nf[0] + (float)cc[1] * nf[1] + (float)cc[2] * nf[2];
    const double dx = c.dx;
    const float dxf = (float)dx;
    // projected triangle (relative to v1) on the plane x_p = v1_p
    const float P0a = 0.0f, P0b = 0.0f;
    const float P1a = V1[q1] - (float)s1 * V1[p], P1b = V1[q2] - (float)s2 * V1[p];
    const float P2a = V2[q1] - (float)s1 * V2[p], P2b = V2[q2] - (float)s2 * V2[p];
    const float cr = P1a * P2b - P1b * P2a;
    const float ext = fmaxf(fmaxf(fabsf(P1a), fabsf(P1b)), fmaxf(fabsf(P2a), fabsf(P2b)));
    // tolerance: eps-cube acceptance (<= 2 sqrt 6 eps after the oblique
    // projection) + FP32 error of coordinates of magnitude ext + dx
    const float tol = 1e-5f * (ext + dxf) + 6.0f * (float)c.eps;
    // (a degenerate projection -- face parallel to c -- keeps only lattice
    // points within tol of the projected segment: the edge tests stay valid)
    const float sg = cr >= 0.0f ? 1.0f : -1.0f;
    // inward edge functions (not normalised): E_k(P) = sg * cross(edge_k, P - P_k)
    const float e0a = P1a - P0a, e0b = P1b - P0b;
    const float e1a = P2a - P1a, e1b = P2b - P1b;
    const float e2a = P0a - P2a, e2b = P0b - P2b;
    const float l0 = sqrtf(e0a * e0a + e0b * e0b), l1 = sqrtf(e1a * e1a + e1b * e1b),
                l2 = sqrtf(e2a * e2a + e2b * e2b);
    // lattice of line traces: coordinate j of the trace of the line through
    // node (i_p, i_q1, i_q2) is ((i_qj - s_j i_p) + delta_j) dx + s_j v1_p,
    // delta_j = (1 - s_j)/2; relative to v1: subtract v1_qj
    const double off1 = (double)s1 * v[p] - v[q1], off2 = (double)s2 * v[p] - v[q2];
    const double d1 = 0.5 * (1 - s1), d2 = 0.5 * (1 - s2);
    const float bmin1 = fminf(fminf(P0a, P1a), P2a) - tol, bmax1 = fmaxf(fmaxf(P0a, P1a), P2a) + tol;
    const float bmin2 = fminf(fminf(P0b, P1b), P2b) - tol, bmax2 = fmaxf(fmaxf(P0b, P1b), P2b) + tol;
    const double inv = 1.0 / dx;
    const int m1a = (int)ceil(((double)bmin1 - off1) * inv - d1 - 1e-6);
    const int m1b = (int)floor(((double)bmax1 - off1) * inv - d1 + 1e-6);
    const int m2a = (int)ceil(((double)bmin2 - off2) * inv - d2 - 1e-6);
    const int m2b = (int)floor(((double)bmax2 - off2) * inv - d2 + 1e-6);
    const bool steep = fabsf(dn) >= 1e-3f;
    for (int m2 = m2a; m2 <= m2b; ++m2) {
        const float Rb = (float)(((double)m2 + d2) * dx + off2);
        for (int m1 = m1a; m1 <= m1b; ++m1) {
            const float Ra = (float)(((double)m1 + d1) * dx + off1);
            // inside the projected triangle (with tolerance)
            const float E0 = sg * (e0a * (Rb - P0b) - e0b * (Ra - P0a));
            const float E1 = sg * (e1a * (Rb - P1b) - e1b * (Ra - P1a));
            const float E2 = sg * (e2a * (Rb - P2b) - e2b * (Ra - P2a));
            if (E0 < -tol * l0 || E1 < -tol * l1 || E2 < -tol * l2) continue;
            // crossing with the face plane: Q = v1 + Ra e_q1 + Rb e_q2 (+0 e_p),
            // points Q + lam c; n.(Q + lam c - v1) = 0
            int ip_lo, ip_hi;
            if (steep) {
                const float lam = -(nf[q1] * Ra + nf[q2] * Rb) / dn;
                const float xs = (float)cc[p] * lam;  // x_p* - v1_p
                const float wid = dxf * (1.0f + 1e-4f) + (Ef + 1e-6f * fabsf(xs)) / fabsf(dn) + 1e-5f * dxf;
                // node index i_p with |x_p* - (i_p + 0.5) dx| <= dx
                ip_lo = (int)ceil(((double)(xs - wid) + v[p]) * inv - 0.5);
                ip_hi = (int)floor(((double)(xs + wid) + v[p]) * inv - 0.5);
                ip_lo = max(ip_lo, lo_p[p]);
                ip_hi = min(ip_hi, hi_p[p]);
            } else {  // ill-conditioned crossing: every node of the face's p-range +- dx
                ip_lo = lo_p[p];
                ip_hi = hi_p[p];
            }
            for (int ip = ip_lo; ip <= ip_hi; ++ip) {
                int idx[3];
                idx[p] = ip;
                // i_qj = m_j + s_j i_p
                idx[q1] = m1 + s1 * ip;
                idx[q2] = m2 + s2 * ip;
                if (idx[q1] < 0 || idx[q1] >= c.cells[q1] || idx[q2] < 0 || idx[q2] >= c.cells[q2]) continue;
                const int32_t slot =
                    c.bmap[(idx[0] >> 2) + (int64_t)c.bx * ((idx[1] >> 2) + (int64_t)c.by * (idx[2] >> 2))];
                if (slot < 0) continue;
                push_candidate(Q, w, c, f, slot, idx[0], idx[1], idx[2], R);
            }
        }
    }
}


__global__ void __launch_bounds__(kLinkWarps * 32)
    k_links(LinkCtx c, double inv_dx, int widen, int64_t F, const int32_t *__restrict__ map,
            const int32_t *__restrict__ d_n_map) {
    __shared__ LinkQueue Q;
    const int64_t n = d_n_map ? (int64_t)*d_n_map : F;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (lane == 0) Q.n[w] = 0;
    __syncwarp();
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    // all lanes of a warp iterate together (uniform trip count) so drains are
    // warp-synchronous; lanes past the end are inactive
    const int64_t first = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31);
    for (int64_t base = first; base < n; base += stride) {
        const int64_t m = base + lane;
        const bool active = m < n;
        double v[9] = {0, 0, 0, 0, 0, 0, 0, 0, 0}, nn[3] = {0, 0, 0};
        int f = 0;
        float nf[3] = {0, 0, 0}, V1[3] = {0, 0, 0}, V2[3] = {0, 0, 0}, Ef = 0.0f;
        int lo_p[3] = {0, 0, 0}, hi_p[3] = {-1, -1, -1};
        if (active) {
            f = map ? map[m] : (int)m;
            load_face(c.faces, f, v, nn);
            double ext = 0.0;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                nf[d] = (float)nn[d];
                V1[d] = (float)(v[3 + d] - v[d]);
                V2[d] = (float)(v[6 + d] - v[d]);
                const double lo = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
                const double hi = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
                ext = fmax(ext, hi - lo);
                // nodes within one link of the face AABB (fallback range)
                lo_p[d] = max((int)floor((lo - c.dx - 2.0 * c.eps) * inv_dx - 0.5) - widen, 0);
                hi_p[d] = min((int)floor((hi + c.dx + 2.0 * c.eps) * inv_dx - 0.5) + 1 + widen, c.cells[d] - 1);
            }
            Ef = 4e-6f * (float)(ext + 2.0 * c.dx);
        }
#pragma unroll 1
        for (int r = 0; r < 13; ++r) {
            if (active) face_direction(Q, w, c, f, r, v, nf, V1, V2, Ef, lo_p, hi_p);
            drain(Q, w, lane, c, false);
        }
    }
    drain(Q, w, lane, c, true);
}

size_t link_workspace_size(const vf_config &cfg, int finest) {
    const int64_t nb = (int64_t)(cfg.nb[0] << finest) * (cfg.nb[1] << finest) * (cfg.nb[2] << finest);
    return ((size_t)nb * sizeof(int32_t) + 255) & ~(size_t)255;
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

int link_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
              int64_t F, const int32_t *map, const int32_t *d_n_map, float *lengths, void *ws,
              size_t ws_bytes, cudaStream_t st, void **events, const int32_t *d_n_b,
              int64_t lengths_cap) {
    const int L = g->n_levels - 1;
    if (ws_bytes < link_workspace_size(cfg, L)) return set_error(VF_EARG, "link workspace too small");
    const LevelInfo li = make_level(cfg, L);
    if (li.cells[0] > 32767 || li.cells[1] > 32767 || li.cells[2] > 32767)
        return set_error(VF_EARG, "link lengths: > 32767 cells per axis");
    const int64_t nb = (int64_t)li.bins[0] * li.bins[1] * li.bins[2];
    int32_t *bmap = (int32_t *)ws;
    cudaMemsetAsync(bmap, 0xff, sizeof(int32_t) * (size_t)nb, st);
    k_blockmap<<<max_ctas(8), 256, 0, st>>>(li, L, g->d_level_start, g->d_coords, cmap, bmap, d_n_b,
                                            lengths_cap);
    int rc = check_launch("k_blockmap");
    if (rc) return rc;
    LinkCtx c;
    c.faces = faces;
    c.bmap = bmap;
    c.lengths = lengths;
    c.dx = li.dx;
    c.eps = li.eps;
    c.eps_par = li.eps_par;
    c.bx = li.bins[0];
    c.by = li.bins[1];
    for (int d = 0; d < 3; ++d) c.cells[d] = li.cells[d];
    // 1/dx is exact when dx is a power of two; otherwise widen the ranges by one
    int ex = 0;
    const double mant = frexp(li.dx, &ex);
    const int widen = (mant == 0.5) ? 0 : 1;
    const double inv_dx = 1.0 / li.dx;
    int64_t grid = (F + 32 * kLinkWarps - 1) / (32 * kLinkWarps);
    if (grid > max_ctas(6)) grid = max_ctas(6);
    if (grid < 1) grid = 1;
    if (events) cudaEventRecord((cudaEvent_t)events[0], st);
    k_links<<<(int)grid, kLinkWarps * 32, 0, st>>>(c, inv_dx, widen, F, map, d_n_map);
    rc = check_launch("k_links");
    if (events) cudaEventRecord((cudaEvent_t)events[1], st);
    return rc;
}

}  // namespace vf
