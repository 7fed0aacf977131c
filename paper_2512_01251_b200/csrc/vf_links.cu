// vf_links.cu -- boundary cells, boundary tables and the cut-link LUT
// (SPEC.md:319-345).
//
//   K-bnd    one CTA (64 threads = cells) per finest-level block that is solid
//            or touches a solid block; direct neighbour reads through the A15
//            index maps (the paper's faster "direct" variant).
//            Single pass: pass 1 only tests "== SOLID" and pass 2 only turns
//            FLUID into BOUNDARY, so fusing the two kernels of PAPER.md:941 is
//            race-free in outcome.
//   K-tab    contraction map = exclusive scan of (count > 0) over the finest
//            level in ascending block id (pin A16).
//   K-link   FACE-parallel link lengths: every face enumerates the lattice
//            nodes of its (dx-widened) AABB and the 13 antiparallel direction
//            pairs; accepted links scatter q = d/dx into the LUT with an
//            atomicMin on the IEEE bits (order-free, hence deterministic and
//            equal to the per-cell minimum of PAPER.md:975; -1.0f sorts above
//            every positive float as uint32, so the -1 initialisation doubles
//            as "no hit").  A dense block map of the finest level replaces the
//            per-cell bin traversal; MD binning therefore drops out of the
//            embed path (its result is invariant).
#include <math.h>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

constexpr int kBndWarps = 8;

// warp per finest-level block: the 27 neighbour ids decide candidacy (the
// block or a neighbour is solid); a 6x6x6 shared-memory halo of SOLID bits is
// gathered once, then every FLUID cell ORs its 26 halo neighbours (constant
// offsets).  Reads of concurrently re-marked cells see FLUID or BOUNDARY,
// both "not SOLID", so the fused single pass equals PAPER.md:941's two passes.
__global__ void __launch_bounds__(kBndWarps * 32)
    k_boundary(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ nbr,
               uint8_t *__restrict__ bflags, uint8_t *__restrict__ masks,
               int32_t *__restrict__ bcount) {
    __shared__ uint8_t s_halo[kBndWarps][216];
    __shared__ int32_t s_nb[kBndWarps][27];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kBndWarps + w, nw = (int64_t)gridDim.x * kBndWarps;
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + gw; b < e; b += nw) {
        int32_t myn = -1;
        if (lane < 27) myn = (lane == 0) ? (int32_t)b : nbr[27 * b + lane];
        const bool sol = (lane < 27 && myn >= 0) ? (bflags[myn] & VF_BF_SOLID) != 0 : false;
        if (!__any_sync(0xffffffffu, sol)) {  // not a candidate (A18): no boundary cell
            if (lane == 0) {
                bcount[b] = 0;
                bflags[b] = (uint8_t)(bflags[b] & ~VF_BF_BOUNDARY);
            }
            continue;
        }
        if (lane < 27) s_nb[w][lane] = myn;
        __syncwarp();
        for (int h = lane; h < 216; h += 32) {
            const int hx = h % 6 - 1, hy = (h / 6) % 6 - 1, hz = h / 36 - 1;
            const int ox = hx < 0 ? -1 : (hx > 3 ? 1 : 0);
            const int oy = hy < 0 ? -1 : (hy > 3 ? 1 : 0);
            const int oz = hz < 0 ? -1 : (hz > 3 ? 1 : 0);
            const int32_t nbk = s_nb[w][slot_of(ox, oy, oz)];
            s_halo[w][h] = (nbk >= 0) ? (uint8_t)(masks[64 * (int64_t)nbk + (hx & 3) + 4 * (hy & 3) +
                                                       16 * (hz & 3)] == VF_SOLID)
                                      : (uint8_t)0;
        }
        __syncwarp();
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int c = lane + 32 * k;
            const int I = c & 3, J = (c >> 2) & 3, K = c >> 4;
            if (masks[64 * b + c] != VF_FLUID) continue;
            const uint8_t *hp = &s_halo[w][(I + 1) + 6 * (J + 1) + 36 * (K + 1)];
            uint32_t any = 0;
#pragma unroll
            for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx)
                        if (dx || dy || dz) any |= hp[dx + 6 * dy + 36 * dz];
            if (any) {
                masks[64 * b + c] = VF_BOUNDARY;
                ++cnt;
            }
        }
        cnt = warp_sum(cnt);
        if (lane == 0) {
            bcount[b] = cnt;
            const uint8_t f = bflags[b];
            bflags[b] = (uint8_t)(cnt > 0 ? (f | VF_BF_BOUNDARY) : (f & ~VF_BF_BOUNDARY));
        }
        __syncwarp();
    }
}

int boundary_impl(vf_grid *g, int32_t *bcount, cudaStream_t st) {
    const int L = g->n_levels - 1;
    cudaMemsetAsync(bcount, 0, sizeof(int32_t) * (size_t)g->capacity, st);
    k_boundary<<<max_ctas(8), kBndWarps * 32, 0, st>>>(L, g->d_level_start, g->d_nbr, g->d_bflags,
                                                       g->d_masks, bcount);
    return check_launch("k_boundary");
}

// ---------------------------------------------------------------------------
// tables

struct LoadBnd {
    const int32_t *level_start;
    int L;
    const int32_t *bcount;
    __device__ int operator()(int64_t i) const { return bcount[level_start[L] + i] > 0 ? 1 : 0; }
};
struct EmitCmap {
    const int32_t *level_start;
    int L;
    int32_t *cmap;
    __device__ void operator()(int64_t i, int v, int ex) const {
        cmap[level_start[L] + i] = v ? ex : -1;
    }
};

__global__ void k_level_count2(int L, const int32_t *__restrict__ level_start, int32_t *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = level_start[L + 1] - level_start[L];
}

size_t tables_workspace_size(int32_t capacity) {
    return 256 + ((scan_workspace_bytes(capacity) + 255) & ~(size_t)255);
}

int tables_impl(vf_grid *g, const int32_t *bcount, int32_t *cmap, int32_t *d_n_b, void *ws,
                size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < tables_workspace_size(g->capacity)) return set_error(VF_EARG, "tables workspace too small");
    const int L = g->n_levels - 1;
    int32_t *scal = (int32_t *)ws;
    void *scan_ws = (char *)ws + 256;
    // non-finest blocks are never mapped
    cudaMemsetAsync(cmap, 0xff, sizeof(int32_t) * (size_t)g->capacity, st);
    k_level_count2<<<1, 32, 0, st>>>(L, g->d_level_start, scal);
    int rc = check_launch("k_level_count2");
    if (rc) return rc;
    cudaError_t ce = scan_launch(LoadBnd{g->d_level_start, L, bcount}, EmitCmap{g->d_level_start, L, cmap},
                                 g->capacity, scal, d_n_b, scan_ws, st);
    return ce == cudaSuccess ? VF_OK : set_cuda_error(ce, "tables scan");
}

// ---------------------------------------------------------------------------
// link lengths

__global__ void k_blockmap(int L, int bx, int by, const int32_t *__restrict__ level_start,
                           const int32_t *__restrict__ coords, const int32_t *__restrict__ cmap,
                           int32_t *__restrict__ bmap) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t slot = cmap[b];
        if (slot < 0) continue;
        const int4 c = reinterpret_cast<const int4 *>(coords)[b];
        bmap[c.x + (int64_t)bx * (c.y + (int64_t)by * c.z)] = slot;
    }
}

// zero-component mask of the representative direction q = 2r+1
__device__ __forceinline__ uint32_t zero_axes(int r) {
    const int q = 2 * r + 1;
    return (uint32_t)(c27(q, 0) == 0) | ((uint32_t)(c27(q, 1) == 0) << 1) |
           ((uint32_t)(c27(q, 2) == 0) << 2);
}

// lattice-node index range whose centres can lie in [A, B] (superset)
__device__ __forceinline__ void node_range(double A, double B, double dx, int n, int &a, int &b) {
    double fa = floor(VF_DSUB(VF_DDIV(A, dx), 0.5));
    double fb = floor(VF_DSUB(VF_DDIV(B, dx), 0.5)) + 1.0;
    fa = fmax(fa, 0.0);
    fb = fmin(fb, (double)(n - 1));
    a = (int)fa;
    b = fa > fb ? a - 1 : (int)fb;
}

// exact decision for one (face, node, direction pair) candidate: num and
// d = num/den bit-identical to the oracle (orc_link_lengths), then the
// eps-box SAT at the piercing point; accepted q = d/dx is min-merged into the
// LUT through the IEEE bits (uint32 order == float order for q > 0, and
// -1.0f = 0xBF800000 sorts above all of them).
__device__ __noinline__ void link_candidate(const double *__restrict__ faces, int64_t f, int r,
                                            int i, int j, int k, double dx, double eps, double eps_par,
                                            int32_t slot, float *__restrict__ lengths) {
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

// K-link: one WARP per face.  An accepted link (node v, direction c,
// 0 < d <= dx) needs |num| = |d (c.n)| <= sqrt(3) dx, so the candidate
// nodes lie in a slab around the face plane: the warp sweeps the columns of
// the face's dx-widened AABB along the plane's dominant normal axis and
// keeps only the <= 8 nodes per column inside the slab (work ~ face area /
// dx^2 instead of AABB volume).  Lanes take (column, slab position) pairs.
// Per node an FP32 pre-filter -- relative coordinates, |num| <= dx |c.n|,
// piercing point inside the face AABB +- eps -- rejects almost everything
// with generous margins (1e-5 dx, >> FP32 rounding); survivors run the exact
// FP64 path above, so the pre-filter never changes a result.
constexpr int kLinkWarps = 8;

__global__ void __launch_bounds__(kLinkWarps * 32)
    k_links(LevelInfo li, const double *__restrict__ faces, int64_t F,
            const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map,
            const int32_t *__restrict__ bmap, float *__restrict__ lengths) {
    const int64_t n = d_n_map ? (int64_t)*d_n_map : F;
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * kLinkWarps + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * kLinkWarps;
    const double dx = li.dx, eps = li.eps;
    const float dxf = (float)dx;
    const float slack = 1e-5f * dxf;
    const float Tf = 1.7320508f * dxf * (1.0f + 1e-5f) + slack;  // sqrt(3) dx bound on |num|
    __shared__ int4 s_node[kLinkWarps][32];
    __shared__ uint16_t s_q[kLinkWarps][32 * 13];
    const int wib = threadIdx.x >> 5;
    for (int64_t m = gw; m < n; m += nw) {
        const int64_t f = map ? (int64_t)map[m] : m;
        double v[9], nn[3];
        load_face(faces, f, v, nn);
        int a1[3], b1[3], a0[3], b0[3];
        float rlo[3], rhi[3];  // face AABB +- (eps + margin), relative to v1
        bool empty = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            const double lo = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
            const double hi = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
            node_range(lo - dx - 2.0 * eps, hi + dx + 2.0 * eps, dx, li.cells[d], a1[d], b1[d]);
            node_range(lo - 2.0 * eps, hi + 2.0 * eps, dx, li.cells[d], a0[d], b0[d]);
            rlo[d] = (float)(lo - v[d]) - (float)eps - 1e-4f * dxf;
            rhi[d] = (float)(hi - v[d]) + (float)eps + 1e-4f * dxf;
            if (a1[d] > b1[d]) empty = true;
        }
        if (empty) continue;  // warp-uniform
        const float nf0 = (float)nn[0], nf1 = (float)nn[1], nf2 = (float)nn[2];
        // sweep axis = dominant normal component (|n_a| >= 1/sqrt(3))
        const float ax0 = fabsf(nf0), ax1 = fabsf(nf1), ax2 = fabsf(nf2);
        const int a = (ax0 >= ax1 && ax0 >= ax2) ? 0 : (ax1 >= ax2 ? 1 : 2);
        const int u = (a + 1) % 3, w = (a + 2) % 3;
        const float na = a == 0 ? nf0 : (a == 1 ? nf1 : nf2);
        const float nu = u == 0 ? nf0 : (u == 1 ? nf1 : nf2);
        const float nwv = w == 0 ? nf0 : (w == 1 ? nf1 : nf2);
        const int span = (int)floorf(2.0f * Tf / (fabsf(na) * dxf)) + 2;
        const int ncu = b1[u] - a1[u] + 1, ncw = b1[w] - a1[w] + 1;
        const int total = ncu * ncw * span;
        float denf[13];
#pragma unroll
        for (int r = 0; r < 13; ++r) {
            const int q = 2 * r + 1;
            denf[r] = (float)c27(q, 0) * nf0 + (float)c27(q, 1) * nf1 + (float)c27(q, 2) * nf2;
        }
        for (int base = 0; base < total; base += 32) {
            const int kk = base + lane;
            uint32_t cand = 0;  // bit r: direction pair r survives the FP32 pre-filter
            int idx[3] = {0, 0, 0};
            int32_t slot = -1;
            if (kk < total) {
                const int col = kk / span, sidx = kk - col * span;
                const int iu = a1[u] + col % ncu, iw = a1[w] + col / ncu;
                const float Xu = (float)(node_c(iu, dx) - v[u]);
                const float Xw = (float)(node_c(iw, dx) - v[w]);
                const float C = Xu * nu + Xw * nwv;
                // |Xa na + C| <= Tf  <=>  Xa in [(-C - Tf)/na, (-C + Tf)/na]
                float xa0 = (-C - Tf) / na, xa1 = (-C + Tf) / na;
                if (xa0 > xa1) { const float tmp = xa0; xa0 = xa1; xa1 = tmp; }
                const int ia_lo = max((int)floor(((double)xa0 + v[a]) / dx - 0.5), a1[a]);
                const int ia_hi = min((int)floor(((double)xa1 + v[a]) / dx - 0.5) + 1, b1[a]);
                const int ia = ia_lo + sidx;
                idx[a] = ia; idx[u] = iu; idx[w] = iw;
                if (ia <= ia_hi)
                    slot = bmap[(idx[0] >> 2) +
                                (int64_t)li.bins[0] * ((idx[1] >> 2) + (int64_t)li.bins[1] * (idx[2] >> 2))];
                if (slot >= 0) {
                    float X[3];
                    X[a] = (float)(node_c(ia, dx) - v[a]); X[u] = Xu; X[w] = Xw;
                    const float numf = -(X[0] * nf0 + X[1] * nf1 + X[2] * nf2);  // (v1 - x).n
                    uint32_t m0 = 0;  // per axis: node inside the eps-tight AABB range
#pragma unroll
                    for (int d = 0; d < 3; ++d) m0 |= (uint32_t)(idx[d] >= a0[d] && idx[d] <= b0[d]) << d;
                    if (fabsf(numf) <= Tf) {
#pragma unroll
                        for (int r = 0; r < 13; ++r) {
                            if (zero_axes(r) & ~m0) continue;  // c_k = 0 axes keep v_k: must be in R0
                            const float dn = denf[r];
                            if (fabsf(numf) > fabsf(dn) * dxf * (1.0f + 1e-5f) + slack) continue;
                            if (fabsf(dn) >= 0.1f) {  // piercing point inside the AABB
                                const float da = numf / dn;
                                const int q = 2 * r + 1;
                                bool out = false;
#pragma unroll
                                for (int d = 0; d < 3; ++d) {
                                    const int cd = c27(q, d);
                                    if (cd == 0) continue;
                                    const float p = X[d] + (float)cd * da;
                                    out |= (p < rlo[d]) || (p > rhi[d]);
                                }
                                if (out) continue;
                            }
                            cand |= 1u << r;
                        }
                    }
                }
            }
            // warp-cooperative exact path: queue (lane, r) candidates in shared
            // memory and give every lane one, so the FP64 SAT runs converged
            const int nc = __popc(cand);
            int off = nc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, off, o);
                if (lane >= o) off += y;
            }
            const int ntot = __shfl_sync(0xffffffffu, off, 31);
            off -= nc;
            s_node[wib][lane] = make_int4(idx[0], idx[1], idx[2], slot);
            for (uint32_t c = cand; c; c &= c - 1) s_q[wib][off++] = (uint16_t)((lane << 4) | (__ffs(c) - 1));
            __syncwarp();
            for (int qi = lane; qi < ntot; qi += 32) {
                const int e = s_q[wib][qi];
                const int4 nd = s_node[wib][e >> 4];
                link_candidate(faces, f, e & 15, nd.x, nd.y, nd.z, dx, eps, li.eps_par, nd.w, lengths);
            }
            __syncwarp();
        }
        // reconverge before the next face: without it the lanes drift apart
        // (independent thread scheduling) and re-run the per-face setup per
        // lane subset (measured 27x instruction inflation)
        __syncwarp();
    }
}

size_t link_workspace_size(const vf_config &cfg, int finest) {
    const int64_t nb = (int64_t)(cfg.nb[0] << finest) * (cfg.nb[1] << finest) * (cfg.nb[2] << finest);
    return ((size_t)nb * sizeof(int32_t) + 255) & ~(size_t)255;
}

int link_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
              int64_t F, const int32_t *map, const int32_t *d_n_map, float *lengths, void *ws,
              size_t ws_bytes, cudaStream_t st, void **events) {
    const int L = g->n_levels - 1;
    if (ws_bytes < link_workspace_size(cfg, L)) return set_error(VF_EARG, "link workspace too small");
    const LevelInfo li = make_level(cfg, L);
    const int64_t nb = (int64_t)li.bins[0] * li.bins[1] * li.bins[2];
    int32_t *bmap = (int32_t *)ws;
    cudaMemsetAsync(bmap, 0xff, sizeof(int32_t) * (size_t)nb, st);
    k_blockmap<<<max_ctas(8), 256, 0, st>>>(L, li.bins[0], li.bins[1], g->d_level_start, g->d_coords,
                                            cmap, bmap);
    int rc = check_launch("k_blockmap");
    if (rc) return rc;
    int64_t grid = (F + kLinkWarps - 1) / kLinkWarps;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    if (grid < 1) grid = 1;
    if (events) cudaEventRecord((cudaEvent_t)events[0], st);
    k_links<<<(int)grid, kLinkWarps * 32, 0, st>>>(li, faces, F, map, d_n_map, bmap, lengths);
    rc = check_launch("k_links");
    if (events) cudaEventRecord((cudaEvent_t)events[1], st);
    return rc;
}

}  // namespace vf
