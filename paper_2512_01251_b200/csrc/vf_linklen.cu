// vf_linklen.cu -- cut-link lengths (pin A17).
//
// FACE-parallel formulation.  A link (lattice node v of a mapped finest-level
// block, direction c_q, 0 < d <= dx) is accepted when the eps-cube around its
// piercing point v + d c_q overlaps the face (exact SAT), and the LUT keeps the
// minimum q = d/dx over faces.  Instead of every cell scanning its block's
// all-directions bin (the paper's per-cell loop), every face enumerates the
// nodes that can pierce it and min-merges q into the LUT with atomicMin on the
// IEEE bits -- order-free, hence deterministic and equal to the per-cell
// minimum (for q > 0 the uint32 order is the float order, and the -1.0f
// initialisation 0xBF800000 sorts above every positive float, so "no hit"
// needs no finalisation pass).  A dense block map of the finest level replaces
// the bin lookup; the all-directions binning drops out of the embed path (the
// result is invariant to it; the oracle uses the MD bins).
//
// K-link, per warp and chunk of 32 faces:
//   1. lane-parallel face setup into shared memory (struct-of-arrays: lanes
//      reading different faces hit different banks): sweep axis a = dominant
//      normal component, column range, slab half-width, 2D edge functions of
//      the face projected along a.
//   2. the items (column, slab position) of the 32 faces are flattened so the
//      32 lanes stay busy whatever the face sizes; per node an FP32
//      pre-filter (|num| <= |c.n| dx, piercing point inside the projected
//      triangle, margins >= 10x the FP32 error bound) keeps candidates.
//   3. candidates enter a per-warp shared-memory queue that is drained 32 at a
//      time through the exact FP64 path, so the SAT runs warp-converged.
// The pre-filter only ever passes a superset of the exact decisions; every
// stored value comes from the exact path, bit-identical to the oracle.
#include <math.h>

#include "vf_common.cuh"
#include "vf_internal.h"

namespace vf {

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
constexpr int kQueue = 32 + 32 * 13;

// per-warp face table, struct-of-arrays
struct LinkFaces {
    double v1[3][32];
    float nf[3][32];
    float ea[3][32], eb[3][32], ec[3][32];  // inward unit edge functions (u,w plane)
    float Ef[32];                            // FP32 error bound of num (absolute)
    float Tf[32];                            // slab half-width for |num|
    int f[32], ax[32], cu0[32], cw0[32], ncu[32], span[32], a1a[32], b1a[32];
    int pref[33];
};

__device__ __forceinline__ int floor_idx(double xs) { return (int)floor(xs); }

__global__ void __launch_bounds__(kLinkWarps * 32)
    k_links(LevelInfo li, double inv_dx, int widen, const double *__restrict__ faces, int64_t F,
            const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map,
            const int32_t *__restrict__ bmap, float *__restrict__ lengths) {
    __shared__ LinkFaces s_tab[kLinkWarps];
    __shared__ int4 s_q[kLinkWarps][kQueue];
    const int64_t n = d_n_map ? (int64_t)*d_n_map : F;
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kLinkWarps + wib;
    const int64_t nw = (int64_t)gridDim.x * kLinkWarps;
    const double dx = li.dx, eps = li.eps;
    const float dxf = (float)dx;
    LinkFaces &T = s_tab[wib];
    int qn = 0;  // warp-uniform queue length

    for (int64_t chunk = gw * 32; chunk < n; chunk += nw * 32) {
        // ---- 1. face setup, one face per lane --------------------------------
        const int64_t m = chunk + lane;
        int total = 0;
        if (m < n) {
            const int64_t f = map ? (int64_t)map[m] : m;
            double v[9], nn[3];
            load_face(faces, f, v, nn);
            int a1[3], b1[3];
            double ext = 0.0;
            bool empty = false;
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                const double lo = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
                const double hi = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
                ext = fmax(ext, hi - lo);
                // nodes whose centres can lie in [lo - dx - 2eps, hi + dx + 2eps]
                // (superset; inv_dx is exact for power-of-two dx, else widened)
                int ia = floor_idx((lo - dx - 2.0 * eps) * inv_dx - 0.5) - widen;
                int ib = floor_idx((hi + dx + 2.0 * eps) * inv_dx - 0.5) + 1 + widen;
                ia = max(ia, 0);
                ib = min(ib, li.cells[d] - 1);
                a1[d] = ia;
                b1[d] = ib;
                empty |= ia > ib;
            }
            if (!empty) {
                const float nf0 = (float)nn[0], nf1 = (float)nn[1], nf2 = (float)nn[2];
                const float ax0 = fabsf(nf0), ax1 = fabsf(nf1), ax2 = fabsf(nf2);
                const int a = (ax0 >= ax1 && ax0 >= ax2) ? 0 : (ax1 >= ax2 ? 1 : 2);
                const int u = a == 2 ? 0 : a + 1, w = a == 0 ? 2 : a - 1;  // cyclic (a,u,w)
                const float na = a == 0 ? nf0 : (a == 1 ? nf1 : nf2);
                const float Ef = 4e-6f * (float)(ext + 2.0 * dx);
                const float Tf = 1.7320508f * dxf * (1.0f + 1e-5f) + Ef;
                const int span = (int)floorf(2.0f * Tf / (fabsf(na) * dxf)) + 2;
                const int ncu = b1[u] - a1[u] + 1, ncw = b1[w] - a1[w] + 1;
                total = ncu * ncw * span;
                // 2D edge functions in the (u,w) projection, relative to v1
                const float p1u = (float)(v[3 + u] - v[u]), p1w = (float)(v[3 + w] - v[w]);
                const float p2u = (float)(v[6 + u] - v[u]), p2w = (float)(v[6 + w] - v[w]);
                const float cr = p1u * p2w - p1w * p2u;
                const float sg = cr >= 0.0f ? 1.0f : -1.0f;
                const float Pu[3] = {0.0f, p1u, p2u}, Pw[3] = {0.0f, p1w, p2w};
#pragma unroll
                for (int e = 0; e < 3; ++e) {
                    const int e1 = e == 2 ? 0 : e + 1;
                    const float du = Pu[e1] - Pu[e], dw = Pw[e1] - Pw[e];
                    const float len = sqrtf(du * du + dw * dw);
                    const float il = len > 0.0f ? sg / len : 0.0f;
                    T.ea[e][lane] = -dw * il;
                    T.eb[e][lane] = du * il;
                    T.ec[e][lane] = (dw * Pu[e] - du * Pw[e]) * il;
                }
                T.v1[0][lane] = v[0]; T.v1[1][lane] = v[1]; T.v1[2][lane] = v[2];
                T.nf[0][lane] = nf0; T.nf[1][lane] = nf1; T.nf[2][lane] = nf2;
                T.Ef[lane] = Ef;
                T.Tf[lane] = Tf;
                T.f[lane] = (int)f;
                T.ax[lane] = a;
                T.cu0[lane] = a1[u];
                T.cw0[lane] = a1[w];
                T.ncu[lane] = ncu;
                T.span[lane] = span;
                T.a1a[lane] = a1[a];
                T.b1a[lane] = b1[a];
            }
        }
        int incl = total;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
        }
        T.pref[lane + 1] = incl;
        if (lane == 0) T.pref[0] = 0;
        const int grand = __shfl_sync(0xffffffffu, incl, 31);
        __syncwarp();

        // ---- 2. flattened items ---------------------------------------------
        for (int base = 0; base < grand; base += 32) {
            const int g = base + lane;
            uint32_t cand = 0;
            int ni = 0, nj = 0, nk = 0, slot = -1, fid = 0;
            if (g < grand) {
                int lo = 0, hi = 32;  // largest fi with pref[fi] <= g
                while (hi - lo > 1) {
                    const int mid = (lo + hi) >> 1;
                    if (T.pref[mid] <= g) lo = mid;
                    else hi = mid;
                }
                const int fi = lo;
                const int kk = g - T.pref[fi];
                const int a = T.ax[fi];
                const int u = a == 2 ? 0 : a + 1, w = a == 0 ? 2 : a - 1;
                const int span = T.span[fi], ncu = T.ncu[fi];
                const int col = kk / span, sidx = kk - col * span;
                const int iu = T.cu0[fi] + col % ncu, iw = T.cw0[fi] + col / ncu;
                const double va = T.v1[a][fi], vu = T.v1[u][fi], vw = T.v1[w][fi];
                const float na = T.nf[a][fi], nu = T.nf[u][fi], nwv = T.nf[w][fi];
                const float Tf = T.Tf[fi], Ef = T.Ef[fi];
                const float Xu = (float)(node_c(iu, dx) - vu);
                const float Xw = (float)(node_c(iw, dx) - vw);
                const float C = Xu * nu + Xw * nwv;
                // |Xa na + C| <= Tf  <=>  Xa in [(-C - Tf)/na, (-C + Tf)/na]
                float xa0 = (-C - Tf) / na, xa1 = (-C + Tf) / na;
                if (xa0 > xa1) { const float tmp = xa0; xa0 = xa1; xa1 = tmp; }
                const int ia_lo = max(floor_idx(((double)xa0 + va) * inv_dx - 0.5) - widen, T.a1a[fi]);
                const int ia_hi = min(floor_idx(((double)xa1 + va) * inv_dx - 0.5) + 1 + widen, T.b1a[fi]);
                const int ia = ia_lo + sidx;
                if (ia <= ia_hi) {
                    ni = a == 0 ? ia : (u == 0 ? iu : iw);
                    nj = a == 1 ? ia : (u == 1 ? iu : iw);
                    nk = a == 2 ? ia : (u == 2 ? iu : iw);
                    slot = bmap[(ni >> 2) + (int64_t)li.bins[0] * ((nj >> 2) + (int64_t)li.bins[1] * (nk >> 2))];
                }
                if (slot >= 0) {
                    fid = T.f[fi];
                    const float Xa = (float)(node_c(ia, dx) - va);
                    const float numf = -(Xa * na + C);  // (v1 - x).n
                    if (fabsf(numf) <= Tf) {
                        const float ea0 = T.ea[0][fi], eb0 = T.eb[0][fi], ec0 = T.ec[0][fi];
                        const float ea1 = T.ea[1][fi], eb1 = T.eb[1][fi], ec1 = T.ec[1][fi];
                        const float ea2 = T.ea[2][fi], eb2 = T.eb[2][fi], ec2 = T.ec[2][fi];
                        const float base_tol = 1e-5f * dxf + 2.0f * (float)eps;
#pragma unroll
                        for (int r = 0; r < 13; ++r) {
                            const int q = 2 * r + 1;
                            const int cx = c27(q, 0), cy = c27(q, 1), cz = c27(q, 2);
                            const int ca = a == 0 ? cx : (a == 1 ? cy : cz);
                            const int cu = u == 0 ? cx : (u == 1 ? cy : cz);
                            const int cw = w == 0 ? cx : (w == 1 ? cy : cz);
                            const float dn = (float)ca * na + (float)cu * nu + (float)cw * nwv;
                            const float adn = fabsf(dn);
                            bool ok = fabsf(numf) <= fmaf(adn, dxf * (1.0f + 1e-5f), Ef);
                            ok &= adn > 0.0f;  // exact |den| >= 1e-12 |c|
                            const float rd = 1.0f / dn;
                            const float da = numf * rd;  // ~ d
                            const float Pu = Xu + (float)cu * da, Pw = Xw + (float)cw * da;
                            const float tol = fmaf(Ef, fabsf(rd), fmaf(1e-6f, fabsf(da), base_tol));
                            ok &= fmaf(ea0, Pu, fmaf(eb0, Pw, ec0)) >= -tol;
                            ok &= fmaf(ea1, Pu, fmaf(eb1, Pw, ec1)) >= -tol;
                            ok &= fmaf(ea2, Pu, fmaf(eb2, Pw, ec2)) >= -tol;
                            cand |= (uint32_t)ok << r;
                        }
                    }
                }
            }
            // ---- 3. enqueue, drain in full warps ------------------------------
            const int nc = __popc(cand);
            int off = nc;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, off, o);
                if (lane >= o) off += y;
            }
            const int added = __shfl_sync(0xffffffffu, off, 31);
            off += qn - nc;
            for (uint32_t c = cand; c; c &= c - 1)
                s_q[wib][off++] = make_int4(fid, slot, ni | (nj << 16), nk | ((__ffs(c) - 1) << 16));
            qn += added;
            __syncwarp();
            while (qn >= 32) {
                const int4 e = s_q[wib][qn - 32 + lane];
                __syncwarp();
                link_candidate(faces, e.x, e.w >> 16, e.z & 0xffff, e.z >> 16, e.w & 0xffff, dx, eps,
                               li.eps_par, e.y, lengths);
                qn -= 32;
            }
            __syncwarp();
        }
        __syncwarp();
    }
    // drain the remainder
    if (lane < qn) {
        const int4 e = s_q[wib][lane];
        link_candidate(faces, e.x, e.w >> 16, e.z & 0xffff, e.z >> 16, e.w & 0xffff, dx, eps,
                       li.eps_par, e.y, lengths);
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
    if (li.cells[0] > 65535 || li.cells[1] > 65535 || li.cells[2] > 65535)
        return set_error(VF_EARG, "link lengths: > 65535 cells per axis");
    const int64_t nb = (int64_t)li.bins[0] * li.bins[1] * li.bins[2];
    int32_t *bmap = (int32_t *)ws;
    cudaMemsetAsync(bmap, 0xff, sizeof(int32_t) * (size_t)nb, st);
    k_blockmap<<<max_ctas(8), 256, 0, st>>>(L, li.bins[0], li.bins[1], g->d_level_start, g->d_coords,
                                            cmap, bmap);
    int rc = check_launch("k_blockmap");
    if (rc) return rc;
    // 1/dx is exact when dx is a power of two; otherwise widen the ranges by one
    int ex = 0;
    const double mant = frexp(li.dx, &ex);
    const int widen = (mant == 0.5) ? 0 : 1;
    const double inv_dx = 1.0 / li.dx;
    int64_t grid = (F + 32 * kLinkWarps - 1) / (32 * kLinkWarps);
    if (grid > max_ctas(4)) grid = max_ctas(4);
    if (grid < 1) grid = 1;
    if (events) cudaEventRecord((cudaEvent_t)events[0], st);
    k_links<<<(int)grid, kLinkWarps * 32, 0, st>>>(li, inv_dx, widen, faces, F, map, d_n_map, bmap,
                                                  lengths);
    rc = check_launch("k_links");
    if (events) cudaEventRecord((cudaEvent_t)events[1], st);
    return rc;
}

}  // namespace vf
