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

__global__ void __launch_bounds__(64)
    k_boundary(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ nbr,
               uint8_t *__restrict__ bflags, uint8_t *__restrict__ masks,
               int32_t *__restrict__ bcount) {
    __shared__ int32_t s_nb[27];
    __shared__ int s_cand;
    const int32_t s = level_start[L], e = level_start[L + 1];
    const int t = threadIdx.x;
    const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
    for (int64_t b = s + blockIdx.x; b < e; b += gridDim.x) {
        if (t < 27) s_nb[t] = (t == 0) ? (int32_t)b : nbr[27 * b + t];
        __syncthreads();
        if (t == 0) s_cand = 0;
        __syncthreads();
        if (t < 27) {
            const int32_t v = s_nb[t];
            if (v >= 0 && (bflags[v] & VF_BF_SOLID)) s_cand = 1;
        }
        __syncthreads();
        const bool cand = s_cand;
        bool bnd = false;
        if (cand && masks[64 * b + t] == VF_FLUID) {
            for (int q = 1; q < 27 && !bnd; ++q) {
                const int ux = I + c27(q, 0), uy = J + c27(q, 1), uz = K + c27(q, 2);
                // A15: I' = mod(4 + mod(I + c, 4), 4); neighbour block direction
                const int dxs = (ux < 0 || ux > 3) ? c27(q, 0) : 0;
                const int dys = (uy < 0 || uy > 3) ? c27(q, 1) : 0;
                const int dzs = (uz < 0 || uz > 3) ? c27(q, 2) : 0;
                const int32_t nbk = s_nb[slot_of(dxs, dys, dzs)];
                if (nbk < 0) continue;
                const int tt = (ux & 3) + 4 * (uy & 3) + 16 * (uz & 3);
                bnd = masks[64 * (int64_t)nbk + tt] == VF_SOLID;
            }
        }
        const int cnt = __syncthreads_count(bnd);
        if (bnd) masks[64 * b + t] = VF_BOUNDARY;
        if (t == 0) {
            bcount[b] = cnt;
            const uint8_t f = bflags[b];
            bflags[b] = (uint8_t)(cnt > 0 ? (f | VF_BF_BOUNDARY) : (f & ~VF_BF_BOUNDARY));
        }
        __syncthreads();
    }
}

int boundary_impl(vf_grid *g, int32_t *bcount, cudaStream_t st) {
    const int L = g->n_levels - 1;
    cudaMemsetAsync(bcount, 0, sizeof(int32_t) * (size_t)g->capacity, st);
    k_boundary<<<max_ctas(24), 64, 0, st>>>(L, g->d_level_start, g->d_nbr, g->d_bflags,
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

__global__ void __launch_bounds__(128)
    k_links(LevelInfo li, const double *__restrict__ faces, int64_t F,
            const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map,
            const int32_t *__restrict__ bmap, float *__restrict__ lengths) {
    const int64_t n = d_n_map ? (int64_t)*d_n_map : F;
    const double dx = li.dx, eps = li.eps;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = map ? (int64_t)map[m] : m;
        double v[9], nn[3];
        load_face(faces, f, v, nn);
        SatFace sf;
        sat_face_init(sf, v);
        int a[3], b[3];
        bool empty = false;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
            double fa = floor(VF_DDIV(sf.lo[d], dx)) - 1.0, fb = floor(VF_DDIV(sf.hi[d], dx)) + 1.0;
            fa = fmax(fa, 0.0);
            fb = fmin(fb, (double)(li.cells[d] - 1));
            if (fa > fb) empty = true;
            a[d] = (int)fa;
            b[d] = (int)fb;
        }
        if (empty) continue;
        // 13 representative directions (odd slots): den and |den|*dx
        double den[13];
        uint32_t valid = 0;
#pragma unroll
        for (int r = 0; r < 13; ++r) {
            const int q = 2 * r + 1;
            const double c0 = c27(q, 0), c1 = c27(q, 1), c2 = c27(q, 2);
            const double cn = __dsqrt_rn(VF_DADD(VF_DADD(VF_DMUL(c0, c0), VF_DMUL(c1, c1)), VF_DMUL(c2, c2)));
            den[r] = VF_DADD(VF_DADD(VF_DMUL(c0, nn[0]), VF_DMUL(c1, nn[1])), VF_DMUL(c2, nn[2]));
            if (!(fabs(den[r]) < VF_DMUL(li.eps_par, cn))) valid |= 1u << r;
        }
        for (int k = a[2]; k <= b[2]; ++k) {
            const double z = node_c(k, dx);
            for (int j = a[1]; j <= b[1]; ++j) {
                const double y = node_c(j, dx);
                for (int i = a[0]; i <= b[0]; ++i) {
                    const int32_t slot =
                        bmap[(i >> 2) + (int64_t)li.bins[0] * ((j >> 2) + (int64_t)li.bins[1] * (k >> 2))];
                    if (slot < 0) continue;
                    const double x = node_c(i, dx);
                    const double num = plane_num(v, nn, x, y, z);
                    if (num == 0.0) continue;  // d = 0 is never a link (0 < d)
                    const double anum = fabs(num);
                    const int t = (i & 3) + 4 * (j & 3) + 16 * (k & 3);
#pragma unroll 1
                    for (int r = 0; r < 13; ++r) {
                        if (!(valid >> r & 1)) continue;
                        // |d| > 2dx for sure -> neither direction of the pair
                        if (anum > VF_DMUL(2.0 * dx, fabs(den[r]))) continue;
                        const double d = VF_DDIV(num, den[r]);
                        // d > 0: slot q = 2r+1; d < 0: opposite slot, d' = -d
                        // exactly (den' = -den bitwise), v + d'c' == v + d c
                        const bool pos = d > 0.0;
                        const double dd = pos ? d : -d;
                        if (!(dd > 0.0 && dd <= dx)) continue;
                        const int q = pos ? 2 * r + 1 : 2 * r + 2;
                        const double c0 = c27(q, 0), c1 = c27(q, 1), c2 = c27(q, 2);
                        const double xi = VF_DADD(x, VF_DMUL(dd, c0));
                        const double yi = VF_DADD(y, VF_DMUL(dd, c1));
                        const double zi = VF_DADD(z, VF_DMUL(dd, c2));
                        if (!sat_exact(sf, VF_DSUB(xi, eps), VF_DSUB(yi, eps), VF_DSUB(zi, eps),
                                       VF_DADD(xi, eps), VF_DADD(yi, eps), VF_DADD(zi, eps)))
                            continue;
                        const float qv = __double2float_rn(VF_DDIV(dd, dx));
                        atomicMin(reinterpret_cast<unsigned int *>(lengths) +
                                      ((int64_t)slot * 27 + q) * 64 + t,
                                  __float_as_uint(qv));
                    }
                }
            }
        }
    }
}

size_t link_workspace_size(const vf_config &cfg, int finest) {
    const int64_t nb = (int64_t)(cfg.nb[0] << finest) * (cfg.nb[1] << finest) * (cfg.nb[2] << finest);
    return ((size_t)nb * sizeof(int32_t) + 255) & ~(size_t)255;
}

int link_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
              int64_t F, const int32_t *map, const int32_t *d_n_map, float *lengths, void *ws,
              size_t ws_bytes, cudaStream_t st) {
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
    int64_t grid = (F + 127) / 128;
    if (grid > max_ctas(16)) grid = max_ctas(16);
    if (grid < 1) grid = 1;
    k_links<<<(int)grid, 128, 0, st>>>(li, faces, F, map, d_n_map, bmap, lengths);
    return check_launch("k_links");
}

}  // namespace vf
