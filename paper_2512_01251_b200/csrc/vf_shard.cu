// vf_shard.cu -- block-sharded multi-GPU embed: balanced
// contiguous ownership of level-L block rows and the face subset of a rank's
// cut links.
//
//   K-rowhist  blocks per block row (j, k) of level L (replicated topology,
//              so every rank computes the same histogram)
//   K-rowown   owner[row] = rank whose 1/N share of the level's blocks holds
//              the row's first block: contiguous row ranges (row = j + B_y k),
//              balanced to within one row; a face, an x-run and a 3x3 block
//              neighbourhood then touch the rows of one or two ranks
//   K-facesub  faces with a lattice node of an owned row within one link
//              (the candidate node range of k_links), compacted into the
//              map k_links takes -- each rank enumerates ~F/N faces
#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

__global__ void k_row_hist(int L, LevelInfo li, const int32_t *__restrict__ level_start,
                           const int32_t *__restrict__ coords, int32_t *__restrict__ counts) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int4 c = reinterpret_cast<const int4 *>(coords)[b];
        atomicAdd(&counts[c.y + (int64_t)li.bins[1] * c.z], 1);
    }
}

__global__ void k_row_assign(int64_t rows, const int32_t *__restrict__ excl,
                             const int32_t *__restrict__ d_total, int n_ranks,
                             uint8_t *__restrict__ owner) {
    const int64_t total = *d_total;
    for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < rows;
         r += (int64_t)gridDim.x * blockDim.x) {
        const int64_t o = total > 0 ? ((int64_t)excl[r] * n_ranks) / total : 0;
        owner[r] = (uint8_t)(o < n_ranks ? o : n_ranks - 1);
    }
}

struct LoadRows {
    const int32_t *p;
    __device__ int operator()(int64_t i) const { return p[i]; }
};
struct EmitRows {
    int32_t *out;
    __device__ void operator()(int64_t i, int, int ex) const { out[i] = ex; }
};

size_t shard_owner_bytes(const vf_config &cfg) {
    int64_t n = 0;
    for (int l = 0; l < cfg.l_max; ++l) n += (int64_t)(cfg.nb[1] << l) * (cfg.nb[2] << l);
    return (size_t)n;
}

size_t shard_scratch_size(const vf_config &cfg, int64_t F) {
    const int Lf = cfg.l_max - 1;
    const int64_t rows = (int64_t)(cfg.nb[1] << Lf) * (cfg.nb[2] << Lf);
    const int64_t n = rows > F ? rows : F;
    return 2 * (((size_t)(rows + 1) * sizeof(int32_t) + 255) & ~(size_t)255) + 256 +
           ((scan_workspace_bytes(n + 1) + 255) & ~(size_t)255) + (((size_t)F + 256) & ~(size_t)255);
}

int shard_owner_map_impl(const vf_config &cfg, vf_grid *g, int L, void *scratch, cudaStream_t st) {
    const LevelInfo li = make_level(cfg, L);
    if (li.shard_count <= 1 || !li.owner) return VF_OK;
    const int Lf = cfg.l_max - 1;
    const int64_t rows_f = (int64_t)(cfg.nb[1] << Lf) * (cfg.nb[2] << Lf);
    const size_t rb = ((size_t)(rows_f + 1) * sizeof(int32_t) + 255) & ~(size_t)255;
    int32_t *counts = (int32_t *)scratch;
    int32_t *excl = (int32_t *)((char *)scratch + rb);
    int32_t *total = (int32_t *)((char *)scratch + 2 * rb);
    void *scan_ws = (char *)scratch + 2 * rb + 256;
    const int64_t rows = (int64_t)li.bins[1] * li.bins[2];
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)rows, st);
    k_row_hist<<<max_ctas(8), 256, 0, st>>>(L, li, g->d_level_start, g->d_coords, counts);
    int rc = check_launch("k_row_hist");
    if (rc) return rc;
    cudaError_t e = scan_launch(LoadRows{counts}, EmitRows{excl}, rows, nullptr, total, scan_ws, st);
    if (e != cudaSuccess) return set_cuda_error(e, "row scan");
    int64_t grid = (rows + 255) / 256;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_row_assign<<<(int)grid, 256, 0, st>>>(rows, excl, total, li.shard_count,
                                            const_cast<uint8_t *>(li.owner));
    return check_launch("k_row_assign");
}

// faces whose k_links candidate nodes (face AABB +- one link) reach an owned
// row of the finest level
__global__ void k_face_near_owned(LevelInfo li, double inv_dx, int widen,
                                  const double *__restrict__ faces, int64_t F,
                                  uint8_t *__restrict__ keep) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F;
         f += (int64_t)gridDim.x * blockDim.x) {
        double v[9], n[3];
        load_face(faces, f, v, n);
        int lo[3], hi[3];
#pragma unroll
        for (int d = 1; d < 3; ++d) {
            const double flo = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
            const double fhi = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
            lo[d] = max((int)floor((flo - li.dx - 2.0 * li.eps) * inv_dx - 0.5) - widen, 0) >> 2;
            hi[d] = min((int)floor((fhi + li.dx + 2.0 * li.eps) * inv_dx - 0.5) + 1 + widen,
                        li.cells[d] - 1) >> 2;
        }
        bool k_ = false;
        for (int k = lo[2]; k <= hi[2] && !k_; ++k)
            for (int j = lo[1]; j <= hi[1]; ++j)
                if (owns_row(li, j, k)) { k_ = true; break; }
        keep[f] = k_;
    }
}

int shard_face_subset_impl(const vf_config &cfg, const double *faces, int64_t F, int32_t *map,
                           int32_t *d_n_map, void *scratch, cudaStream_t st) {
    const int Lf = cfg.l_max - 1;
    const LevelInfo li = make_level(cfg, Lf);
    const int64_t rows_f = (int64_t)(cfg.nb[1] << Lf) * (cfg.nb[2] << Lf);
    const int64_t n = rows_f > F ? rows_f : F;
    const size_t rb = ((size_t)(rows_f + 1) * sizeof(int32_t) + 255) & ~(size_t)255;
    void *scan_ws = (char *)scratch + 2 * rb + 256;
    uint8_t *keep = (uint8_t *)((char *)scan_ws + ((scan_workspace_bytes(n + 1) + 255) & ~(size_t)255));
    int ex = 0;
    const int widen = (frexp(li.dx, &ex) == 0.5) ? 0 : 1;
    int64_t grid = (F + 255) / 256;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_face_near_owned<<<(int)grid, 256, 0, st>>>(li, 1.0 / li.dx, widen, faces, F, keep);
    int rc = check_launch("k_face_near_owned");
    if (rc) return rc;
    return launch_compact(keep, F, map, d_n_map, scan_ws, st);
}

}  // namespace vf
