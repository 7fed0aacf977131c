// vf_internal.h -- host-side glue shared by the .cu translation units.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/voxforest_b200.h"
#include "vf_common.cuh"

namespace vf {

// error plumbing (thread-local message, vf_last_error)
int set_error(int code, const char *msg);
int set_cuda_error(cudaError_t e, const char *what);
int check_launch(const char *what);
// per-kernel timing (vf_ktimer_*): an event on the timed stream after each
// launch / memset while the timer is on; no-op otherwise
void kt_point(const char *name);
bool kt_on();

int sm_count();
inline int max_ctas(int per_sm) { return sm_count() * per_sm; }
// CTAs of `kernel` resident per SM at this block size (occupancy API, cached)
int resident_ctas(const void *kernel, int threads, size_t smem = 0);
// one full wave of a grid-stride kernel: SMs x resident CTAs (a grid that is
// not a whole number of waves leaves the last wave partly idle)
template <typename K>
int wave_ctas(K kernel, int threads, size_t smem = 0) {
    return sm_count() * resident_ctas(reinterpret_cast<const void *>(kernel), threads, smem);
}
// grid sizes (CTAs per SM) of grid-stride kernels (build-time tunables)
#ifndef VF_GRID_PAIRS
#define VF_GRID_PAIRS 8
#endif
#ifndef VF_GRID_RESOLVE
#define VF_GRID_RESOLVE 8
#endif
#ifndef VF_GRID_XS4
#define VF_GRID_XS4 8
#endif

LevelInfo make_level(const vf_config &cfg, int L);
inline int nlim_of(const vf_config &cfg) {
    const int a = 2 + cfg.n_spec;
    return a * a * a;
}

int launch_iota(int32_t *out, int64_t n, int32_t *d_n, cudaStream_t st);

// scans
int launch_compact(const uint8_t *ind, int64_t n, int32_t *map, int32_t *d_count, void *ws,
                   cudaStream_t st);
int launch_compact_bits(const uint16_t *bits, int L, int64_t n, int32_t *map, int32_t *d_count,
                        void *ws, cudaStream_t st);
int launch_exclusive_scan(const int32_t *in, int64_t n_bound, const int32_t *d_n, int32_t *out,
                          int32_t *d_total, void *ws, cudaStream_t st);

// bins
int launch_indicators(const LevelInfo &li, int mode, const double *faces, int64_t F,
                      uint8_t *out, cudaStream_t st);
size_t bins_workspace_size(int64_t F, int nlim, int64_t n_bins);
size_t assemble_workspace_size(int64_t pair_cap, int64_t n_bins);
int build_bins_impl(const LevelInfo &li, int nlim, const double *faces, int64_t F, int mode,
                    int use_filter, vf_bins *bins, int32_t *d_status, void *ws, size_t ws_bytes,
                    cudaStream_t st, const uint16_t *ind_bits = nullptr, bool sorted = true);
// 1D indicators of every level in one pass (bit L of out[f])
struct LevelSet {
    LevelInfo li[VF_MAX_LEVELS];
    double inv_dx[VF_MAX_LEVELS];
    int widen[VF_MAX_LEVELS];
    int n;
};
// out: bit L of out[f]; maps (nullable): level L's kept faces at
// maps + L * map_stride, count n_maps[L] (unordered, from the bits)
int launch_indicators_all(const vf_config &cfg, const double *faces, int64_t F, uint16_t *out,
                          int32_t *maps, int64_t map_stride, int32_t *n_maps, cudaStream_t st);
int sort_bins(int64_t n_bins, const int32_t *offsets, const int32_t *d_total, int32_t *counts,
              int32_t *face_ids, int32_t *large, int32_t *scalars, int32_t *scratch,
              cudaStream_t st);
int bin_pairs_impl(const LevelInfo &li, int nlim, const double *faces, int64_t F,
                   const int32_t *map, const int32_t *d_n_map, int32_t *pair_bin,
                   int32_t *pair_face, int64_t pair_cap, int32_t *d_n_pairs, int32_t *d_status,
                   void *ws, size_t ws_bytes, cudaStream_t st);
int assemble_impl(const int32_t *pair_bin, const int32_t *pair_face, const int32_t *d_n_pairs,
                  int64_t pair_cap, int64_t n_bins, int32_t *counts, int32_t *offsets,
                  int32_t *face_ids, void *ws, size_t ws_bytes, cudaStream_t st);

// block-indexed bins of one level (the embed's bins; pin A4): the bin faces
// of level-local block u are face_ids[base[u] .. base[u] + cnt[u]); ne lists
// the blocks with at least one face (unordered)
struct BlockBins {
    int32_t *blk;       // [pair_cap] level-local block of each pair (-1: no block)
    int32_t *face_ids;  // [pair_cap] grouped by block
    int32_t *cnt;       // [capacity] pairs per block (all zero between levels)
    int32_t *base;      // [capacity] first face_ids slot of the block
    int32_t *cur;       // [capacity] scatter cursors
    int32_t *ne;        // [capacity] nonempty blocks
    int32_t *d_n_ne;    // [1]
    int32_t *d_total;   // [1] pairs kept
    void *scan_ws;      // scan over capacity
};
size_t block_bins_bytes(int32_t capacity, int64_t pair_cap);
void block_bins_layout(int32_t capacity, int64_t pair_cap, char *base, BlockBins *bb);
// embed pairs: compact (bin, face) list of one level (k_pairs' accepted set)
int pairs_append_impl(const LevelInfo &li, int nlim, const double *faces, int64_t F,
                      const int32_t *map, const int32_t *d_n_map, int2 *pairs, int32_t *d_n_pairs,
                      int64_t cap, int32_t *d_status, cudaStream_t st);
// pairs -> level-L blocks (forest descent), counts, scan, scatter
int block_bins_impl(const LevelInfo &li, int L, vf_grid *g, const int2 *pairs,
                    const int32_t *d_n_pairs, int64_t cap, const BlockBins &bb, cudaStream_t st);

// voxelizer
// block-indexed bins (embed): zero_cnt restores bb.cnt to zero for the next level
int voxelize_blocks_impl(const LevelInfo &li, vf_grid *g, int L, const BlockBins &bb,
                         const double *faces, bool zero_cnt, cudaStream_t st);
// dense BinLevel (SPEC op partial_surface_voxelize): gathered per block first
int voxelize_impl(const LevelInfo &li, vf_grid *g, int L, const vf_bins *bins,
                  const double *faces, cudaStream_t st);
size_t propagate_workspace_size(int32_t capacity);
int propagate_impl(const LevelInfo &li, vf_grid *g, int L, int dir, int finalize, void *ws,
                   size_t ws_bytes, cudaStream_t st);
int finalize_impl(vf_grid *g, int L, cudaStream_t st);
int shard_zero_impl(const LevelInfo &li, vf_grid *g, int L, int32_t *bcount, cudaStream_t st);
// sparse block rows (vf_rows.cu): level 0 after init_forest, level L+1 after
// adapt(L); Alg. 5 (+x, -x for L > 0) + finalize of level L over them
size_t rows_workspace_size(int32_t capacity);
int rows_init_impl(const vf_config &cfg, vf_grid *g, void *ws, cudaStream_t st);
int rows_next_impl(vf_grid *g, int L, void *ws, cudaStream_t st);
int propagate_rows_impl(const LevelInfo &li, vf_grid *g, int L, void *ws, cudaStream_t st);

// forest
int init_forest_impl(const vf_config &cfg, vf_grid *g, cudaStream_t st);
size_t mark_workspace_size(int32_t capacity);
int mark_impl(const vf_config &cfg, vf_grid *g, int L, void *ws, size_t ws_bytes,
              cudaStream_t st);
size_t adapt_workspace_size(int32_t capacity);
// links = false: the trailing neighbour-child / interface kernel is left to
// the caller (adapt_links_impl, after the children)
int adapt_impl(const vf_config &cfg, vf_grid *g, int L, void *ws, size_t ws_bytes,
               cudaStream_t st, bool links = true);
int adapt_links_impl(vf_grid *g, int L, cudaStream_t st);

// boundary / tables / links
int boundary_impl(const vf_config &cfg, vf_grid *g, int32_t *bcount, cudaStream_t st);
size_t tables_workspace_size(int32_t capacity);
// inv (nullable): slot -> block id of every mapped block
int tables_impl(vf_grid *g, const int32_t *bcount, int32_t *cmap, int32_t *d_n_b, void *ws,
                size_t ws_bytes, cudaStream_t st, int32_t *inv = nullptr);
size_t link_workspace_size(const vf_config &cfg, int finest, int32_t capacity, int64_t F);
int link_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
              int64_t F, const int32_t *map, const int32_t *d_n_map, float *lengths, void *ws,
              size_t ws_bytes, cudaStream_t st, void **events, const int32_t *d_n_b,
              int64_t lengths_cap);
// multi-GPU sharding (vf_shard.cu)
size_t shard_owner_bytes(const vf_config &cfg);
size_t shard_scratch_size(const vf_config &cfg, int64_t F);
int shard_owner_map_impl(const vf_config &cfg, vf_grid *g, int L, void *scratch, cudaStream_t st);
int shard_face_subset_impl(const vf_config &cfg, const double *faces, int64_t F, int32_t *map,
                           int32_t *d_n_map, void *scratch, cudaStream_t st);
// embed split of the link lengths: grid-independent line enumeration (side
// stream, early) + resolution once the grid and the LUT slots exist
size_t link_lines_bytes(const vf_config &cfg, int64_t F, int32_t capacity);
const void *link_enum_kernel(int small);  // graph node priorities
int link_stats(const vf_config &cfg, int64_t F, void *ws, void *lines_ws, int64_t out[7]);
int link_enum_impl(const vf_config &cfg, const double *faces, int64_t F, void *ws, void *lines_ws,
                   int32_t capacity, cudaStream_t st, void **events, const int32_t *map = nullptr,
                   const int32_t *d_n_map = nullptr);
int link_inverse_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const int32_t *d_n_b, int64_t cap,
                      int64_t F, void *lines_ws, cudaStream_t st);
// inv: slot -> finest block (tables_impl's inverse output; nullptr: the
// lines workspace's copy, link_slot_inverse)
int link_resolve_impl(const vf_config &cfg, vf_grid *g, const int32_t *cmap, const double *faces,
                      int64_t F, float *lengths, void *ws, void *lines_ws, cudaStream_t st,
                      void **events, const int32_t *d_n_b, int64_t lengths_cap, const int32_t *inv = nullptr);
int32_t *link_slot_inverse(const vf_config &cfg, int64_t F, void *lines_ws, int32_t capacity);
int fill_lut_impl(const int32_t *d_n_b, float *lengths, int64_t cap, int32_t *d_status,
                  cudaStream_t st);

}  // namespace vf
