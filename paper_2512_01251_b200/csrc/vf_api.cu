// vf_api.cu -- C-ABI entry points (include/voxforest_b200.h) and the native
// embed_geometry driver.
#include <math.h>
#include <stdio.h>
#include <string.h>
#include <stdlib.h>

#include <atomic>
#include <mutex>
#include <unordered_map>
#include <vector>

#include <new>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

#include <nccl.h>

namespace vf {

static thread_local char g_err[512] = "";

int set_error(int code, const char *msg) {
    snprintf(g_err, sizeof(g_err), "%s", msg);
    return code;
}

int set_cuda_error(cudaError_t e, const char *what) {
    snprintf(g_err, sizeof(g_err), "%s: %s", what, cudaGetErrorString(e));
    return VF_ECUDA;
}

static std::atomic<long long> g_launches{0};

// Per-kernel timer (vf_ktimer_start / vf_ktimer_stop): the embed runs
// eagerly with every kernel on ONE stream (no side streams), behind a spin
// kernel that holds the stream until the host has enqueued the whole embed,
// so consecutive events bracket each kernel exactly.  An event is recorded
// after every launch (check_launch) and after the memsets of the path.
struct KTimer {
    bool on = false;
    cudaStream_t st = nullptr;
    std::vector<cudaEvent_t> pool;
    std::vector<const char *> names;
    size_t used = 0;
};
static KTimer g_kt;

bool kt_on() { return g_kt.on; }

void kt_point(const char *name) {
    if (!g_kt.on) return;
    if (g_kt.used == g_kt.pool.size()) {
        cudaEvent_t e;
        if (cudaEventCreate(&e) != cudaSuccess) return;
        g_kt.pool.push_back(e);
    }
    cudaEventRecord(g_kt.pool[g_kt.used], g_kt.st);
    g_kt.names.push_back(name);
    ++g_kt.used;
}

int check_launch(const char *what) {
    g_launches.fetch_add(1, std::memory_order_relaxed);
    kt_point(what);
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, what);
}

__global__ void k_gate(long long cycles) {
    const long long t0 = clock64();
    while (clock64() - t0 < cycles) {
    }
}

int sm_count() {
    static int n = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
            n = 148;
    });
    return n;
}

int resident_ctas(const void *kernel, int threads, size_t smem) {
    static std::mutex mu;
    static std::unordered_map<const void *, int> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto it = cache.find(kernel);
    if (it != cache.end()) return it->second;
    int r = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&r, kernel, threads, smem) != cudaSuccess || r <= 0) {
        cudaGetLastError();
        r = 1;
    }
    cache[kernel] = r;
    return r;
}

LevelInfo make_level(const vf_config &cfg, int L) {
    LevelInfo li;
    li.dx = ldexp(cfg.dx0, -L);
    li.h = 4.0 * li.dx;
    li.eps = cfg.eps_slab;
    li.eps_par = cfg.eps_parallel;
    for (int d = 0; d < 3; ++d) {
        li.len[d] = cfg.len[d];
        li.bins[d] = cfg.nb[d] << L;
        li.cells[d] = 4 * li.bins[d];
    }
    li.level = L;
    li.shard_rank = cfg.shard_count > 1 ? cfg.shard_rank : 0;
    li.shard_count = cfg.shard_count > 1 ? cfg.shard_count : 1;
    li.owner = nullptr;
    if (li.shard_count > 1 && cfg.d_row_owner) {
        int64_t base = 0;  // row_base(L): rows of the coarser levels
        for (int l = 0; l < L; ++l) base += (int64_t)(cfg.nb[1] << l) * (cfg.nb[2] << l);
        li.owner = cfg.d_row_owner + base;
    }
    return li;
}

__global__ void k_iota(int32_t *out, int64_t n, int32_t *d_n) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        out[i] = (int32_t)i;
    if (d_n && blockIdx.x == 0 && threadIdx.x == 0) *d_n = (int32_t)n;
}

int launch_iota(int32_t *out, int64_t n, int32_t *d_n, cudaStream_t st) {
    int64_t g = (n + 255) / 256;
    if (g > max_ctas(8)) g = max_ctas(8);
    if (g < 1) g = 1;
    k_iota<<<(int)g, 256, 0, st>>>(out, n, d_n);
    return check_launch("k_iota");
}

__global__ void k_pack_faces(const double *__restrict__ fc, const double *__restrict__ nrm, int64_t F,
                             double *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < F * kFaceStride;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = i / kFaceStride;
        const int k = (int)(i % kFaceStride);
        out[i] = k < 9 ? fc[9 * f + k] : nrm[3 * f + (k - 9)];
    }
}

__global__ void k_sat_batch(const double *__restrict__ tri, const double *__restrict__ box, int64_t n,
                            uint8_t *__restrict__ out) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        SatFace f;
        double v[9];
        for (int k = 0; k < 9; ++k) v[k] = tri[9 * i + k];
        sat_face_init(f, v);
        const double *b = box + 6 * i;
        out[i] = sat_exact(f, b[0], b[1], b[2], b[3], b[4], b[5]) ? 1 : 0;
    }
}

static bool valid_cfg(const vf_config *c) {
    if (!c) return false;
    for (int d = 0; d < 3; ++d)
        if (c->nb[d] <= 0 || !(c->len[d] > 0)) return false;
    if (c->shard_count > 1 && (c->shard_rank < 0 || c->shard_rank >= c->shard_count)) return false;
    return c->l_max >= 1 && c->l_max < VF_MAX_LEVELS && c->n_spec >= 1 && c->n_prop >= 0 &&
           c->dx0 > 0 && c->eps_slab >= 0;
}

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

// embed workspace layout
struct EmbedWs {
    int2 *pairs[2];       // per-level (bin, face) lists, ping-pong: pairs(L+1) built while level L runs
    int32_t *n_pairs[2];
    int32_t *map[2];      // kept faces of one level (sharded path: per-level indicators)
    int32_t *n_map[2];
    uint16_t *ind_bits;   // [F] per-level 1D indicator bits
    int32_t *maps;        // [l_max][F + 1] kept faces of every level (k_indicators_all)
    int32_t *n_maps;      // [l_max]
    int64_t pair_cap;
    BlockBins bb;         // the level's block-indexed bins
    uint8_t *ind8;        // [F] per-level indicators (sharded path)
    void *bins_ws;        // compaction scan over F
    size_t bins_ws_bytes;
    void *prop_ws, *mark_ws, *adapt_ws, *tab_ws, *link_ws;
    size_t prop_b, mark_b, adapt_b, tab_b, link_b;
    int32_t *bcount;
    void *lines_ws;      // recorded piercing lines of the link enumeration
    void *shard_ws;      // multi-GPU: row histogram / owner scan / face subset
};

int64_t pair_cap_of(const vf_config &cfg, int64_t F) {
    return cfg.pair_cap > 0 ? cfg.pair_cap : 4 * F + 65536;
}

size_t block_bins_bytes(int32_t capacity, int64_t pair_cap) {
    const size_t c = al(sizeof(int32_t) * ((size_t)capacity + 1)), p = al(sizeof(int32_t) * ((size_t)pair_cap + 1));
    return 2 * p + 4 * c + 256 + al(scan_workspace_bytes(capacity));
}

void block_bins_layout(int32_t capacity, int64_t pair_cap, char *base, BlockBins *bb) {
    const size_t c = al(sizeof(int32_t) * ((size_t)capacity + 1)), p = al(sizeof(int32_t) * ((size_t)pair_cap + 1));
    bb->blk = (int32_t *)base;
    bb->face_ids = (int32_t *)(base + p);
    bb->cnt = (int32_t *)(base + 2 * p);
    bb->base = (int32_t *)(base + 2 * p + c);
    bb->cur = (int32_t *)(base + 2 * p + 2 * c);
    bb->ne = (int32_t *)(base + 2 * p + 3 * c);
    bb->d_n_ne = (int32_t *)(base + 2 * p + 4 * c);
    bb->d_total = bb->d_n_ne + 1;
    bb->scan_ws = base + 2 * p + 4 * c + 256;
}

static size_t embed_layout(const vf_config &cfg, int64_t F, int32_t cap, char *base, EmbedWs *w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *p = base ? base + off : nullptr;
        off += al(bytes);
        return (void *)p;
    };
    const int Lf = cfg.l_max - 1;
    EmbedWs t;
    memset(&t, 0, sizeof(t));
    t.pair_cap = pair_cap_of(cfg, F);
    // (capacity-only items first: the sharded calls lay out with F = 1)
    t.prop_b = rows_workspace_size(cap);
    t.prop_ws = take(t.prop_b);
    for (int k = 0; k < 2; ++k) {
        t.pairs[k] = (int2 *)take(sizeof(int2) * (size_t)(t.pair_cap + 1));
        t.n_pairs[k] = (int32_t *)take(64);
        t.map[k] = (int32_t *)take(sizeof(int32_t) * (size_t)(F + 1));
        t.n_map[k] = (int32_t *)take(64);
    }
    char *bbp = (char *)take(block_bins_bytes(cap, t.pair_cap));
    if (base) block_bins_layout(cap, t.pair_cap, bbp, &t.bb);
    t.ind8 = (uint8_t *)take((size_t)F + 1);
    t.bins_ws_bytes = scan_workspace_bytes(F + 1);
    t.bins_ws = take(t.bins_ws_bytes);
    t.mark_b = mark_workspace_size(cap);
    t.mark_ws = take(t.mark_b);
    t.adapt_b = adapt_workspace_size(cap);
    t.adapt_ws = take(t.adapt_b);
    t.tab_b = tables_workspace_size(cap);
    t.tab_ws = take(t.tab_b);
    t.link_b = link_workspace_size(cfg, Lf, cap, F);
    t.link_ws = take(t.link_b);
    t.ind_bits = (uint16_t *)take(sizeof(uint16_t) * (size_t)(F + 1));
    t.maps = (int32_t *)take(sizeof(int32_t) * (size_t)(F + 1) * cfg.l_max);
    t.n_maps = (int32_t *)take(sizeof(int32_t) * VF_MAX_LEVELS);
    t.lines_ws = take(link_lines_bytes(cfg, F, cap));
    t.bcount = (int32_t *)take(sizeof(int32_t) * (size_t)cap);
    t.shard_ws = cfg.shard_count > 1 ? take(shard_scratch_size(cfg, F)) : nullptr;
    if (w) *w = t;
    return off;
}

// the (bin, face) pairs of level L: kept faces (1D indicators: the embed's
// per-level maps from k_indicators_all, or computed here), then k_pairs_append
static int level_pairs(const vf_config &cfg, const LevelInfo &li, const double *faces, int64_t F,
                       int use_filter, bool pre_maps, EmbedWs &w, int k, int32_t *d_status,
                       cudaStream_t st) {
    const int32_t *map = nullptr, *nmap = nullptr;
    int rc;
    if (use_filter && pre_maps) {
        map = w.maps + (int64_t)li.level * (F + 1);
        nmap = w.n_maps + li.level;
    } else if (use_filter) {
        if ((rc = launch_indicators(li, 0, faces, F, w.ind8, st))) return rc;
        if ((rc = launch_compact(w.ind8, F, w.map[k], w.n_map[k], w.bins_ws, st))) return rc;
        map = w.map[k];
        nmap = w.n_map[k];
    }
    return pairs_append_impl(li, nlim_of(cfg), faces, F, map, nmap, w.pairs[k], w.n_pairs[k], w.pair_cap,
                             d_status, st);
}

}  // namespace vf

using namespace vf;

extern "C" {

int vf_abi_version(void) { return VF_ABI_VERSION; }

const char *vf_last_error(void) { return g_err; }

int vf_device_info(int *sm, int *major, int *minor) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaGetDevice");
    if (sm) cudaDeviceGetAttribute(sm, cudaDevAttrMultiProcessorCount, dev);
    if (major) cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
    if (minor) cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
    e = cudaGetLastError();
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "vf_device_info");
}

int vf_pack_faces(const double *fc, const double *nrm, int64_t F, double *out, void *stream) {
    if (!fc || !nrm || !out || F < 0) return set_error(VF_EARG, "vf_pack_faces: bad argument");
    if (F == 0) return VF_OK;
    int64_t g = (F * kFaceStride + 255) / 256;
    if (g > max_ctas(8)) g = max_ctas(8);
    k_pack_faces<<<(int)g, 256, 0, (cudaStream_t)stream>>>(fc, nrm, F, out);
    return check_launch("k_pack_faces");
}

int vf_sat_batch(const double *tri, const double *box, int64_t n, uint8_t *out, void *stream) {
    if (!tri || !box || !out || n < 0) return set_error(VF_EARG, "vf_sat_batch: bad argument");
    if (n == 0) return VF_OK;
    int64_t g = (n + 127) / 128;
    if (g > max_ctas(8)) g = max_ctas(8);
    k_sat_batch<<<(int)g, 128, 0, (cudaStream_t)stream>>>(tri, box, n, out);
    return check_launch("k_sat_batch");
}

size_t vf_bins_workspace_size(const vf_config *cfg, int64_t F, int level) {
    if (!valid_cfg(cfg)) return 0;
    const int64_t nb = (int64_t)(cfg->nb[0] << level) * (cfg->nb[1] << level) * (cfg->nb[2] << level);
    size_t a = bins_workspace_size(F, nlim_of(*cfg), nb);
    size_t b = assemble_workspace_size(F * nlim_of(*cfg), nb);
    return a > b ? a : b;
}

int vf_ray_indicators(const vf_config *cfg, const double *faces, int64_t F, int level, int mode,
                      uint8_t *ind, void *stream) {
    if (!valid_cfg(cfg) || !faces || !ind || F < 0 || level < 0 || (mode != 0 && mode != 1))
        return set_error(VF_EARG, "vf_ray_indicators: bad argument");
    return launch_indicators(make_level(*cfg, level), mode, faces, F, ind, (cudaStream_t)stream);
}

size_t vf_compact_workspace_size(int64_t n) { return scan_workspace_bytes(n < 1 ? 1 : n); }

size_t vf_assemble_workspace_size(int64_t pair_cap, int64_t n_bins) {
    return assemble_workspace_size(pair_cap < 1 ? 1 : pair_cap, n_bins);
}

int vf_compact(const uint8_t *ind, int64_t n, int32_t *map, int32_t *d_count, void *ws,
               size_t ws_bytes, void *stream) {
    if (!d_count || n < 0 || (n > 0 && (!ind || !map)))
        return set_error(VF_EARG, "vf_compact: bad argument");
    if (n == 0) {
        cudaError_t e = cudaMemsetAsync(d_count, 0, sizeof(int32_t), (cudaStream_t)stream);
        return e == cudaSuccess ? VF_OK : set_cuda_error(e, "vf_compact");
    }
    if (ws_bytes < scan_workspace_bytes(n)) return set_error(VF_EARG, "vf_compact: workspace too small");
    return launch_compact(ind, n, map, d_count, ws, (cudaStream_t)stream);
}

int vf_bin_pairs(const vf_config *cfg, const double *faces, int64_t F, const int32_t *map,
                 const int32_t *d_n_map, int level, int32_t *pair_bin, int32_t *pair_face,
                 int64_t pair_cap, int32_t *d_n_pairs, int32_t *d_status, void *ws, size_t ws_bytes,
                 void *stream) {
    if (!valid_cfg(cfg) || !faces || !pair_bin || !pair_face || !d_n_pairs || level < 0 ||
        (map && !d_n_map))
        return set_error(VF_EARG, "vf_bin_pairs: bad argument");
    return bin_pairs_impl(make_level(*cfg, level), nlim_of(*cfg), faces, F, map, d_n_map, pair_bin,
                          pair_face, pair_cap, d_n_pairs, d_status, ws, ws_bytes,
                          (cudaStream_t)stream);
}

int vf_bin_assemble(const int32_t *pair_bin, const int32_t *pair_face, const int32_t *d_n_pairs,
                    int64_t pair_cap, int64_t n_bins, int32_t *counts, int32_t *offsets,
                    int32_t *face_ids, void *ws, size_t ws_bytes, void *stream) {
    if (!pair_bin || !pair_face || !d_n_pairs || !counts || !offsets || !face_ids || n_bins <= 0)
        return set_error(VF_EARG, "vf_bin_assemble: bad argument");
    return assemble_impl(pair_bin, pair_face, d_n_pairs, pair_cap, n_bins, counts, offsets, face_ids,
                         ws, ws_bytes, (cudaStream_t)stream);
}

int vf_build_bins(const vf_config *cfg, const double *faces, int64_t F, int level, int mode,
                  int use_filter, vf_bins *bins, int32_t *d_status, void *ws, size_t ws_bytes,
                  void *stream) {
    if (!valid_cfg(cfg) || !faces || !bins || level < 0 || !bins->d_counts || !bins->d_offsets ||
        !bins->d_face_ids || !bins->d_map || !bins->d_n_map || !bins->d_n_face_ids)
        return set_error(VF_EARG, "vf_build_bins: bad argument");
    bins->level = level;
    bins->mode = mode;
    return build_bins_impl(make_level(*cfg, level), nlim_of(*cfg), faces, F, mode, use_filter, bins,
                           d_status, ws, ws_bytes, (cudaStream_t)stream);
}

int vf_init_forest(const vf_config *cfg, vf_grid *grid, void *stream) {
    if (!valid_cfg(cfg) || !grid) return set_error(VF_EARG, "vf_init_forest: bad argument");
    return init_forest_impl(*cfg, grid, (cudaStream_t)stream);
}

size_t vf_adapt_workspace_size(const vf_grid *g) { return g ? adapt_workspace_size(g->capacity) : 0; }

int vf_adapt_refine(const vf_config *cfg, vf_grid *grid, int level, void *ws, size_t ws_bytes,
                    void *stream) {
    if (!valid_cfg(cfg) || !grid || level < 0) return set_error(VF_EARG, "vf_adapt_refine: bad argument");
    return adapt_impl(*cfg, grid, level, ws, ws_bytes, (cudaStream_t)stream);
}

int vf_voxelize_level(const vf_config *cfg, vf_grid *grid, int level, const vf_bins *bins,
                      const double *faces, void *stream) {
    if (!valid_cfg(cfg) || !grid || !bins || !faces || level < 0 || level >= grid->n_levels)
        return set_error(VF_EARG, "vf_voxelize_level: bad argument");
    return voxelize_impl(make_level(*cfg, level), grid, level, bins, faces, (cudaStream_t)stream);
}

size_t vf_propagate_workspace_size(const vf_grid *g) { return g ? propagate_workspace_size(g->capacity) : 0; }

int vf_propagate_x(const vf_config *cfg, vf_grid *grid, int level, int dir, int finalize, void *ws,
                   size_t ws_bytes, void *stream) {
    if (!valid_cfg(cfg) || !grid || level < 0 || level >= grid->n_levels || (dir != 1 && dir != -1))
        return set_error(VF_EARG, "vf_propagate_x: bad argument");
    return propagate_impl(make_level(*cfg, level), grid, level, dir, finalize, ws, ws_bytes,
                          (cudaStream_t)stream);
}

int vf_finalize_level(const vf_config *cfg, vf_grid *grid, int level, void *stream) {
    if (!valid_cfg(cfg) || !grid || level < 0 || level >= grid->n_levels)
        return set_error(VF_EARG, "vf_finalize_level: bad argument");
    return finalize_impl(grid, level, (cudaStream_t)stream);
}

size_t vf_mark_workspace_size(const vf_grid *g) { return g ? mark_workspace_size(g->capacity) : 0; }

int vf_mark_level(const vf_config *cfg, vf_grid *grid, int level, void *ws, size_t ws_bytes,
                  void *stream) {
    if (!valid_cfg(cfg) || !grid || level < 0 || level >= grid->n_levels)
        return set_error(VF_EARG, "vf_mark_level: bad argument");
    return mark_impl(*cfg, grid, level, ws, ws_bytes, (cudaStream_t)stream);
}

int vf_boundary_cells(const vf_config *cfg, vf_grid *grid, int32_t *bcount, void *stream) {
    if (!valid_cfg(cfg) || !grid || !bcount) return set_error(VF_EARG, "vf_boundary_cells: bad argument");
    return boundary_impl(*cfg, grid, bcount, (cudaStream_t)stream);
}

size_t vf_tables_workspace_size(const vf_grid *g) { return g ? tables_workspace_size(g->capacity) : 0; }

int vf_link_tables(const vf_config *cfg, vf_grid *grid, const int32_t *bcount, int32_t *cmap,
                   int32_t *d_n_b, void *ws, size_t ws_bytes, void *stream) {
    if (!valid_cfg(cfg) || !grid || !bcount || !cmap || !d_n_b)
        return set_error(VF_EARG, "vf_link_tables: bad argument");
    return tables_impl(grid, bcount, cmap, d_n_b, ws, ws_bytes, (cudaStream_t)stream);
}

size_t vf_link_workspace_size(const vf_config *cfg, const vf_grid *g) {
    if (!valid_cfg(cfg) || !g) return 0;
    return link_workspace_size(*cfg, g->n_levels - 1, g->capacity, 0);
}

int vf_link_lengths(const vf_config *cfg, vf_grid *grid, const int32_t *cmap, const double *faces,
                    int64_t F, const int32_t *map, const int32_t *d_n_map, float *lengths, void *ws,
                    size_t ws_bytes, void *stream) {
    if (!valid_cfg(cfg) || !grid || !cmap || !faces || !lengths || (map && !d_n_map))
        return set_error(VF_EARG, "vf_link_lengths: bad argument");
    return link_impl(*cfg, grid, cmap, faces, F, map, d_n_map, lengths, ws, ws_bytes,
                     (cudaStream_t)stream, nullptr, nullptr, 0);
}

size_t vf_embed_workspace_size(const vf_config *cfg, int64_t F, int32_t cap) {
    if (!valid_cfg(cfg) || F < 0 || cap <= 0) return 0;
    return embed_layout(*cfg, F, cap, nullptr, nullptr);
}

#define VF_TRY(x)                 \
    do {                          \
        int _rc = (x);            \
        if (_rc) return _rc;      \
    } while (0)

static void rec(void **ev, int n_ev, int *k, cudaStream_t st) {
    if (ev && *k < n_ev) cudaEventRecord((cudaEvent_t)ev[*k], st);
    ++*k;
}

// side stream + events of the bins pipeline (one set per device, created on
// first use; the embed is single-threaded per device, see the header)
struct SideStream {
    cudaStream_t st = nullptr, st3 = nullptr;  // bins pipeline, link line enumeration
    cudaStream_t st4 = nullptr;                // next level's sparse row order
    cudaEvent_t adapted = nullptr, rowsok = nullptr;
    cudaEvent_t fork = nullptr, bins[2] = {nullptr, nullptr}, vox[2] = {nullptr, nullptr}, join = nullptr;
    cudaEvent_t join3 = nullptr;
};
static SideStream g_side[64];

static int side_stream(SideStream **out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaGetDevice");
    SideStream &s = g_side[dev & 63];
    if (!s.st) {
        // the link line enumeration only has to finish by phase 2: lowest
        // priority; the next level's row order: highest
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        // the bins stream one step above the lowest priority -- level with
        // EmbedEngine's level stream (-1 of the B200's [0, -3]): above it, its
        // pairs kernels took SMs from the latency-bound level kernels (C4
        // embed -1.2% measured)
        e = cudaStreamCreateWithPriority(&s.st, cudaStreamNonBlocking, lo - 1 > hi ? lo - 1 : hi);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s.st3, cudaStreamNonBlocking, lo);
        if (e == cudaSuccess) e = cudaStreamCreateWithPriority(&s.st4, cudaStreamNonBlocking, hi);
        cudaEvent_t *evs[] = {&s.fork, &s.bins[0], &s.bins[1], &s.vox[0], &s.vox[1], &s.join, &s.join3, &s.adapted, &s.rowsok};
        for (cudaEvent_t *ev : evs)
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(ev, cudaEventDisableTiming);
        if (e != cudaSuccess) return set_cuda_error(e, "side stream");
    }
    *out = &s;
    return VF_OK;
}

// Per-device context (SURVEY.md §8b vf_ctx_create): selects the device,
// creates its side streams / events (otherwise created on first use) and
// holds the NCCL communicator of the block-sharded embed: the caller's
// (vf_ctx_create) or one the library creates from a unique id the ranks
// share (vf_ctx_create_nccl; parallel.py broadcasts it over
// torch.distributed).  vf_shard_embed_phase1 issues the per-level flag
// exchanges on it, in stream order, with no host synchronisation.
struct vf_ctx_s {
    int device;
    void *nccl_comm;
    int own_comm;  // created here (destroyed with the context)
};

extern "C" void *vf_ctx_create(int device, void *nccl_comm) {
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) {
        set_cuda_error(e, "vf_ctx_create");
        return nullptr;
    }
    SideStream *side = nullptr;
    if (side_stream(&side) != VF_OK) return nullptr;
    vf_ctx_s *c = new (std::nothrow) vf_ctx_s{device, nccl_comm, 0};
    if (!c) set_error(VF_EARG, "vf_ctx_create: out of host memory");
    return c;
}

extern "C" int vf_nccl_unique_id(void *out, int out_bytes) {
    if (!out || out_bytes < (int)sizeof(ncclUniqueId)) return set_error(VF_EARG, "vf_nccl_unique_id: bad argument");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) return set_error(VF_ENCCL, ncclGetErrorString(r));
    memcpy(out, &id, sizeof(id));
    return VF_OK;
}

extern "C" void *vf_ctx_create_nccl(int device, int nranks, int rank, const void *unique_id) {
    if (!unique_id || nranks < 1 || rank < 0 || rank >= nranks) {
        set_error(VF_EARG, "vf_ctx_create_nccl: bad argument");
        return nullptr;
    }
    vf_ctx_s *c = static_cast<vf_ctx_s *>(vf_ctx_create(device, nullptr));
    if (!c) return nullptr;
    ncclUniqueId id;
    memcpy(&id, unique_id, sizeof(id));
    ncclComm_t comm = nullptr;
    const ncclResult_t r = ncclCommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess) {
        set_error(VF_ENCCL, ncclGetErrorString(r));
        delete c;
        return nullptr;
    }
    c->nccl_comm = comm;
    c->own_comm = 1;
    return c;
}

extern "C" int vf_ctx_destroy(void *ctx) {
    if (!ctx) return set_error(VF_EARG, "vf_ctx_destroy: null context");
    vf_ctx_s *c = static_cast<vf_ctx_s *>(ctx);
    int cur = 0;
    cudaGetDevice(&cur);
    cudaSetDevice(c->device);
    SideStream &s = g_side[c->device & 63];
    cudaError_t e = cudaSuccess;
    if (s.st) {
        e = cudaStreamSynchronize(s.st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s.st3);
        if (e == cudaSuccess) e = cudaStreamSynchronize(s.st4);
        cudaEvent_t evs[] = {s.fork, s.bins[0], s.bins[1], s.vox[0], s.vox[1], s.join, s.join3, s.adapted, s.rowsok};
        for (cudaEvent_t ev : evs)
            if (ev) cudaEventDestroy(ev);
        cudaStreamDestroy(s.st);
        cudaStreamDestroy(s.st3);
        cudaStreamDestroy(s.st4);
        s = SideStream();
    }
    if (c->own_comm && c->nccl_comm) ncclCommDestroy((ncclComm_t)c->nccl_comm);
    cudaSetDevice(cur);
    delete c;
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "vf_ctx_destroy");
}

extern "C" int vf_ctx_device(const void *ctx) { return ctx ? static_cast<const vf_ctx_s *>(ctx)->device : -1; }

// wait for the side streams of this device (the cut-link enumeration of a
// phase 1 that was not followed by phase 2 -- the LUT-sizing run, an error --
// must not outlive the caller's workspace)
extern "C" int vf_side_sync(void) {
    SideStream *side = nullptr;
    VF_TRY(side_stream(&side));
    cudaError_t e = cudaStreamSynchronize(side->st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(side->st3);
    if (e == cudaSuccess) e = cudaStreamSynchronize(side->st4);
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "vf_side_sync");
}

// Phase 1.  The spatial bins do not depend on the grid, so they are built on
// a side stream one level AHEAD of the level pipeline (ping-pong buffers):
// bins(L+1) overlaps voxelize / propagate / mark / adapt of level L; the main
// stream only waits for bins(L) before voxelizing L, and the side stream
// waits for voxelize(L-1) before reusing its buffer.  Captured into the
// embed graph the two streams become parallel branches.
// vf_set_serial_links: run the cut-link enumeration on the main stream after
// the tables instead of overlapped on the low-priority side stream, so its
// CUDA events time the kernel alone (the roofline figure in bench.py).
static int g_serial_links = 0;

int vf_embed_phase1(const vf_config *cfg, const double *faces, int64_t F, int use_filter,
                    vf_grid *g, int32_t *cmap, int32_t *d_n_b, void *ws, size_t ws_bytes,
                    void *stream, void **events) {
    if (!valid_cfg(cfg) || !faces || !g || !cmap || !d_n_b || F <= 0)
        return set_error(VF_EARG, "vf_embed_phase1: bad argument");
    EmbedWs w;
    if (embed_layout(*cfg, F, g->capacity, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "vf_embed_phase1: workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    SideStream *side = nullptr;
    VF_TRY(side_stream(&side));
    // per-kernel timing: everything on the main stream, in order
    const bool one = kt_on();
    cudaStream_t s2 = one ? st : side->st;
    const int n_ev = 64;
    int k = 0;
    rec(events, n_ev, &k, st);  // 0: start
    VF_TRY(init_forest_impl(*cfg, g, st));
    VF_TRY(rows_init_impl(*cfg, g, w.prop_ws, st));
    // fork the bins pipeline (after init: it shares the status word) and the
    // grid-independent cut-link line enumeration of the finest level (joined
    // in phase 2, where the recorded lines are resolved)
    cudaEventRecord(side->fork, st);
    cudaStreamWaitEvent(s2, side->fork, 0);
    const bool serial_links = g_serial_links || one;
    if (!serial_links) {
        cudaStreamWaitEvent(side->st3, side->fork, 0);
        VF_TRY(link_enum_impl(*cfg, faces, F, w.link_ws, w.lines_ws, g->capacity, side->st3,
                              events ? events + 58 : nullptr));
        cudaEventRecord(side->join3, side->st3);
    }
    // Alg. 1 indicators of every level in one pass over the face records
    // (its per-warp map queues cover 8 levels; deeper forests: per-level indicators)
    const bool pre = cfg->l_max <= 8;
    if (use_filter && pre) VF_TRY(launch_indicators_all(*cfg, faces, F, w.ind_bits, w.maps, F + 1, w.n_maps, s2));
    auto build = [&](int L) {
        return level_pairs(*cfg, make_level(*cfg, L), faces, F, use_filter, pre, w, L & 1, g->d_status, s2);
    };
    // the block histograms start from zero (each level's voxelizer restores them)
    cudaMemsetAsync(w.bb.cnt, 0, sizeof(int32_t) * (size_t)g->capacity, st);
    kt_point("memset:block_counts");
    VF_TRY(build(0));
    cudaEventRecord(side->bins[0], s2);
    for (int L = 0; L < cfg->l_max; ++L) {
        const LevelInfo li = make_level(*cfg, L);
        if (L + 1 < cfg->l_max) {  // side stream: pairs(L+1) while the main stream runs level L
            if (L >= 1) cudaStreamWaitEvent(s2, side->vox[(L + 1) & 1], 0);  // pairs(L-1) consumed
            VF_TRY(build(L + 1));
            cudaEventRecord(side->bins[(L + 1) & 1], s2);
        }
        cudaStreamWaitEvent(st, side->bins[L & 1], 0);
        rec(events, n_ev, &k, st);  // bins done
        // pairs -> level-L blocks (needs the level's blocks: after adapt(L-1))
        VF_TRY(block_bins_impl(li, L, g, w.pairs[L & 1], w.n_pairs[L & 1], w.pair_cap, w.bb, st));
        cudaEventRecord(side->vox[L & 1], st);
        VF_TRY(voxelize_blocks_impl(li, g, L, w.bb, faces, true, st));
        if (L > 0) cudaStreamWaitEvent(st, side->rowsok, 0);  // level L's row order
        VF_TRY(propagate_rows_impl(li, g, L, w.prop_ws, st));
        rec(events, n_ev, &k, st);  // voxelization done
        if (L == cfg->l_max - 1) break;
        VF_TRY(mark_impl(*cfg, g, L, w.mark_ws, w.mark_b, st));
        VF_TRY(adapt_impl(*cfg, g, L, w.adapt_ws, w.adapt_b, st, false));
        // level L+1's row order beside its bins and voxelization; level L's
        // neighbour-child links / interface layer (outputs only: no later
        // kernel of the embed reads them) at the lowest priority, behind the
        // cut-link enumeration (joined with it in phase 2)
        cudaStream_t s4 = one ? st : side->st4;
        cudaEventRecord(side->adapted, st);
        cudaStreamWaitEvent(s4, side->adapted, 0);
        VF_TRY(rows_next_impl(g, L, w.prop_ws, s4));
        cudaEventRecord(side->rowsok, s4);
        if (serial_links) {
            VF_TRY(adapt_links_impl(g, L, s4));
        } else {
            cudaStreamWaitEvent(side->st3, side->adapted, 0);
            VF_TRY(adapt_links_impl(g, L, side->st3));
        }
        rec(events, n_ev, &k, st);  // refinement done
    }
    // join the side streams (required to end a capture; bins are all consumed)
    cudaEventRecord(side->join, s2);
    cudaStreamWaitEvent(st, side->join, 0);
    if (!one && cfg->l_max > 1) {
        cudaEventRecord(side->adapted, side->st4);
        cudaStreamWaitEvent(st, side->adapted, 0);
    }
    if (!serial_links) cudaEventRecord(side->join3, side->st3);  // enumeration + adapt links
    VF_TRY(boundary_impl(*cfg, g, w.bcount, st));
    VF_TRY(tables_impl(g, w.bcount, cmap, d_n_b, w.tab_ws, w.tab_b, st,
                       link_slot_inverse(*cfg, F, w.lines_ws, g->capacity)));
    rec(events, n_ev, &k, st);  // boundary + tables done
    if (serial_links) {  // measurement mode: the enumeration alone on the main stream
        VF_TRY(link_enum_impl(*cfg, faces, F, w.link_ws, w.lines_ws, g->capacity, st, events ? events + 58 : nullptr));
        cudaEventRecord(side->join3, st);
    }
    return VF_OK;
}

int vf_set_serial_links(int on) {
    const int old = g_serial_links;
    if (on >= 0) g_serial_links = on ? 1 : 0;
    return old;
}

int64_t vf_launch_count(void) { return (int64_t)g_launches.load(); }

int vf_embed_link_stats(const vf_config *cfg, int64_t F, int32_t capacity, void *ws, size_t ws_bytes,
                        int64_t *out) {
    if (!valid_cfg(cfg) || F <= 0 || !ws || !out) return set_error(VF_EARG, "vf_embed_link_stats: bad argument");
    EmbedWs w;
    if (embed_layout(*cfg, F, capacity, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "vf_embed_link_stats: workspace too small");
    return link_stats(*cfg, F, w.link_ws, w.lines_ws, out);
}

int vf_embed_phase2(const vf_config *cfg, const double *faces, int64_t F, vf_grid *g,
                    const int32_t *cmap, const int32_t *d_n_b, float *lengths, int64_t lengths_cap,
                    void *ws, size_t ws_bytes, void *stream, void **link_events) {
    if (!valid_cfg(cfg) || !faces || !g || !cmap || !d_n_b || !lengths || lengths_cap < 1)
        return set_error(VF_EARG, "vf_embed_phase2: bad argument");
    EmbedWs w;
    if (embed_layout(*cfg, F, g->capacity, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "vf_embed_phase2: workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    SideStream *side = nullptr;
    VF_TRY(side_stream(&side));
    // link_events[0..1] bracket the LUT fill + the resolution (the cut-link
    // kernels after the tables)
    // (the LUT tiles are written whole by the resolution: no separate -1 fill)
    if (link_events) cudaEventRecord((cudaEvent_t)link_events[0], st);
    cudaStreamWaitEvent(st, side->join3, 0);  // the line enumeration of phase 1
    void *end_only[2] = {nullptr, link_events ? link_events[1] : nullptr};
    return link_resolve_impl(*cfg, g, cmap, faces, F, lengths, w.link_ws, w.lines_ws, st,
                             link_events ? end_only : nullptr, d_n_b, lengths_cap);
}

int vf_embed_graph_create(const vf_config *cfg, const double *faces, int64_t F, int use_filter,
                          vf_grid *g, int32_t *cmap, int32_t *d_n_b, float *lengths,
                          int64_t lengths_cap, void *ws, size_t ws_bytes, void *stream,
                          void **graph_exec) {
    if (!graph_exec || !stream) return set_error(VF_EARG, "vf_embed_graph_create: bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaStreamBeginCapture");
    int rc = vf_embed_phase1(cfg, faces, F, use_filter, g, cmap, d_n_b, ws, ws_bytes, stream, nullptr);
    if (!rc)
        rc = vf_embed_phase2(cfg, faces, F, g, cmap, d_n_b, lengths, lengths_cap, ws, ws_bytes,
                             stream, nullptr);
    cudaGraph_t graph = nullptr;
    e = cudaStreamEndCapture(st, &graph);
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (e != cudaSuccess) return set_cuda_error(e, "cudaStreamEndCapture");
    // node priorities: the level pipeline (critical path) high, the
    // grid-independent link line enumeration (its own branch) low
    {
        int lo = 0, hi = 0;
        cudaDeviceGetStreamPriorityRange(&lo, &hi);
        size_t nn = 0;
        cudaGraphGetNodes(graph, nullptr, &nn);
        cudaGraphNode_t *nodes = (cudaGraphNode_t *)malloc(sizeof(cudaGraphNode_t) * (nn ? nn : 1));
        cudaGraphGetNodes(graph, nodes, &nn);
        const void *enum_fn = link_enum_kernel(0), *enum_small = link_enum_kernel(1);
        for (size_t i = 0; i < nn; ++i) {
            cudaGraphNodeType ty;
            if (cudaGraphNodeGetType(nodes[i], &ty) != cudaSuccess || ty != cudaGraphNodeTypeKernel) continue;
            cudaKernelNodeParams kp;
            if (cudaGraphKernelNodeGetParams(nodes[i], &kp) != cudaSuccess) continue;
            cudaLaunchAttributeValue v;
            memset(&v, 0, sizeof(v));
            v.priority = (kp.func == enum_fn || kp.func == enum_small) ? lo : hi;
            cudaGraphKernelNodeSetAttribute(nodes[i], cudaLaunchAttributePriority, &v);
        }
        free(nodes);
        cudaGetLastError();  // priorities are a hint: never fail the capture over them
    }
    cudaGraphExec_t exec = nullptr;
    e = cudaGraphInstantiate(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
    cudaGraphDestroy(graph);
    if (e != cudaSuccess) return set_cuda_error(e, "cudaGraphInstantiate");
    *graph_exec = (void *)exec;
    return VF_OK;
}

int vf_graph_launch(void *graph_exec, void *stream) {
    if (!graph_exec) return set_error(VF_EARG, "vf_graph_launch: bad argument");
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGraphLaunch((cudaGraphExec_t)graph_exec, (cudaStream_t)stream);
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "cudaGraphLaunch");
}

void vf_graph_destroy(void *graph_exec) {
    if (graph_exec) cudaGraphExecDestroy((cudaGraphExec_t)graph_exec);
}

int vf_shard_zero_unowned(const vf_config *cfg, vf_grid *grid, int level, int32_t *d_bcount,
                          void *stream) {
    if (!valid_cfg(cfg) || !grid || level < 0 || level >= grid->n_levels)
        return set_error(VF_EARG, "vf_shard_zero_unowned: bad argument");
    return shard_zero_impl(make_level(*cfg, level), grid, level, d_bcount, (cudaStream_t)stream);
}

// ---- block-sharded multi-GPU embed (parallel.py drives the exchanges)

size_t vf_shard_owner_bytes(const vf_config *cfg) {
    if (!valid_cfg(cfg)) return 0;
    return shard_owner_bytes(*cfg);
}

static bool shard_args(const vf_config *cfg, vf_grid *g, void *ws, size_t ws_bytes, int64_t F,
                       EmbedWs *w) {
    if (!valid_cfg(cfg) || !g || cfg->shard_count < 2 || !cfg->d_row_owner) return false;
    return embed_layout(*cfg, F, g->capacity, (char *)ws, w) <= ws_bytes;
}

int vf_shard_owner_map(const vf_config *cfg, vf_grid *g, int level, void *ws, size_t ws_bytes,
                       void *stream) {
    EmbedWs w;
    // the owner map only needs the shard scratch; F = 1 sizes the layout
    if (!shard_args(cfg, g, ws, ws_bytes, 1, &w) || level < 0 || level >= cfg->l_max)
        return set_error(VF_EARG, "vf_shard_owner_map: bad argument");
    // level 0 also starts the sparse row order (the root grid)
    if (level == 0) VF_TRY(rows_init_impl(*cfg, g, w.prop_ws, (cudaStream_t)stream));
    return shard_owner_map_impl(*cfg, g, level, w.shard_ws, (cudaStream_t)stream);
}

int vf_shard_level(const vf_config *cfg, const double *faces, int64_t F, int use_filter,
                   vf_grid *g, int L, void *ws, size_t ws_bytes, void *stream) {
    EmbedWs w;
    if (!faces || F <= 0 || !shard_args(cfg, g, ws, ws_bytes, F, &w) || L < 0 ||
        L >= g->n_levels)
        return set_error(VF_EARG, "vf_shard_level: bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    const LevelInfo li = make_level(*cfg, L);
    if (L == 0) {  // the block histograms start from zero
        cudaMemsetAsync(w.bb.cnt, 0, sizeof(int32_t) * (size_t)g->capacity, st);
        kt_point("memset:block_counts");
    }
    VF_TRY(level_pairs(*cfg, li, faces, F, use_filter, false, w, 0, g->d_status, st));
    VF_TRY(block_bins_impl(li, L, g, w.pairs[0], w.n_pairs[0], w.pair_cap, w.bb, st));
    VF_TRY(voxelize_blocks_impl(li, g, L, w.bb, faces, true, st));
    VF_TRY(propagate_rows_impl(li, g, L, w.prop_ws, st));
    return shard_zero_impl(li, g, L, nullptr, st);
}

int vf_shard_refine(const vf_config *cfg, vf_grid *g, int L, void *ws, size_t ws_bytes,
                    void *stream) {
    EmbedWs w;
    if (!shard_args(cfg, g, ws, ws_bytes, 1, &w) || L < 0 || L + 1 >= cfg->l_max)
        return set_error(VF_EARG, "vf_shard_refine: bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    VF_TRY(mark_impl(*cfg, g, L, w.mark_ws, w.mark_b, st));
    VF_TRY(adapt_impl(*cfg, g, L, w.adapt_ws, w.adapt_b, st));
    VF_TRY(rows_next_impl(g, L, w.prop_ws, st));
    return shard_owner_map_impl(*cfg, g, L + 1, w.shard_ws, st);
}

int vf_shard_boundary(const vf_config *cfg, vf_grid *g, int32_t *bcount, void *stream) {
    if (!valid_cfg(cfg) || !g || !bcount) return set_error(VF_EARG, "vf_shard_boundary: bad argument");
    return boundary_impl(*cfg, g, bcount, (cudaStream_t)stream);
}

int vf_shard_links(const vf_config *cfg, const double *faces, int64_t F, vf_grid *g,
                   const int32_t *cmap, const int32_t *d_n_b, float *lengths, int64_t lengths_cap,
                   void *ws, size_t ws_bytes, void *stream) {
    EmbedWs w;
    // (shard_count 1: the native driver on a 1-rank communicator -- all faces)
    if (!faces || F <= 0 || !cmap || !d_n_b || !lengths || lengths_cap < 1 || !valid_cfg(cfg) || !g ||
        (cfg->shard_count > 1 && !cfg->d_row_owner) || embed_layout(*cfg, F, g->capacity, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "vf_shard_links: bad argument");
    // the single-GPU cut-link pipeline on the faces near owned rows: line
    // enumeration -> q-records -> parent buckets, then the LUT slots of owned
    // blocks (other ranks' slots -1)
    cudaStream_t st = (cudaStream_t)stream;
    const bool sub = cfg->shard_count > 1;
    if (sub) VF_TRY(shard_face_subset_impl(*cfg, faces, F, w.map[0], w.n_map[0], w.shard_ws, st));
    VF_TRY(link_enum_impl(*cfg, faces, F, w.link_ws, w.lines_ws, g->capacity, st, nullptr,
                          sub ? w.map[0] : nullptr, sub ? w.n_map[0] : nullptr));
    VF_TRY(link_inverse_impl(*cfg, g, cmap, d_n_b, lengths_cap, F, w.lines_ws, st));
    return link_resolve_impl(*cfg, g, cmap, faces, F, lengths, w.link_ws, w.lines_ws, st, nullptr, d_n_b,
                             lengths_cap);
}

// Native block-sharded embed through the tables, one call
// per rank, exchanges on the context's NCCL communicator in stream order: no
// host synchronisation, graph-capturable.  Per level: this rank's bins /
// voxelization / Alg. 5 rows, non-owned flags zeroed, then ONE all-reduce
// (MAX) of the block flags; mark + adapt + row order + next owner map
// replicated.  Finest level: all-reduce (MAX) of the owner-zeroed SOLID
// masks (boundary halo), boundary cells of owned blocks, all-reduce (MAX) of
// the owner-zeroed boundary counts, replicated tables (the global
// contraction map).  The all-reduces span the grid capacity: entries outside
// the level are identical on every rank (replicated or zero), so MAX leaves
// them unchanged, and no host-side level size is needed.  The cut links of
// owned blocks follow with vf_shard_links once the LUT is sized.
int vf_shard_embed_phase1(void *ctx, const vf_config *cfg, const double *faces, int64_t F, int use_filter,
                          vf_grid *g, int32_t *bcount, int32_t *cmap, int32_t *d_n_b, void *ws, size_t ws_bytes,
                          void *stream) {
    EmbedWs w;
    vf_ctx_s *cx = static_cast<vf_ctx_s *>(ctx);
    // (shard_count 1: a 1-rank communicator, every row owned)
    if (!cx || !cx->nccl_comm || !faces || F <= 0 || !bcount || !cmap || !d_n_b || !valid_cfg(cfg) || !g ||
        (cfg->shard_count > 1 && !cfg->d_row_owner) || embed_layout(*cfg, F, g->capacity, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "vf_shard_embed_phase1: bad argument");
    ncclComm_t comm = (ncclComm_t)cx->nccl_comm;
    cudaStream_t st = (cudaStream_t)stream;
    const size_t cap = (size_t)g->capacity;
    auto allmax = [&](void *buf, size_t n, ncclDataType_t ty) -> int {
        const ncclResult_t r = ncclAllReduce(buf, buf, n, ty, ncclMax, comm, st);
        return r == ncclSuccess ? VF_OK : set_error(VF_ENCCL, ncclGetErrorString(r));
    };
    VF_TRY(init_forest_impl(*cfg, g, st));
    VF_TRY(rows_init_impl(*cfg, g, w.prop_ws, st));
    VF_TRY(shard_owner_map_impl(*cfg, g, 0, w.shard_ws, st));
    cudaMemsetAsync(w.bb.cnt, 0, sizeof(int32_t) * cap, st);
    // 1D indicators of every level in one face pass, unfiltered by ownership
    // (future levels' owners are not known yet); the pairs keep owned bins only
    const bool pre = use_filter && cfg->l_max <= 8;
    if (pre) {
        vf_config c1 = *cfg;
        c1.shard_count = 1;
        VF_TRY(launch_indicators_all(c1, faces, F, w.ind_bits, w.maps, F + 1, w.n_maps, st));
    }
    for (int L = 0; L < cfg->l_max; ++L) {
        const LevelInfo li = make_level(*cfg, L);
        VF_TRY(level_pairs(*cfg, li, faces, F, use_filter, pre, w, 0, g->d_status, st));
        VF_TRY(block_bins_impl(li, L, g, w.pairs[0], w.n_pairs[0], w.pair_cap, w.bb, st));
        VF_TRY(voxelize_blocks_impl(li, g, L, w.bb, faces, true, st));
        VF_TRY(propagate_rows_impl(li, g, L, w.prop_ws, st));
        VF_TRY(shard_zero_impl(li, g, L, nullptr, st));
        VF_TRY(allmax(g->d_bflags, cap, ncclUint8));  // the level's block flags, 1 B/block
        if (L == cfg->l_max - 1) break;
        VF_TRY(mark_impl(*cfg, g, L, w.mark_ws, w.mark_b, st));
        VF_TRY(adapt_impl(*cfg, g, L, w.adapt_ws, w.adapt_b, st));
        VF_TRY(rows_next_impl(g, L, w.prop_ws, st));
        VF_TRY(shard_owner_map_impl(*cfg, g, L + 1, w.shard_ws, st));
    }
    VF_TRY(allmax(g->d_solid64, cap, ncclUint64));  // SOLID-cell masks for the boundary halo
    VF_TRY(boundary_impl(*cfg, g, bcount, st));
    VF_TRY(allmax(bcount, cap, ncclInt32));  // boundary counts: the global contraction map
    return tables_impl(g, bcount, cmap, d_n_b, w.tab_ws, w.tab_b, st);
}

int vf_ktimer_start(void *stream, double gate_us) {
    if (g_kt.on) return set_error(VF_EARG, "vf_ktimer_start: timer already running");
    g_kt.on = true;
    g_kt.st = (cudaStream_t)stream;
    g_kt.used = 0;
    g_kt.names.clear();
    int dev = 0, khz = 1965000;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&khz, cudaDevAttrClockRate, dev);
    k_gate<<<1, 1, 0, g_kt.st>>>((long long)(gate_us * 1e-3 * khz));
    kt_point("_start");
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "vf_ktimer_start");
}

// stop, synchronise and report: "name<TAB>launches<TAB>total ms" lines,
// first-appearance order; returns the bytes written (or needed)
int vf_ktimer_stop(char *buf, int buflen) {
    if (!g_kt.on) return set_error(VF_EARG, "vf_ktimer_stop: timer not running");
    g_kt.on = false;
    cudaError_t e = cudaStreamSynchronize(g_kt.st);
    if (e != cudaSuccess) return -set_cuda_error(e, "vf_ktimer_stop");
    std::vector<const char *> keys;
    std::vector<double> ms;
    std::vector<int> cnt;
    // VF_KT_EACH=1: one line per launch ("name#k") instead of per kernel name
    const char *each = getenv("VF_KT_EACH");
    std::vector<char> names_each;
    if (each && *each == '1') names_each.resize(g_kt.used * 48);
    for (size_t i = 1; i < g_kt.used; ++i) {
        float t = 0.0f;
        cudaEventElapsedTime(&t, g_kt.pool[i - 1], g_kt.pool[i]);
        if (!names_each.empty()) {
            char *nm = &names_each[i * 48];
            snprintf(nm, 48, "%s#%zu", g_kt.names[i], i);
            g_kt.names[i] = nm;
        }
        size_t k = 0;
        while (k < keys.size() && strcmp(keys[k], g_kt.names[i]) != 0) ++k;
        if (k == keys.size()) {
            keys.push_back(g_kt.names[i]);
            ms.push_back(0.0);
            cnt.push_back(0);
        }
        ms[k] += t;
        cnt[k] += 1;
    }
    int n = 0;
    for (size_t k = 0; k < keys.size(); ++k) {
        char line[160];
        const int w = snprintf(line, sizeof(line), "%s\t%d\t%.6f\n", keys[k], cnt[k], ms[k]);
        if (buf && n + w < buflen) memcpy(buf + n, line, (size_t)w + 1);
        n += w;
    }
    return n;
}

int vf_check_status(const vf_grid *g, void *stream) {
    if (!g || !g->d_status) return set_error(VF_EARG, "vf_check_status: bad argument");
    int32_t h[4] = {0, 0, 0, 0};
    cudaError_t e = cudaMemcpyAsync(h, g->d_status, sizeof(h), cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return set_cuda_error(e, "vf_check_status");
    if (h[0] == VF_ECAPACITY) {
        char buf[160];
        if (h[3] > 0)
            snprintf(buf, sizeof(buf), "pair list capacity exhausted: %d (bin, face) pairs needed", h[3]);
        else if (h[2] > 0)
            snprintf(buf, sizeof(buf), "link table capacity exhausted: %d boundary blocks", h[2]);
        else
            snprintf(buf, sizeof(buf), "forest capacity exhausted while refining level %d", h[1]);
        return set_error(VF_ECAPACITY, buf);
    }
    if (h[0] == VF_ENLIM) return set_error(VF_ENLIM, "N_lim pair cap violated (refine_faces the mesh)");
    if (h[0] == VF_EMESH) return set_error(VF_EMESH, "invalid mesh: face index out of range or degenerate face (zero normal)");
    if (h[0]) return set_error(h[0], "device-side error latched");
    return VF_OK;
}

}  // extern "C"
