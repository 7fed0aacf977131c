// vf_rows.cu -- Alg. 5 (+x / -x external propagation) and
// finalize over SPARSE block rows.
//
// Each level keeps its blocks in row order: rid[] lists the level's block
// ids grouped by block row (j, k) and sorted by x inside a row, rows[] the
// (first position, length) of every row that holds at least one block, and
// rrow[] the row of each position.  A row's x-runs (Alg. 5's chains of
// same-level blocks) are its maximal stretches of consecutive x.  The order
// is derived level by level without sorting, from the forest's structure:
// the children of a level-L row (j, k) fill exactly the 4 level-(L+1) rows
// (2j + dy, 2k + dz), each holding the children (2x, 2x + 1) of the row's
// refined blocks in x order.  With g = the exclusive count of refined blocks
// in row order and (g0, m) = the row's first count and its number of refined
// blocks, the child (dx, dy, dz) of the refined block at position p goes to
// position 8 g0 + (dy + 2 dz) 2m + 2 (g[p] - g0) + dx.  Level 0 is the root
// grid (ids are i + N_x (j + N_y k): rows are contiguous already).
//
// Memory is O(blocks) per level (no dense B_L^3 level map), and the row
// kernel touches only existing blocks.
#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"
#include "vf_rowops.cuh"

namespace vf {

struct RowSet {
    int32_t *rid;    // [capacity] block ids in row order
    int32_t *rrow;   // [capacity] row of each position
    int2 *rows;      // [capacity] (first position, length)
    int32_t *n_rows; // [1] (for level L > 0: the count of non-empty parent rows; x 4)
};

struct RowWs {
    RowSet set[2];  // level parity
    int32_t *g;     // [capacity] exclusive refined counts in row order (level L)
    int32_t *gtot;  // [1]
    int32_t *rank;  // [capacity] rank of each non-empty row of level L
    void *scan_ws;
};

static size_t al(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t rows_layout(int32_t cap, char *base, RowWs *w) {
    const size_t a = al(sizeof(int32_t) * ((size_t)cap + 1));
    size_t off = 0;
    auto take = [&](size_t b) {
        char *p = base ? base + off : nullptr;
        off += al(b);
        return p;
    };
    RowWs t;
    for (int k = 0; k < 2; ++k) {
        t.set[k].rid = (int32_t *)take(a);
        t.set[k].rrow = (int32_t *)take(a);
        t.set[k].rows = (int2 *)take(2 * a);
        t.set[k].n_rows = (int32_t *)take(64);
    }
    t.g = (int32_t *)take(a);
    t.gtot = (int32_t *)take(64);
    t.rank = (int32_t *)take(a);
    t.scan_ws = take(scan_workspace_bytes(cap));
    if (w) *w = t;
    return off;
}

size_t rows_workspace_size(int32_t capacity) { return rows_layout(capacity, nullptr, nullptr); }

// row count of level L: the root rows, or 4 per non-empty parent row
__device__ __forceinline__ int64_t rows_of(const int32_t *n_rows, int L) { return L == 0 ? *n_rows : 4ll * *n_rows; }

__global__ void k_rows_init(int nx, int ny, int nz, RowSet rs) {
    const int64_t n = (int64_t)nx * ny * nz, nr = (int64_t)ny * nz;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
        rs.rid[p] = (int32_t)p;
        rs.rrow[p] = (int32_t)(p / nx);
        if (p < nr) rs.rows[p] = make_int2((int32_t)(p * nx), nx);
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) *rs.n_rows = (int32_t)nr;
}

int rows_init_impl(const vf_config &cfg, vf_grid *g, void *ws, cudaStream_t st) {
    RowWs w;
    rows_layout(g->capacity, (char *)ws, &w);
    const int64_t n = (int64_t)cfg.nb[0] * cfg.nb[1] * cfg.nb[2];
    int grid = (int)((n + 255) / 256);
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_rows_init<<<grid, 256, 0, st>>>(cfg.nb[0], cfg.nb[1], cfg.nb[2], w.set[0]);
    return check_launch("k_rows_init");
}

// scan 1: refined flags of level L in row order
struct LoadRefined {
    const int32_t *rid, *child;
    __device__ int operator()(int64_t p) const { return child[rid[p]] >= 0 ? 1 : 0; }
};
struct EmitG {
    int32_t *g;
    __device__ void operator()(int64_t p, int, int ex) const { g[p] = ex; }
};

// scan 2: non-empty rows of level L -> the 4 child rows of each
__device__ __forceinline__ void row_gm(const RowSet &rs, const int32_t *g, const int32_t *gtot, int64_t nL,
                                       int64_t r, int32_t &g0, int32_t &m) {
    const int2 row = rs.rows[r];
    g0 = g[row.x];
    const int64_t end = (int64_t)row.x + row.y;
    m = (end < nL ? g[end] : *gtot) - g0;
}
struct LoadRowNonEmpty {
    RowSet rs;
    const int32_t *g, *gtot, *level_start;
    int L;
    __device__ int operator()(int64_t r) const {
        int32_t g0, m;
        row_gm(rs, g, gtot, (int64_t)level_start[L + 1] - level_start[L], r, g0, m);
        return m > 0 ? 1 : 0;
    }
};
struct EmitChildRows {
    RowSet rs, nx;
    const int32_t *g, *gtot, *level_start;
    int32_t *rank;
    int L;
    __device__ void operator()(int64_t r, int v, int ex) const {
        rank[r] = ex;
        if (!v) return;
        int32_t g0, m;
        row_gm(rs, g, gtot, (int64_t)level_start[L + 1] - level_start[L], r, g0, m);
#pragma unroll
        for (int q = 0; q < 4; ++q) nx.rows[4 * (int64_t)ex + q] = make_int2(8 * g0 + q * 2 * m, 2 * m);
    }
};
struct RowsN {
    const int32_t *n_rows;
    int L;
    __device__ int64_t operator()() const { return rows_of(n_rows, L); }
};

// children of level L's refined blocks into level L+1's row order
__global__ void __launch_bounds__(256)
    k_rows_children(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ child,
                    RowSet rs, RowSet nx, const int32_t *__restrict__ g, const int32_t *__restrict__ gtot,
                    const int32_t *__restrict__ rank) {
    const int64_t nL = (int64_t)level_start[L + 1] - level_start[L];
    const int64_t nN = (int64_t)level_start[L + 2] - level_start[L + 1];  // 0 if the level was dropped
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nL; p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t c = child[rs.rid[p]];
        if (c < 0) continue;
        const int32_t r = rs.rrow[p];
        int32_t g0, m;
        row_gm(rs, g, gtot, nL, r, g0, m);
        const int64_t k = g[p] - g0;
        const int32_t cr = 4 * rank[r];
#pragma unroll
        for (int o = 0; o < 8; ++o) {
            const int dx = o & 1, q = o >> 1;  // q = dy + 2 dz
            const int64_t pos = 8ll * g0 + (int64_t)q * 2 * m + 2 * k + dx;
            if (pos >= nN) continue;
            nx.rid[pos] = c + o;
            nx.rrow[pos] = cr + q;
        }
    }
}

int rows_next_impl(vf_grid *g, int L, void *ws, cudaStream_t st) {
    RowWs w;
    rows_layout(g->capacity, (char *)ws, &w);
    const RowSet &rs = w.set[L & 1], &nx = w.set[(L + 1) & 1];
    cudaError_t e = scan_launch_fn(LoadRefined{rs.rid, g->d_child}, EmitG{w.g}, (int64_t)g->capacity,
                                   ScanLevelN{g->d_level_start, L}, w.gtot, w.scan_ws, st);
    kt_point("scan_kernel");
    if (e != cudaSuccess) return set_cuda_error(e, "row order scan");
    e = scan_launch_fn(LoadRowNonEmpty{rs, w.g, w.gtot, g->d_level_start, L},
                       EmitChildRows{rs, nx, w.g, w.gtot, g->d_level_start, w.rank, L}, (int64_t)g->capacity,
                       RowsN{rs.n_rows, L}, nx.n_rows, w.scan_ws, st);
    kt_point("scan_kernel");
    if (e != cudaSuccess) return set_cuda_error(e, "row list scan");
    k_rows_children<<<max_ctas(8), 256, 0, st>>>(L, g->d_level_start, g->d_child, rs, nx, w.g, w.gtot, w.rank);
    return check_launch("k_rows_children");
}

// ---------------------------------------------------------------------------
// Alg. 5 over the sorted rows (warp per row), + finalize.  Per 32-block
// chunk: transfer functions of the blocks (row_fn), a warp segmented scan
// with compose() -- segments start at run starts (a block whose x-predecessor
// in the row is not a level-L block: it carries f_b(sigma) from its back
// neighbour's code) and at lane 0, which continues the
// previous chunk's run -- the status entering each block, the fill, and on
// the last pass the finalize.  Same f_b, composition and apply as the
// pointer-jumping operators (vf_voxelize.cu).
template <int DIR>
__device__ __forceinline__ void xrow_pass_sorted(int L, int lane, const int32_t *__restrict__ rid, int32_t st0,
                                                 int32_t len, const int32_t *__restrict__ coords,
                                                 const int32_t *__restrict__ nbr, uint8_t *__restrict__ masks,
                                                 bool finalize, uint8_t *__restrict__ bflags,
                                                 uint64_t *__restrict__ solid64) {
    constexpr int back = DIR > 0 ? 2 : 1, trail = DIR > 0 ? 3 : 0;
    uint32_t carry = 0;  // status leaving the last block of the previous chunk
    int prev_x = -2;     // x of that block (-2: none)
    for (int c0 = 0; c0 < len; c0 += 32) {
        const bool present = c0 + lane < len;
        const int idx = DIR > 0 ? c0 + lane : len - 1 - (c0 + lane);
        const int32_t id = present ? rid[st0 + idx] : -1;
        const int x = present ? coords[4 * (int64_t)id] : -1000000;
        int px = __shfl_up_sync(0xffffffffu, x, 1);
        if (lane == 0) px = prev_x;
        const bool pred = present && px == x - DIR;  // x-predecessor (pass order) is a level-L block
        uint32_t w[16];
        uint32_t fn = 0;
        bool head = true;
        if (present) {
            load_masks64(masks, id, w);
            uint32_t A, B;
            row_fn(w, trail, A, B);
            fn = A | (B << 16);
            if (!pred) {  // run start: back neighbour is not a level-L block
                const int32_t code = nbr[27 * (int64_t)id + back];
                const uint32_t c = (code == VF_NB_SOLID_NBR) ? A : B;  // f_b(sigma)
                fn = c | (c << 16);
            } else if (lane == 0) {  // continue the previous chunk's run
                fn = compose(fn, carry | (carry << 16));
            } else {
                head = false;
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t gq = __shfl_up_sync(0xffffffffu, fn, o);
            const int hd = __shfl_up_sync(0xffffffffu, (int)head, o);
            if (lane >= o && !head) {
                fn = compose(fn, gq);
                head = hd;
            }
        }
        const uint32_t out = fn & 0xffffu;  // constant: status leaving this block
        uint32_t s = __shfl_up_sync(0xffffffffu, out, 1);
        if (lane == 0) s = carry;
        if (present) {
            bool changed = false;
            if (pred) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t xw = row_apply(w[r], (s >> r) & 1u, L == 0);
                    changed |= (xw != w[r]);
                    w[r] = xw;
                }
            }
            if (finalize) finalize_block(w, changed, bflags, solid64, id);
            if (changed) store_masks64(masks, id, w);
        }
        carry = __shfl_sync(0xffffffffu, out, 31);
        prev_x = __shfl_sync(0xffffffffu, x, 31);
    }
}

constexpr int kRowWarps = 8;
#ifndef VF_XROWS_MINB
#define VF_XROWS_MINB 1
#endif

__global__ void __launch_bounds__(kRowWarps * 32, VF_XROWS_MINB)
    k_xrows(LevelInfo li, int L, RowSet rs, const int32_t *__restrict__ level_start,
            const int32_t *__restrict__ coords, const int32_t *__restrict__ nbr,
            uint8_t *__restrict__ masks, uint8_t *__restrict__ bflags, uint64_t *__restrict__ solid64) {
    const int lane = threadIdx.x & 31;
    const int64_t nr = rows_of(rs.n_rows, L);
    const int64_t nL = (int64_t)level_start[L + 1] - level_start[L];  // 0: the level was dropped
    for (int64_t r = (int64_t)blockIdx.x * kRowWarps + (threadIdx.x >> 5); r < nr;
         r += (int64_t)gridDim.x * kRowWarps) {
        const int2 row = rs.rows[r];
        if (row.y <= 0 || (int64_t)row.x + row.y > nL) continue;
        if (li.shard_count > 1) {  // multi-GPU: rows of other ranks
            const int4 c = reinterpret_cast<const int4 *>(coords)[rs.rid[row.x]];
            if (!owns_row(li, c.y, c.z)) continue;
        }
        xrow_pass_sorted<+1>(L, lane, rs.rid, row.x, row.y, coords, nbr, masks, L == 0, bflags, solid64);
        if (L > 0) {
            __syncwarp();
            xrow_pass_sorted<-1>(L, lane, rs.rid, row.x, row.y, coords, nbr, masks, true, bflags, solid64);
        }
    }
}

int propagate_rows_impl(const LevelInfo &li, vf_grid *g, int L, void *ws, cudaStream_t st) {
    RowWs w;
    rows_layout(g->capacity, (char *)ws, &w);
    k_xrows<<<max_ctas(8), kRowWarps * 32, 0, st>>>(li, L, w.set[L & 1], g->d_level_start, g->d_coords, g->d_nbr,
                                                    g->d_masks,
                                                    g->d_bflags, g->d_solid64);
    return check_launch("k_xrows");
}

}  // namespace vf
