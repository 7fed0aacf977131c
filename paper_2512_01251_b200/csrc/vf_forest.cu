// vf_forest.cu -- forest-of-octrees kernels: root grid, near-wall marking and
// refine-only adaptation.
//
//   K-init    root blocks + full-halo links
//   K-mark*   (i) solid-boundary, (ii) adjacent + solid-adjacent, (iii) N_prop
//             ping-pong sweeps; block-parallel, 26-neighbour reads (pin A12)
//   K-adapt   child ids by exclusive scan over the level's marks (deterministic,
//             no hash table, no free-list atomics: the gap set is always
//             [n_used, capacity), pin A13), child metadata + links from the
//             parent's neighbours, ghost layer (A14); then the level's
//             neighbour-child links and interface layer.
#include <algorithm>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

__global__ void k_init_forest(int nx, int ny, int nz, int32_t *__restrict__ coords,
                              int32_t *__restrict__ nbr, int32_t *__restrict__ nbr_child,
                              int32_t *__restrict__ child, uint8_t *__restrict__ bflags,
                              uint8_t *__restrict__ masks, int32_t *__restrict__ level_start,
                              int32_t *__restrict__ status, uint64_t *__restrict__ solid64) {
    const int64_t n = (int64_t)nx * ny * nz;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int i = (int)(b % nx), j = (int)((b / nx) % ny), k = (int)(b / ((int64_t)nx * ny));
        reinterpret_cast<int4 *>(coords)[b] = make_int4(i, j, k, 0);
        for (int q = 0; q < 27; ++q) {
            const int ti = i + c27(q, 0), tj = j + c27(q, 1), tk = k + c27(q, 2);
            int32_t v = VF_NB_OUTSIDE;
            if (ti >= 0 && tj >= 0 && tk >= 0 && ti < nx && tj < ny && tk < nz)
                v = (int32_t)(ti + nx * (tj + ny * tk));
            nbr[27 * b + q] = v;
            nbr_child[27 * b + q] = -1;
        }
        child[b] = -1;
        bflags[b] = 0;
        solid64[b] = 0;
        uint4 *m = reinterpret_cast<uint4 *>(masks + 64 * b);
        m[0] = m[1] = m[2] = m[3] = make_uint4(0, 0, 0, 0);  // VF_FLUID
    }
    if (blockIdx.x == 0 && threadIdx.x <= VF_MAX_LEVELS) {
        level_start[threadIdx.x] = threadIdx.x == 0 ? 0 : (int32_t)n;
        if (threadIdx.x < 4) status[threadIdx.x] = 0;
    }
}

int init_forest_impl(const vf_config &cfg, vf_grid *g, cudaStream_t st) {
    const int64_t n = (int64_t)cfg.nb[0] * cfg.nb[1] * cfg.nb[2];
    if (n > g->capacity) return set_error(VF_ECAPACITY, "capacity below root block count");
    int grid = (int)((n + 255) / 256);
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_init_forest<<<grid, 256, 0, st>>>(cfg.nb[0], cfg.nb[1], cfg.nb[2], g->d_coords, g->d_nbr,
                                        g->d_nbr_child, g->d_child, g->d_bflags, g->d_masks,
                                        g->d_level_start, g->d_status, g->d_solid64);
    g->n_levels = 1;
    return check_launch("k_init_forest");
}

// --------------------------------------------------------------------------
// marking (pin A12).  aux bits: 1 eligible, 2 solid-boundary.

enum { AUX_ELIG = 1, AUX_SB = 2 };

__global__ void __launch_bounds__(256)
    k_mark_sb(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ nbr,
              const uint8_t *__restrict__ bflags, uint8_t *__restrict__ aux) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t *nb = nbr + 27 * b;
        bool el = true, fluid_nb = false;
        // fully unrolled: the 26 id loads, then the 26 flag gathers, in flight together
#pragma unroll
        for (int q = 1; q < 27; ++q) {
            const int32_t v = nb[q];
            if (v == VF_NB_MISSING || v == VF_NB_SOLID_NBR) el = false;
            if (v >= 0 && !(bflags[v] & VF_BF_SOLID)) fluid_nb = true;
        }
        const bool sb = (bflags[b] & VF_BF_SOLID) && fluid_nb;
        aux[b] = (uint8_t)((el ? AUX_ELIG : 0) | (sb ? AUX_SB : 0));
    }
}

__global__ void __launch_bounds__(256)
    k_mark_adj(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ nbr,
               uint8_t *__restrict__ bflags, const uint8_t *__restrict__ aux,
               uint8_t *__restrict__ m0, int commit) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t *nb = nbr + 27 * b;
        bool has_sb = false;
#pragma unroll
        for (int q = 1; q < 27; ++q) {
            const int32_t v = nb[q];
            if (v >= 0 && (aux[v] & AUX_SB)) has_sb = true;
        }
        const uint8_t a = aux[b];
        const uint8_t f0 = bflags[b];
        const bool solid = f0 & VF_BF_SOLID, sb = a & AUX_SB, el = a & AUX_ELIG;
        uint8_t f = (uint8_t)(f0 & ~(VF_BF_SB | VF_BF_SA | VF_BF_MARK));
        if (sb) f |= VF_BF_SB;
        if (has_sb && !solid) f |= VF_BF_SA;
        const uint8_t mk = (uint8_t)(el && (sb || has_sb));
        if (commit && mk) f |= VF_BF_MARK;  // N_prop = 0: this is the last phase
        bflags[b] = f;
        m0[b] = mk;
    }
}

__global__ void __launch_bounds__(256)
    k_mark_prop(int L, int it, const int32_t *__restrict__ level_start,
                const int32_t *__restrict__ nbr, uint8_t *__restrict__ bflags,
                const uint8_t *__restrict__ aux, const uint8_t *__restrict__ src,
                uint8_t *__restrict__ dst, int commit) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint8_t m = src[b];
        if (!m && (aux[b] & AUX_ELIG) && (!(bflags[b] & VF_BF_SOLID) || it == 0)) {
            const int32_t *nb = nbr + 27 * b;
            bool any = false;
#pragma unroll
            for (int q = 1; q < 27; ++q) {
                const int32_t v = nb[q];
                any |= v >= 0 && src[v];
            }
            m = any ? 1 : 0;
        }
        dst[b] = m;
        // last sweep: commit (only this thread touches bflags[b]; neighbours
        // are read through src, never through bflags' MARK bit)
        if (commit && m) bflags[b] |= VF_BF_MARK;
    }
}

size_t mark_workspace_size(int32_t capacity) { return 3 * (((size_t)capacity + 255) & ~(size_t)255); }

int mark_impl(const vf_config &cfg, vf_grid *g, int L, void *ws, size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < mark_workspace_size(g->capacity)) return set_error(VF_EARG, "mark workspace too small");
    const size_t stride = ((size_t)g->capacity + 255) & ~(size_t)255;
    uint8_t *aux = (uint8_t *)ws, *m[2] = {aux + stride, aux + 2 * stride};
    const int grid = max_ctas(8);
    k_mark_sb<<<grid, 256, 0, st>>>(L, g->d_level_start, g->d_nbr, g->d_bflags, aux);
    int rc = check_launch("k_mark_sb");
    if (rc) return rc;
    // the last phase also commits the MARK bits (no separate commit pass)
    k_mark_adj<<<grid, 256, 0, st>>>(L, g->d_level_start, g->d_nbr, g->d_bflags, aux, m[0],
                                     cfg.n_prop == 0);
    if ((rc = check_launch("k_mark_adj"))) return rc;
    int cur = 0;
    for (int it = 0; it < cfg.n_prop; ++it) {
        k_mark_prop<<<grid, 256, 0, st>>>(L, it, g->d_level_start, g->d_nbr, g->d_bflags, aux,
                                          m[cur], m[cur ^ 1], it == cfg.n_prop - 1);
        if ((rc = check_launch("k_mark_prop"))) return rc;
        cur ^= 1;
    }
    return VF_OK;
}

// --------------------------------------------------------------------------
// adapt (pins A13, A14)

struct LoadMark {
    const int32_t *level_start;
    int L;
    const uint8_t *bflags;
    __device__ int operator()(int64_t i) const {
        return (bflags[level_start[L] + i] & VF_BF_MARK) ? 1 : 0;
    }
};
struct EmitChild {
    const int32_t *level_start;
    int L;
    int32_t *child;
    uint8_t *bflags;
    int32_t *parents;
    __device__ void operator()(int64_t i, int v, int ex) const {
        const int32_t s = level_start[L], e = level_start[L + 1];
        const int64_t b = s + i;
        const uint8_t f = bflags[b];
        if (v) {
            child[b] = e + 8 * ex;
            parents[ex] = (int32_t)b;
            bflags[b] = (uint8_t)(f | VF_BF_REFINED);
        } else {
            child[b] = -1;
            bflags[b] = (uint8_t)(f & ~VF_BF_REFINED);
        }
    }
};

// appends level L+1 once the number of marked blocks is known (runs as the
// adapt scan's epilogue on the thread that publishes the total)
struct AdaptFinish {
    int L;
    int32_t capacity;
    int32_t *level_start;
    int32_t *status;
    __device__ void operator()(int n_marked) const {
        const int64_t e = level_start[L + 1];
        int64_t ne = e + 8 * (int64_t)n_marked;
        if (ne > capacity) {
            atomicMax(status, VF_ECAPACITY);
            status[1] = L;  // level context
            ne = e;         // drop the level: later stages see no blocks, no OOB ids
        }
        for (int k = L + 2; k <= VF_MAX_LEVELS; ++k) level_start[k] = (int32_t)ne;
    }
};

// bit index of a direction in {-1,0,1}^3: (dx+1) + 3(dy+1) + 9(dz+1)
__device__ __forceinline__ int dir_code(int dx, int dy, int dz) {
    return (dx + 1) + 3 * (dy + 1) + 9 * (dz + 1);
}
__device__ __forceinline__ int dir_code_of_slot(int q) {
    return dir_code(c27(q, 0), c27(q, 1), c27(q, 2));
}
// any direction (ox,oy,oz) != 0 with o_d in {0, e_d} set in `bits`
__device__ __forceinline__ bool touches(uint32_t bits, int ex, int ey, int ez) {
    bool any = false;
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
        for (int b2 = 0; b2 < 2; ++b2)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int ox = a ? ex : 0, oy = b2 ? ey : 0, oz = c ? ez : 0;
                if (ox == 0 && oy == 0 && oz == 0) continue;
                any |= (bits >> dir_code(ox, oy, oz)) & 1u;
            }
    return any;
}
// 8 octant bits: octant o = (x>=2) | (y>=2)<<1 | (z>=2)<<2 touches a set direction
__device__ __forceinline__ uint32_t octant_bits(uint32_t bits, int) {
    uint32_t g = 0;
#pragma unroll
    for (int o = 0; o < 8; ++o)
        g |= (uint32_t)touches(bits, (o & 1) ? 1 : -1, (o & 2) ? 1 : -1, (o & 4) ? 1 : -1) << o;
    return g;
}

// Thread per child (256 children = 32 parents per CTA batch): the 27 slots
// are unrolled, so every D3Q27 component is a compile-time constant and the
// parent-side slot of a target reduces to two adds and a shift per axis;
// the child's nbr row is built in shared memory (row stride 27 words: no
// bank conflicts) and copied out coalesced, nbr_child rows are -1 stores.
// Children of the level's marked parents (A13, A14): coords, 27 neighbour
// slots (child of the parent-side neighbour, or MISSING / SOLID_NBR /
// OUTSIDE), nbr_child = -1, flags, and the ghost-layer cell masks.
constexpr int kAdaptTBatch = 256;

#ifndef VF_ADAPT_MINB
#define VF_ADAPT_MINB 3  // 67 registers, no spills (measured: C2 -2%, C4 -1%)
#endif
__global__ void __launch_bounds__(kAdaptTBatch, VF_ADAPT_MINB)
    k_adapt_children_t(int L, int32_t capacity, int nbx1, int nby1, int nbz1,
                       const int32_t *__restrict__ level_start, const int32_t *__restrict__ n_marked,
                       const int32_t *__restrict__ parents, int32_t *__restrict__ coords,
                       int32_t *__restrict__ nbr, int32_t *__restrict__ nbr_child,
                       int32_t *__restrict__ child, uint8_t *__restrict__ bflags,
                       uint8_t *__restrict__ masks, int32_t *__restrict__ status,
                       uint64_t *__restrict__ solid64) {
    __shared__ int32_t s_row[kAdaptTBatch * 27];
    __shared__ int4 s_pc[kAdaptTBatch / 8];
    // per parent and parent-side slot: the neighbour's first child (>= 0: the
    // child's neighbour is that child + sub-octant) or the code the child
    // inherits (OUTSIDE / SOLID_NBR / MISSING)
    __shared__ int32_t s_code[kAdaptTBatch / 8][27];
    __shared__ uint8_t s_slot[27];  // slot of (dx, dy, dz), index (dx+1) + 3 (dy+1) + 9 (dz+1)
    const int64_t e = level_start[L + 1];
    const int64_t nc = 8 * (int64_t)(*n_marked);
    const int t = threadIdx.x;
    if (t < 27) s_slot[t] = (uint8_t)slot_of(t % 3 - 1, (t / 3) % 3 - 1, t / 9 - 1);
    for (int64_t c0 = (int64_t)blockIdx.x * kAdaptTBatch; c0 < nc; c0 += (int64_t)gridDim.x * kAdaptTBatch) {
        const int nb = (int)min((int64_t)kAdaptTBatch, nc - c0);
        const int np = (nb + 7) >> 3;
        if (t < np) s_pc[t] = reinterpret_cast<const int4 *>(coords)[parents[(c0 >> 3) + t]];
        for (int it = t; it < np * 27; it += blockDim.x) {
            const int p = it / 27, q = it - 27 * p;
            const int32_t P = parents[(c0 >> 3) + p];
            const int32_t Pn = (q == 0) ? P : nbr[27 * (int64_t)P + q];
            int32_t code = VF_NB_OUTSIDE;
            if (Pn >= 0) {
                const int32_t ch = child[Pn];
                code = ch >= 0 ? ch : ((bflags[Pn] & VF_BF_SOLID) ? VF_NB_SOLID_NBR : VF_NB_MISSING);
            } else if (Pn != VF_NB_OUTSIDE) {  // marked parents are eligible: cannot happen
                atomicMax(status, VF_EARG);
                code = VF_NB_MISSING;
            }
            s_code[p][q] = code;
        }
        __syncthreads();
        const int64_t id = e + c0 + t;
        if (t < nb && id < capacity) {
            const int p = t >> 3, cc = t & 7;
            const int4 pc = s_pc[p];
            const int ox = cc & 1, oy = (cc >> 1) & 1, oz = cc >> 2;
            const int ci = 2 * pc.x + ox, cj = 2 * pc.y + oy, ck = 2 * pc.z + oz;
            uint32_t missing = 0;
#pragma unroll
            for (int q = 0; q < 27; ++q) {
                const int cx = c27(q, 0), cy = c27(q, 1), cz = c27(q, 2);
                // parent-side direction (o + c) >> 1 per axis (floor); the
                // child's target is outside the domain iff that parent-side
                // neighbour is (its code is then OUTSIDE)
                const int px = cx < 0 ? ox - 1 : (cx > 0 ? ox : 0);
                const int py = cy < 0 ? oy - 1 : (cy > 0 ? oy : 0);
                const int pz = cz < 0 ? oz - 1 : (cz > 0 ? oz : 0);
                const int32_t code = s_code[p][s_slot[(px + 1) + 3 * (py + 1) + 9 * (pz + 1)]];
                const int sub = ((ox + cx) & 1) + 2 * ((oy + cy) & 1) + 4 * ((oz + cz) & 1);
                const int32_t v = code >= 0 ? code + sub : code;
                s_row[27 * t + q] = v;
                if (v == VF_NB_MISSING || v == VF_NB_SOLID_NBR) missing |= 1u << dir_code(cx, cy, cz);
            }
            reinterpret_cast<int4 *>(coords)[id] = make_int4(ci, cj, ck, L + 1);
            child[id] = -1;
            bflags[id] = 0;
            solid64[id] = 0;
            // A14 ghost layer: a cell is within Chebyshev distance 2 (fine
            // cells) of a missing neighbour block iff one of the 7 blocks
            // towards its octant is missing, so 8 octant bits decide all 64 cells
            const uint32_t g8 = octant_bits(missing, 2);
            uint4 *mp = reinterpret_cast<uint4 *>(masks + 64 * id);
#pragma unroll
            for (int part = 0; part < 4; ++part) {
                uint32_t w[4];
#pragma unroll
                for (int rr = 0; rr < 4; ++rr) {
                    const int r = 4 * part + rr;
                    const int J = r & 3, K = r >> 2;
                    uint32_t x = 0;
#pragma unroll
                    for (int I = 0; I < 4; ++I) {
                        const int o = (I >= 2) | ((J >= 2) << 1) | ((K >= 2) << 2);
                        x |= (uint32_t)((g8 >> o & 1u) ? VF_GHOST : VF_FLUID) << (8 * I);
                    }
                    w[rr] = x;
                }
                mp[part] = make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        __syncthreads();
        // coalesced copy-out of the batch's nbr rows; nbr_child rows = -1
        const int64_t nw = (int64_t)min((int64_t)nb, (int64_t)capacity - (e + c0));
        const int64_t base = 27 * (e + c0);
        for (int64_t i = t; i < 27 * nw; i += blockDim.x) {
            nbr[base + i] = s_row[i];
            nbr_child[base + i] = -1;
        }
        __syncthreads();
    }
}

// level-L neighbour-child links + interface layer of refined blocks (A14).
// (block, slot) pairs spread over a CTA (coalesced nbr_child rows), the
// per-block "existing unrefined neighbour" bits OR-ed in shared memory, then
// the interface cells of refined blocks, one 32-bit mask row per thread.
constexpr int kLevelBatch = 64;

__global__ void __launch_bounds__(256)
    k_adapt_level(int L, const int32_t *__restrict__ level_start, const int32_t *__restrict__ nbr,
                  int32_t *__restrict__ nbr_child, const int32_t *__restrict__ child,
                  uint8_t *__restrict__ masks) {
    __shared__ uint32_t s_coarse[kLevelBatch];
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b0 = s + (int64_t)blockIdx.x * kLevelBatch; b0 < e; b0 += (int64_t)gridDim.x * kLevelBatch) {
        const int nb = (int)min((int64_t)kLevelBatch, (int64_t)e - b0);
        if (threadIdx.x < kLevelBatch) s_coarse[threadIdx.x] = 0;
        __syncthreads();
        for (int it = threadIdx.x; it < nb * 27; it += blockDim.x) {
            const int lb = it / 27, q = it - 27 * lb;
            const int64_t b = b0 + lb;
            const int32_t v = (q == 0) ? (int32_t)b : nbr[27 * b + q];
            const int32_t ch = (v >= 0) ? child[v] : -1;
            nbr_child[27 * b + q] = ch;
            if (q > 0 && v >= 0 && ch < 0) atomicOr(&s_coarse[lb], 1u << dir_code_of_slot(q));
        }
        __syncthreads();
        for (int it = threadIdx.x; it < nb * 16; it += blockDim.x) {
            const int lb = it >> 4, r = it & 15;
            const int64_t b = b0 + lb;
            const uint32_t coarse = s_coarse[lb];
            if (!coarse || child[b] < 0) continue;
            uint32_t *m = reinterpret_cast<uint32_t *>(masks + 64 * b);
            const int J = r & 3, K = r >> 2;
            uint32_t x = m[r];
            const uint32_t x0 = x;
#pragma unroll
            for (int I = 0; I < 4; ++I) {
                if (((x >> (8 * I)) & 0xffu) != VF_FLUID) continue;
                // one coarse cell: only the faces / edges / corner the cell touches
                const int ex = I == 0 ? -1 : (I == 3 ? 1 : 0);
                const int ey = J == 0 ? -1 : (J == 3 ? 1 : 0);
                const int ez = K == 0 ? -1 : (K == 3 ? 1 : 0);
                if (touches(coarse, ex, ey, ez)) x = (x & ~(0xffu << (8 * I))) | ((uint32_t)VF_INTERFACE << (8 * I));
            }
            if (x != x0) m[r] = x;
        }
        __syncthreads();
    }
}

static size_t al256(size_t x) { return (x + 255) & ~(size_t)255; }

size_t adapt_workspace_size(int32_t capacity) {
    return al256(sizeof(int32_t) * ((size_t)capacity + 1)) + al256(sizeof(int32_t) * 8) +
           al256(scan_workspace_bytes(capacity));
}

int adapt_impl(const vf_config &cfg, vf_grid *g, int L, void *ws, size_t ws_bytes, cudaStream_t st,
               bool links) {
    if (ws_bytes < adapt_workspace_size(g->capacity)) return set_error(VF_EARG, "adapt workspace too small");
    if (L != g->n_levels - 1 || L + 1 >= VF_MAX_LEVELS) return set_error(VF_EARG, "adapt: level must be the finest");
    char *base = (char *)ws;
    int32_t *parents = (int32_t *)base;
    int32_t *scalars = (int32_t *)(base + al256(sizeof(int32_t) * ((size_t)g->capacity + 1)));
    void *scan_ws = base + al256(sizeof(int32_t) * ((size_t)g->capacity + 1)) + al256(sizeof(int32_t) * 8);
    // child ids = exclusive scan of the level's marks; the publishing thread
    // also appends the new level (AdaptFinish: level_start[L+2..], capacity)
    cudaError_t ce = scan_launch_fn(LoadMark{g->d_level_start, L, g->d_bflags},
                                    EmitChild{g->d_level_start, L, g->d_child, g->d_bflags, parents},
                                    std::min((int64_t)g->capacity, (int64_t)(cfg.nb[0] << L) * (cfg.nb[1] << L) *
                                                                         (int64_t)(cfg.nb[2] << L)),
                                    ScanLevelN{g->d_level_start, L}, scalars + 1, scan_ws,
                                    st, AdaptFinish{L, g->capacity, g->d_level_start, g->d_status});
    if (ce != cudaSuccess) return set_cuda_error(ce, "adapt scan");
    int rc;
    k_adapt_children_t<<<wave_ctas(k_adapt_children_t, kAdaptTBatch), kAdaptTBatch, 0, st>>>(
        L, g->capacity, cfg.nb[0] << (L + 1), cfg.nb[1] << (L + 1), cfg.nb[2] << (L + 1),
        g->d_level_start, scalars + 1, parents, g->d_coords, g->d_nbr, g->d_nbr_child, g->d_child,
        g->d_bflags, g->d_masks, g->d_status, g->d_solid64);
    if ((rc = check_launch("k_adapt_children"))) return rc;
    g->n_levels = L + 2;
    return links ? adapt_links_impl(g, L, st) : VF_OK;
}

// level L's neighbour-child links and interface layer (after its children
// exist): outputs only -- no later stage of the embed reads them -- so the
// embed runs them on a side stream
int adapt_links_impl(vf_grid *g, int L, cudaStream_t st) {
    k_adapt_level<<<max_ctas(8), 256, 0, st>>>(L, g->d_level_start, g->d_nbr, g->d_nbr_child,
                                               g->d_child, g->d_masks);
    return check_launch("k_adapt_level");
}

}  // namespace vf
