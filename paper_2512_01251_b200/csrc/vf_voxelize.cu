// vf_voxelize.cu -- per-block ray-cast solid voxelizer and x-run propagation
// (SPEC.md:283-309).
//
//   K-vox    one warp per level-L block.  The block's bin faces (its matched
//            bin, pin A4) are staged 32 at a time in shared memory with their
//            SAT precomputation; lane = (row r = lane&15, face parity =
//            lane>>4) so the 16 x-rows x bin-faces slab tests run in parallel,
//            each hit row evaluates its 4 cell distances, and the two face
//            parities are merged with the (|d|, face order) tie rule (A7).
//            A row's 4 masks are one 32-bit word, written back with the A9
//            rule only when some cell of the block was hit (eta, Alg. 3).
//            Internal propagation is a provable no-op with matched bins (A8).
//   K-xfun   per block & row: transfer function of Alg. 5's carried status
//            (2 x 16-bit masks: output for input SOLID / OTHER).
//   K-xjump  pointer-jumping composition along same-level x-runs
//            (ceil(log2 B_L) rounds) -- the sequential chain walk of the paper
//             becomes an associative segmented scan (A10).
//   K-xapply status entering each block -> SOLID fill; fused finalize
//            (GUARD->FLUID, block solid flag).
#include <math.h>
#include <string.h>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_rowops.cuh"

namespace vf {

// --------------------------------------------------------------------------
// K-vox: Alg. 3 over block-indexed bins, flattened over (block, face) pairs.
//
// A CTA takes a group of 32 nonempty level-L blocks and spreads the group's
// (block, bin face) pairs over its threads, one pair per thread: every face
// record load is independent, so the dependent coords -> bin -> face-id ->
// record chain of a warp-per-block loop no longer serialises the level.
// Per pair: the x-rows of the block whose centre (y, z) lies within eps of the
// face's y / z extent (the SAT's exact box-axis comparisons), then the FP32
// row classifier (exact SAT in its undecided band); per hit row the 4 cell
// distances d = ((v1 - x) . n) / n_x (A7 association).  The chunk's (pair,
// hit row) items are bucketed by row (shared-memory counts, a warp prefix,
// cursors), and every row -- 4 cells -- is reduced by ONE owner thread: the
// A7 minimum per cell, |d| with ties to the lowest face id, as the
// lexicographic minimum of (|d| bits, face id) over the row's items and the
// best of the group's earlier chunks (IEEE bits of a non-negative double are
// ordered as the values); the winner records SOLID (n_x d > 0) or GUARD.
// Order-free, hence deterministic; no atomics on the cells (the round-based
// atomicMin protocol it replaces needed five barriers per 128 items).  Write-back per row word with the A9 rule,
// only for rows with a hit (eta == 0: no write, Alg. 3 l.648).  Internal
// propagation is a provable no-op with matched bins (A8).
#ifndef VF_VOX_T
#define VF_VOX_T 128
#endif
#ifndef VF_VOX_G
#define VF_VOX_G 16
#endif
constexpr int kVoxT = VF_VOX_T;  // threads per CTA
constexpr int kVoxG = VF_VOX_G;  // nonempty blocks per group (<= 32)

struct VoxGroup {
    unsigned long long bd[kVoxG * 64];  // best |d| per (block, cell); +inf = no hit
    int32_t bfid[kVoxG * 64];           // face id of the best
    uint8_t bval[kVoxG * 64];           // SOLID / GUARD of the best
    int32_t pre[kVoxG + 1];             // exclusive prefix of the blocks' pair counts
    int32_t base[kVoxG];                // first face_ids slot of each block
    int32_t bid[kVoxG];                 // block id (-1: past the list)
    int4 co[kVoxG];                     // block coordinates
    uint4 m[kVoxG][4];                  // the blocks' cell masks (loaded with the header)
    // one chunk of pairs: face v1 / n, id and block of each pair, the
    // (pair, hit row) items
    double pv[kVoxT][6];
    int32_t pfid[kVoxT];
    int16_t pw[kVoxT];
    uint16_t item[kVoxT * 16];      // the chunk's pair slots bucketed by row (block w, row r)
    int32_t rcnt[kVoxG * 16];       // items per row
    int32_t rcur[kVoxG * 16];       // scatter cursors
    int32_t roff[kVoxG * 16 + 1];   // exclusive prefix of rcnt
};

constexpr unsigned long long kInf64 = 0x7ff0000000000000ull;

#ifndef VF_VOX_MINB
#define VF_VOX_MINB 5
#endif
__global__ void __launch_bounds__(kVoxT, VF_VOX_MINB)
    k_voxelize(LevelInfo li, int L, const int32_t *__restrict__ level_start,
               const int32_t *__restrict__ coords, uint8_t *__restrict__ masks,
               const int32_t *__restrict__ ne, const int32_t *__restrict__ d_n_ne,
               const int32_t *__restrict__ base, int32_t *__restrict__ cnt, int zero_cnt,
               const int32_t *__restrict__ face_ids, const double *__restrict__ faces) {
    __shared__ VoxGroup S;
    const int t = threadIdx.x;
    const int n_ne = *d_n_ne;
    const int32_t s = level_start[L];
    const int n_groups = (n_ne + kVoxG - 1) / kVoxG;
    const double dx = li.dx, eps = li.eps, lx = li.len[0];
    uint32_t *masks32 = reinterpret_cast<uint32_t *>(masks);
    for (int gi = blockIdx.x; gi < n_groups; gi += gridDim.x) {
        if (t < 32) {  // group header: blocks, pair counts, prefix
            const int idx = gi * kVoxG + t;
            int u = -1, c = 0, bs = 0;
            if (t < kVoxG && idx < n_ne) {
                u = ne[idx];
                c = cnt[u];
                bs = base[u];
                S.co[t] = reinterpret_cast<const int4 *>(coords)[s + u];
                const uint4 *mp = reinterpret_cast<const uint4 *>(masks + 64 * (int64_t)(s + u));
#pragma unroll
                for (int q = 0; q < 4; ++q) S.m[t][q] = mp[q];
                if (zero_cnt) cnt[u] = 0;  // the next level's histogram starts from zero
            }
            int inc = c;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (t >= o) inc += y;
            }
            if (t < kVoxG) {
                S.pre[t + 1] = inc;
                S.base[t] = bs;
                S.bid[t] = u < 0 ? -1 : s + u;
            }
            if (t == 0) S.pre[0] = 0;
        }
        for (int i = t; i < kVoxG * 64; i += kVoxT) {
            S.bd[i] = kInf64;
            S.bfid[i] = 0x7fffffff;
        }
        __syncthreads();
        const int np = S.pre[kVoxG];
        for (int c0 = 0; c0 < np; c0 += kVoxT) {
            const int j = c0 + t;
            for (int i = t; i < kVoxG * 16; i += kVoxT) S.rcnt[i] = 0;
            uint32_t hm = 0;  // hit rows r = J + 4K of this thread's pair
            int w = 0, fid = 0;
            double v1[3] = {0.0, 0.0, 0.0}, nn[3] = {0.0, 0.0, 0.0};
            int4 co = make_int4(0, 0, 0, 0);
            if (j < np) {
#pragma unroll
                for (int st = kVoxG / 2; st > 0; st >>= 1)  // block of pair j: pre[w] <= j < pre[w + 1]
                    if (S.pre[w + st] <= j) w += st;
                fid = face_ids[S.base[w] + (j - S.pre[w])];
                co = S.co[w];
                double v[9];
                load_face(faces, fid, v, nn);
                v1[0] = v[0]; v1[1] = v[1]; v1[2] = v[2];
                if (!(fabs(nn[0]) < li.eps_par)) {  // A7: no x distance for faces parallel to x
                    const double ylo = fmin(fmin(v[1], v[4]), v[7]), yhi = fmax(fmax(v[1], v[4]), v[7]);
                    const double zlo = fmin(fmin(v[2], v[5]), v[8]), zhi = fmax(fmax(v[2], v[5]), v[8]);
                    uint32_t jm = 0, km = 0;
#pragma unroll
                    for (int q = 0; q < 4; ++q) {
                        const double y = node_c(4 * co.y + q, dx), z = node_c(4 * co.z + q, dx);
                        if (!(yhi < VF_DSUB(y, eps) || VF_DADD(y, eps) < ylo)) jm |= 1u << q;
                        if (!(zhi < VF_DSUB(z, eps) || VF_DADD(z, eps) < zlo)) km |= 1u << q;
                    }
                    if (jm && km) {
                        RowClass rc;
                        row_class_init(rc, v, nn, fmin(fmin(v[0], v[3]), v[6]), fmax(fmax(v[0], v[3]), v[6]),
                                       dx, eps, lx);
                        for (uint32_t kk = km; kk; kk &= kk - 1) {
                            const int K = __ffs(kk) - 1;
                            const double z = node_c(4 * co.z + K, dx);
                            for (uint32_t jj = jm; jj; jj &= jj - 1) {
                                const int J = __ffs(jj) - 1;
                                const double y = node_c(4 * co.y + J, dx);
                                const int cls = row_class(rc, (float)VF_DSUB(y, v[1]), (float)VF_DSUB(z, v[2]));
                                if (cls == 1 || (cls == 2 && row_sat_exact_f(faces, fid, y, z, eps, lx)))
                                    hm |= 1u << (J + 4 * K);
                            }
                        }
                    }
                }
            }
            // the chunk's (pair, hit row) items bucketed by row (block w, row
            // r); every row -- 4 cells -- is then reduced by ONE owner thread:
            // A7's minimum |d| per cell, ties to the lowest face id, as a
            // lexicographic (|d|, face id) minimum over the row's items and the
            // best of the earlier chunks -- order-free, no atomics on the cells
            S.pv[t][0] = v1[0]; S.pv[t][1] = v1[1]; S.pv[t][2] = v1[2];
            S.pv[t][3] = nn[0]; S.pv[t][4] = nn[1]; S.pv[t][5] = nn[2];
            S.pfid[t] = fid;
            S.pw[t] = (int16_t)w;
            __syncthreads();  // rcnt zeroed, pair records staged
            for (uint32_t m = hm; m; m &= m - 1) atomicAdd(&S.rcnt[w * 16 + (__ffs(m) - 1)], 1);
            __syncthreads();
            if (t < 32) {  // exclusive prefix over the rows (warp 0)
                constexpr int kPer = kVoxG * 16 / 32;
                int loc[kPer], sum = 0;
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    loc[k] = S.rcnt[t * kPer + k];
                    sum += loc[k];
                }
                int inc = sum;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if (t >= o) inc += y;
                }
                int ex = inc - sum;
#pragma unroll
                for (int k = 0; k < kPer; ++k) {
                    S.roff[t * kPer + k] = ex;
                    S.rcur[t * kPer + k] = ex;
                    ex += loc[k];
                }
                if (t == 31) S.roff[kVoxG * 16] = inc;
            }
            __syncthreads();
            for (uint32_t m = hm; m; m &= m - 1) S.item[atomicAdd(&S.rcur[w * 16 + (__ffs(m) - 1)], 1)] = (uint16_t)t;
            __syncthreads();
            for (int R = t; R < kVoxG * 16; R += kVoxT) {
                const int e0 = S.roff[R], e1 = S.roff[R + 1];
                if (e0 == e1) continue;
                const int iw = R >> 4, r = R & 15, slot0 = iw * 64 + 4 * r;
                const int4 ico = S.co[iw];
                const double y = node_c(4 * ico.y + (r & 3), dx), z = node_c(4 * ico.z + (r >> 2), dx);
                unsigned long long bd[4];
                int32_t bf[4];
                uint8_t bv[4];
#pragma unroll
                for (int I = 0; I < 4; ++I) {
                    bd[I] = S.bd[slot0 + I];
                    bf[I] = S.bfid[slot0 + I];
                    bv[I] = S.bval[slot0 + I];
                }
                for (int e = e0; e < e1; ++e) {
                    const int pl = S.item[e];
                    const double pv1[3] = {S.pv[pl][0], S.pv[pl][1], S.pv[pl][2]};
                    const double pn[3] = {S.pv[pl][3], S.pv[pl][4], S.pv[pl][5]};
                    const int32_t ifid = S.pfid[pl];
#pragma unroll
                    for (int I = 0; I < 4; ++I) {
                        const double d = VF_DDIV(plane_num(pv1, pn, node_c(4 * ico.x + I, dx), y, z), pn[0]);
                        const unsigned long long db = (unsigned long long)__double_as_longlong(fabs(d));
                        if (db < bd[I] || (db == bd[I] && ifid < bf[I])) {
                            bd[I] = db;
                            bf[I] = ifid;
                            bv[I] = VF_DMUL(pn[0], d) > 0.0 ? VF_SOLID : VF_GUARD;
                        }
                    }
                }
#pragma unroll
                for (int I = 0; I < 4; ++I) {
                    S.bd[slot0 + I] = bd[I];
                    S.bfid[slot0 + I] = bf[I];
                    S.bval[slot0 + I] = bv[I];
                }
            }
            __syncthreads();
        }
        __syncthreads();
        // write-back: one row word (4 cells) per thread, A9 rule
        for (int i = t; i < kVoxG * 16; i += kVoxT) {
            const int w = i >> 4, r = i & 15;
            const int32_t b = S.bid[w];
            if (b < 0) continue;
            uint32_t hit = 0, bh = 0;
#pragma unroll
            for (int I = 0; I < 4; ++I)
                if (S.bd[w * 64 + 4 * r + I] != kInf64) {
                    hit |= 1u << I;
                    bh |= (uint32_t)S.bval[w * 64 + 4 * r + I] << (8 * I);
                }
            if (!hit) continue;
            const uint32_t orig = reinterpret_cast<const uint32_t *>(&S.m[w][0])[r];
            uint32_t out = orig;
#pragma unroll
            for (int I = 0; I < 4; ++I) {
                if (!(hit >> I & 1)) continue;
                const uint32_t o = (orig >> (8 * I)) & 0xffu, hn = (bh >> (8 * I)) & 0xffu;
                if (hn == VF_SOLID || (o != VF_GHOST && o != VF_INTERFACE))
                    out = (out & ~(0xffu << (8 * I))) | (hn << (8 * I));
            }
            if (out != orig) masks32[(int64_t)b * 16 + r] = out;
        }
        __syncthreads();
    }
}

int voxelize_blocks_impl(const LevelInfo &li, vf_grid *g, int L, const BlockBins &bb,
                         const double *faces, bool zero_cnt, cudaStream_t st) {
    k_voxelize<<<max_ctas(VF_VOX_MINB), kVoxT, 0, st>>>(li, L, g->d_level_start, g->d_coords, g->d_masks,
                                                         bb.ne, bb.d_n_ne, bb.base, bb.cnt, zero_cnt ? 1 : 0,
                                                         bb.face_ids, faces);
    return check_launch("k_voxelize");
}

// dense BinLevel -> per-block (base, count) + nonempty list (SPEC op path)
__global__ void k_dense_to_blocks(int L, LevelInfo li, const int32_t *__restrict__ level_start,
                                  const int32_t *__restrict__ coords, const int32_t *__restrict__ counts,
                                  const int32_t *__restrict__ offsets, int32_t *__restrict__ cnt,
                                  int32_t *__restrict__ base, int32_t *__restrict__ ne,
                                  int32_t *__restrict__ d_n_ne) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int4 c = reinterpret_cast<const int4 *>(coords)[b];
        const int64_t bin = c.x + (int64_t)li.bins[0] * (c.y + (int64_t)li.bins[1] * c.z);
        const int32_t u = (int32_t)(b - s), n = counts[bin];
        cnt[u] = n;
        base[u] = offsets[bin];
        if (n > 0) ne[atomicAdd(d_n_ne, 1)] = u;
    }
}

int voxelize_impl(const LevelInfo &li, vf_grid *g, int L, const vf_bins *bins, const double *faces,
                  cudaStream_t st) {
    // stream-ordered scratch (the library keeps no pointer past the call)
    const size_t n = (size_t)g->capacity;
    char *tmp = nullptr;
    cudaError_t e = cudaMallocAsync((void **)&tmp, 3 * n * sizeof(int32_t) + 256, st);
    if (e != cudaSuccess) return set_cuda_error(e, "voxelize scratch");
    BlockBins bb;
    memset(&bb, 0, sizeof(bb));
    bb.cnt = (int32_t *)tmp;
    bb.base = bb.cnt + n;
    bb.ne = bb.base + n;
    bb.d_n_ne = bb.ne + n;
    bb.face_ids = bins->d_face_ids;
    cudaMemsetAsync(bb.d_n_ne, 0, sizeof(int32_t), st);
    k_dense_to_blocks<<<max_ctas(8), 256, 0, st>>>(L, li, g->d_level_start, g->d_coords, bins->d_counts,
                                                   bins->d_offsets, bb.cnt, bb.base, bb.ne, bb.d_n_ne);
    int rc = check_launch("k_dense_to_blocks");
    if (!rc) rc = voxelize_blocks_impl(li, g, L, bb, faces, false, st);
    e = cudaFreeAsync(tmp, st);
    if (!rc && e != cudaSuccess) rc = set_cuda_error(e, "voxelize scratch");
    return rc;
}

// --------------------------------------------------------------------------
// Alg. 5 as a scan.  Per block b and row r (16 rows), with H3 the row's
// trailing cell (I=3 for +x, I=0 for -x):
//   f_b(SOLID) = (H3 != GUARD),  f_b(OTHER) = (H3 == SOLID)      (1 = SOLID)
// packed as A | B << 16.  A run start (back slot < 0) carries the constant
// f_b(sigma) with sigma = SOLID iff its back code is SOLID_NBR.

__global__ void __launch_bounds__(256)
    k_xfun(int L, int back, int trail, const int32_t *__restrict__ level_start,
           const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
           uint32_t *__restrict__ G, int32_t *__restrict__ P) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[16];
        load_masks64(masks, b, w);
        uint32_t A, B;
        row_fn(w, trail, A, B);
        const int32_t code = nbr[27 * b + back];
        uint32_t fn = A | (B << 16);
        if (code < 0) {
            const uint32_t c = (code == VF_NB_SOLID_NBR) ? A : B;  // f_b(sigma)
            fn = c | (c << 16);
        }
        G[b] = fn;
        P[b] = code < 0 ? -1 : code;
    }
}

__global__ void __launch_bounds__(256)
    k_xjump(int L, const int32_t *__restrict__ level_start, const uint32_t *__restrict__ Gi,
            const int32_t *__restrict__ Pi, uint32_t *__restrict__ Go, int32_t *__restrict__ Po) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t p = Pi[b];
        uint32_t g = Gi[b];
        int32_t pn = -1;
        if (p >= 0) {
            g = compose(g, Gi[p]);
            pn = Pi[p];
        }
        Go[b] = g;
        Po[b] = pn;
    }
}

__global__ void __launch_bounds__(256)
    k_xapply(int L, int back, int finalize, const int32_t *__restrict__ level_start,
             const int32_t *__restrict__ nbr, uint8_t *__restrict__ masks,
             const uint32_t *__restrict__ G, uint8_t *__restrict__ bflags,
             uint64_t *__restrict__ solid64) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int32_t pred = nbr[27 * b + back];
        uint32_t w[16];
        load_masks64(masks, b, w);
        bool changed = false;
        if (pred >= 0) {
            const uint32_t st = G[pred] & 0xffffu;  // constant: status leaving pred
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const uint32_t x = row_apply(w[r], (st >> r) & 1u, L == 0);
                changed |= (x != w[r]);
                w[r] = x;
            }
        }
        if (finalize) finalize_block(w, changed, bflags, solid64, b);
        if (changed) store_masks64(masks, b, w);
    }
}

__global__ void __launch_bounds__(256)
    k_finalize(int L, const int32_t *__restrict__ level_start, uint8_t *__restrict__ masks,
               uint8_t *__restrict__ bflags, uint64_t *__restrict__ solid64) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        uint32_t w[16];
        load_masks64(masks, b, w);
        bool changed = false;
        finalize_block(w, changed, bflags, solid64, b);
        if (changed) store_masks64(masks, b, w);
    }
}

// multi-GPU exchange: zero what this rank does not own on level L
__global__ void k_shard_zero(LevelInfo li, int L, const int32_t *__restrict__ level_start,
                             const int32_t *__restrict__ coords, uint8_t *__restrict__ bflags,
                             uint64_t *__restrict__ solid64, int32_t *__restrict__ bcount) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int4 c = reinterpret_cast<const int4 *>(coords)[b];
        if (owns_row(li, c.y, c.z)) continue;
        bflags[b] = 0;
        solid64[b] = 0;
        if (bcount) bcount[b] = 0;
    }
}

int shard_zero_impl(const LevelInfo &li, vf_grid *g, int L, int32_t *bcount, cudaStream_t st) {
    k_shard_zero<<<max_ctas(8), 256, 0, st>>>(li, L, g->d_level_start, g->d_coords, g->d_bflags,
                                              g->d_solid64, bcount);
    return check_launch("k_shard_zero");
}

size_t propagate_workspace_size(int32_t capacity) {
    return 4 * ((size_t)capacity * sizeof(int32_t) + 256);
}

int propagate_impl(const LevelInfo &li, vf_grid *g, int L, int dir, int finalize, void *ws,
                   size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < propagate_workspace_size(g->capacity))
        return set_error(VF_EARG, "propagate workspace too small");
    const size_t stride = ((size_t)g->capacity * sizeof(int32_t) + 255) & ~(size_t)255;
    char *base = (char *)ws;
    uint32_t *G[2] = {(uint32_t *)base, (uint32_t *)(base + stride)};
    int32_t *P[2] = {(int32_t *)(base + 2 * stride), (int32_t *)(base + 3 * stride)};
    const int back = dir > 0 ? 2 : 1, trail = dir > 0 ? 3 : 0;
    const int grid = max_ctas(8);
    k_xfun<<<grid, 256, 0, st>>>(L, back, trail, g->d_level_start, g->d_nbr, g->d_masks, G[0], P[0]);
    int rc = check_launch("k_xfun");
    if (rc) return rc;
    int rounds = 0;
    while ((1 << rounds) < li.bins[0]) ++rounds;  // runs are at most B_L,x blocks long
    int cur = 0;
    for (int k = 0; k < rounds; ++k) {
        k_xjump<<<grid, 256, 0, st>>>(L, g->d_level_start, G[cur], P[cur], G[cur ^ 1], P[cur ^ 1]);
        if ((rc = check_launch("k_xjump"))) return rc;
        cur ^= 1;
    }
    k_xapply<<<grid, 256, 0, st>>>(L, back, finalize, g->d_level_start, g->d_nbr, g->d_masks,
                                   G[cur], g->d_bflags, g->d_solid64);
    return check_launch("k_xapply");
}

int finalize_impl(vf_grid *g, int L, cudaStream_t st) {
    k_finalize<<<max_ctas(8), 256, 0, st>>>(L, g->d_level_start, g->d_masks, g->d_bflags,
                                            g->d_solid64);
    return check_launch("k_finalize");
}

}  // namespace vf
