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
// hit row) items are compacted, and the A7 minimum per cell -- |d|, ties to
// the lowest face id -- is reduced in shared memory in rounds of one item
// (4 cells) per thread:
//   (1) every candidate notes the cell's best |d| before the round,
//   (2) 64-bit atomicMin of |d| (IEEE bits of a non-negative double are
//       ordered as the values),
//   (3) a cell whose best |d| dropped forgets the previous winner's id,
//   (4) atomicMin of the face id among the candidates at the best |d|,
//   (5) the winner records SOLID (n_x d > 0) or GUARD.
// Order-free, hence deterministic.  Write-back per row word with the A9 rule,
// only for rows with a hit (eta == 0: no write, Alg. 3 l.648).  Internal
// propagation is a provable no-op with matched bins (A8).
constexpr int kVoxT = 128;  // threads per CTA
constexpr int kVoxG = 32;   // nonempty blocks per group

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
    uint16_t item[kVoxT * 16];
    int wsum[kVoxT / 32];
    int n_item;
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
            if (idx < n_ne) {
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
            S.pre[t + 1] = inc;
            if (t == 0) S.pre[0] = 0;
            S.base[t] = bs;
            S.bid[t] = u < 0 ? -1 : s + u;
        }
        for (int i = t; i < kVoxG * 64; i += kVoxT) {
            S.bd[i] = kInf64;
            S.bfid[i] = 0x7fffffff;
        }
        __syncthreads();
        const int np = S.pre[kVoxG];
        for (int c0 = 0; c0 < np; c0 += kVoxT) {
            const int j = c0 + t;
            uint32_t hm = 0;  // hit rows r = J + 4K of this thread's pair
            int w = 0, fid = 0;
            double v1[3] = {0.0, 0.0, 0.0}, nn[3] = {0.0, 0.0, 0.0};
            int4 co = make_int4(0, 0, 0, 0);
            if (j < np) {
#pragma unroll
                for (int st = 16; st > 0; st >>= 1)  // block of pair j: pre[w] <= j < pre[w + 1]
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
            // the chunk's (pair, hit row) items, compacted in pair order
            {
                const int c = __popc(hm);
                int inc = c;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, inc, o);
                    if ((t & 31) >= o) inc += y;
                }
                if ((t & 31) == 31) S.wsum[t >> 5] = inc;
                S.pv[t][0] = v1[0]; S.pv[t][1] = v1[1]; S.pv[t][2] = v1[2];
                S.pv[t][3] = nn[0]; S.pv[t][4] = nn[1]; S.pv[t][5] = nn[2];
                S.pfid[t] = fid;
                S.pw[t] = (int16_t)w;
                __syncthreads();
                int pos = inc - c;
                for (int k = 0; k < (t >> 5); ++k) pos += S.wsum[k];
                for (uint32_t m = hm; m; m &= m - 1) S.item[pos++] = (uint16_t)(t | ((__ffs(m) - 1) << 8));
                if (t == kVoxT - 1) S.n_item = pos;
                __syncthreads();
            }
            // rounds of one item per thread (the A7 reduction, see above)
            const int n_item = S.n_item;
            for (int i0 = 0; i0 < n_item; i0 += kVoxT) {
                const bool has = i0 + t < n_item;
                int slot0 = 0, ifid = 0;
                unsigned long long db[4] = {kInf64, kInf64, kInf64, kInf64}, old[4];
                bool solid[4] = {false, false, false, false};
                if (has) {
                    const uint32_t it = S.item[i0 + t];
                    const int pl = it & 0xff, r = it >> 8, iw = S.pw[pl];
                    const int4 ico = S.co[iw];
                    const double pv1[3] = {S.pv[pl][0], S.pv[pl][1], S.pv[pl][2]};
                    const double pn[3] = {S.pv[pl][3], S.pv[pl][4], S.pv[pl][5]};
                    ifid = S.pfid[pl];
                    const double y = node_c(4 * ico.y + (r & 3), dx), z = node_c(4 * ico.z + (r >> 2), dx);
                    slot0 = iw * 64 + 4 * r;
#pragma unroll
                    for (int I = 0; I < 4; ++I) {
                        const double d = VF_DDIV(plane_num(pv1, pn, node_c(4 * ico.x + I, dx), y, z), pn[0]);
                        db[I] = (unsigned long long)__double_as_longlong(fabs(d));
                        solid[I] = VF_DMUL(pn[0], d) > 0.0;
                        old[I] = S.bd[slot0 + I];
                    }
                }
                __syncthreads();
                if (has)
#pragma unroll
                    for (int I = 0; I < 4; ++I) atomicMin(&S.bd[slot0 + I], db[I]);
                __syncthreads();
                bool best[4] = {false, false, false, false};
                if (has)
#pragma unroll
                    for (int I = 0; I < 4; ++I) {
                        const unsigned long long b = S.bd[slot0 + I];
                        best[I] = b == db[I];
                        if (best[I] && b < old[I]) S.bfid[slot0 + I] = 0x7fffffff;  // new best |d|
                    }
                __syncthreads();
#pragma unroll
                for (int I = 0; I < 4; ++I)
                    if (best[I]) atomicMin(&S.bfid[slot0 + I], ifid);
                __syncthreads();
#pragma unroll
                for (int I = 0; I < 4; ++I)
                    if (best[I] && S.bfid[slot0 + I] == ifid) S.bval[slot0 + I] = solid[I] ? VF_SOLID : VF_GUARD;
                __syncthreads();
            }
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

__device__ __forceinline__ uint32_t compose(uint32_t g, uint32_t f) {
    // (g o f)(x) = g(f(x)); per row: f(x)=1 -> g(S) else g(O)
    const uint32_t gA = g & 0xffffu, gB = g >> 16, fA = f & 0xffffu, fB = f >> 16;
    const uint32_t A = (fA & gA) | (~fA & gB & 0xffffu);
    const uint32_t B = (fB & gA) | (~fB & gB & 0xffffu);
    return A | (B << 16);
}

// byte-SIMD on a row word (the 4 cells of an x-row, one mask byte each)
__device__ __forceinline__ uint32_t bytes_eq(uint32_t x, uint32_t v) { return __vcmpeq4(x, v * 0x01010101u); }
// 0xff / 0x00 bytes -> 4 bits (byte i -> bit i)
__device__ __forceinline__ uint32_t nib4(uint32_t m) { return ((m & 0x01010101u) * 0x01020408u) >> 24; }

// Alg. 5 transfer function of a block from its rows' trailing cells (A10):
// bit r of A = (H_trail != GUARD), of B = (H_trail == SOLID)
__device__ __forceinline__ void row_fn(const uint32_t w[16], int trail, uint32_t &A, uint32_t &B) {
    A = B = 0;
    const uint32_t sel = (uint32_t)trail | ((4u + (uint32_t)trail) << 4);
#pragma unroll
    for (int r = 0; r < 16; r += 4) {
        const uint32_t t4 = __byte_perm(__byte_perm(w[r], w[r + 1], sel), __byte_perm(w[r + 2], w[r + 3], sel),
                                        0x5410);  // trailing bytes of rows r..r+3
        A |= nib4(~bytes_eq(t4, VF_GUARD)) << r;
        B |= nib4(bytes_eq(t4, VF_SOLID)) << r;
    }
}

// Alg. 5 update of one row word: carried SOLID turns every non-GUARD cell
// SOLID; on level 0 GUARD -> FLUID afterwards
__device__ __forceinline__ uint32_t row_apply(uint32_t xw, bool solid, bool l0) {
    const uint32_t g = bytes_eq(xw, VF_GUARD);
    if (solid) xw = (xw & g) | ((0x01010101u * VF_SOLID) & ~g);
    if (l0) xw &= ~g;  // GUARD bytes are unchanged by the update; FLUID = 0
    return xw;
}

__device__ __forceinline__ void load_masks64(const uint8_t *masks, int64_t b, uint32_t w[16]) {
    const uint4 *p = reinterpret_cast<const uint4 *>(masks + 64 * b);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        const uint4 u = p[k];
        w[4 * k] = u.x; w[4 * k + 1] = u.y; w[4 * k + 2] = u.z; w[4 * k + 3] = u.w;
    }
}

__device__ __forceinline__ void store_masks64(uint8_t *masks, int64_t b, const uint32_t w[16]) {
    uint4 *p = reinterpret_cast<uint4 *>(masks + 64 * b);
#pragma unroll
    for (int k = 0; k < 4; ++k) p[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
}

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

// finalize (pin A11): GUARD -> FLUID, block solid flag, and the
// block's 64-bit SOLID-cell mask (bit t = cell t) used by the boundary halo
// and exchanged between ranks at the finest level
__device__ __forceinline__ void finalize_block(uint32_t w[16], bool &changed, uint8_t *bflags,
                                               uint64_t *solid64, int64_t b) {
    uint64_t sm = 0;
#pragma unroll
    for (int r = 0; r < 16; ++r) {
        const uint32_t x = w[r] & ~bytes_eq(w[r], VF_GUARD);  // GUARD -> FLUID (0)
        sm |= (uint64_t)nib4(bytes_eq(w[r], VF_SOLID)) << (4 * r);
        changed |= (x != w[r]);
        w[r] = x;
    }
    const uint8_t f0 = bflags[b];
    bflags[b] = (uint8_t)((f0 & ~VF_BF_SOLID) | (sm ? VF_BF_SOLID : 0));
    solid64[b] = sm;
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

// --------------------------------------------------------------------------
// K-xrows: Alg. 5 in both directions + finalize as ONE kernel per level.
//
// A dense map of the level's blocks (B_L^3 ids, -1 = no level-L block) turns
// every x-row of blocks into a contiguous array, so one warp owns one row
// (j, k) and reads its positions 32 at a time (coalesced) instead of walking
// the neighbour chain (the paper's sequential walk) or pointer-jumping over
// it (k_xfun/k_xjump/k_xapply: 2 + ceil(log2 B_L) launches per direction).
// Per chunk: transfer functions of the 32 blocks, a warp segmented scan with
// compose() (segments start at run starts, which carry f_b(sigma), and at
// lane 0, which folds in the status leaving the previous chunk), the status
// entering each block = the scan value of its predecessor, then the fill /
// finalize of that block.  The -x pass re-reads the +x results of the same
// row (same warp, ordered by __syncwarp).  Identical results to the
// pointer-jumping operators (same f_b, same composition, same apply).

__global__ void k_level_map(int L, LevelInfo li, const int32_t *__restrict__ level_start,
                            const int32_t *__restrict__ coords, int32_t *__restrict__ map) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int4 c = reinterpret_cast<const int4 *>(coords)[b];
        map[c.x + (int64_t)li.bins[0] * (c.y + (int64_t)li.bins[1] * c.z)] = (int32_t)b;
    }
}

// one direction over one row; returns nothing, masks updated in place
template <int DIR>
__device__ __forceinline__ void xrow_pass(int L, int lane, const int32_t *__restrict__ row, int bx,
                                          const int32_t *__restrict__ nbr, uint8_t *__restrict__ masks,
                                          bool finalize, uint8_t *__restrict__ bflags,
                                          uint64_t *__restrict__ solid64) {
    constexpr int back = DIR > 0 ? 2 : 1, trail = DIR > 0 ? 3 : 0;
    uint32_t carry = 0;        // status leaving the last block of the previous chunk
    bool prev_present = false;  // ... and whether that position holds a level-L block
    for (int x0 = 0; x0 < bx; x0 += 32) {
        const int x = DIR > 0 ? x0 + lane : bx - 1 - (x0 + lane);
        const int32_t id = (x0 + lane < bx) ? row[x] : -1;
        const bool present = id >= 0;
        const uint32_t pm = __ballot_sync(0xffffffffu, present);
        if (pm == 0) {
            prev_present = false;
            continue;
        }
        const bool pred = lane > 0 ? ((pm >> (lane - 1)) & 1u) : prev_present;
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
        // segmented inclusive scan (compose) across the warp
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t g = __shfl_up_sync(0xffffffffu, fn, o);
            const int hd = __shfl_up_sync(0xffffffffu, (int)head, o);
            if (lane >= o && !head) {
                fn = compose(fn, g);
                head = hd;
            }
        }
        const uint32_t out = fn & 0xffffu;  // constant: status leaving this block
        uint32_t st = __shfl_up_sync(0xffffffffu, out, 1);
        if (lane == 0) st = carry;
        if (present) {
            bool changed = false;
            if (pred) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t xw = row_apply(w[r], (st >> r) & 1u, L == 0);
                    changed |= (xw != w[r]);
                    w[r] = xw;
                }
            }
            if (finalize) finalize_block(w, changed, bflags, solid64, id);
            if (changed) store_masks64(masks, id, w);
        }
        carry = __shfl_sync(0xffffffffu, out, 31);
        prev_present = (pm >> 31) & 1u;
    }
}

constexpr int kXrowWarps = 8;

__global__ void __launch_bounds__(kXrowWarps * 32)
    k_xrows(LevelInfo li, int L, const int32_t *__restrict__ map, const int32_t *__restrict__ nbr,
            uint8_t *__restrict__ masks, uint8_t *__restrict__ bflags,
            uint64_t *__restrict__ solid64) {
    const int lane = threadIdx.x & 31;
    const int64_t gw = (int64_t)blockIdx.x * kXrowWarps + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * kXrowWarps;
    const int bx = li.bins[0], by = li.bins[1];
    const int64_t rows = (int64_t)by * li.bins[2];
    for (int64_t r = gw; r < rows; r += nw) {
        const int j = (int)(r % by), k = (int)(r / by);
        if (!owns_row(li, j, k)) continue;  // multi-GPU: rows of other ranks
        const int32_t *row = map + r * bx;
        xrow_pass<+1>(L, lane, row, bx, nbr, masks, L == 0, bflags, solid64);
        if (L > 0) {
            __syncwarp();
            xrow_pass<-1>(L, lane, row, bx, nbr, masks, true, bflags, solid64);
        }
    }
}

// Staged variant for rows of up to 32 * NCH blocks (levels with B_L <= 128): the row's block ids, masks (row stride 17 words: no bank
// conflicts), run-start neighbour codes of both directions and changed
// flags are staged in shared memory with all global loads issued up front,
// then both passes run out of shared memory and only changed blocks are
// stored -- the chunked passes above wait on a dependent load chain per
// chunk and per direction.
constexpr int kXsWarps = 4;
static int g_xrows_chunked = 0;  // vf_set_xrows_chunked (test hook): force the chunked kernel

template <int NCH>
struct XStage {
    int32_t id[NCH * 32];
    int32_t cp[NCH * 32];  // +x run start: code of the -x neighbour (slot 2)
    int32_t cm[NCH * 32];  // -x run start: code of the +x neighbour (slot 1)
    uint8_t chg[NCH * 32];
    uint32_t m[NCH * 32 * 17];
};

template <int DIR, int NCH>
__device__ __forceinline__ void xrow_pass_s(int L, int lane, int bx, XStage<NCH> &S) {
    constexpr int trail = DIR > 0 ? 3 : 0;
    uint32_t carry = 0;
    bool prev_present = false;
#pragma unroll 1
    for (int x0 = 0; x0 < bx; x0 += 32) {
        const int x = DIR > 0 ? x0 + lane : bx - 1 - (x0 + lane);
        const int32_t id = (x0 + lane < bx) ? S.id[x] : -1;
        const bool present = id >= 0;
        const uint32_t pm = __ballot_sync(0xffffffffu, present);
        if (pm == 0) {
            prev_present = false;
            continue;
        }
        const bool pred = lane > 0 ? ((pm >> (lane - 1)) & 1u) : prev_present;
        uint32_t *w = S.m + 17 * (x < 0 ? 0 : x);
        uint32_t fn = 0;
        bool head = true;
        if (present) {
            uint32_t A, B;
            row_fn(w, trail, A, B);
            fn = A | (B << 16);
            if (!pred) {
                const int32_t code = DIR > 0 ? S.cp[x] : S.cm[x];
                const uint32_t c = (code == VF_NB_SOLID_NBR) ? A : B;
                fn = c | (c << 16);
            } else if (lane == 0) {
                fn = compose(fn, carry | (carry << 16));
            } else {
                head = false;
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t g = __shfl_up_sync(0xffffffffu, fn, o);
            const int hd = __shfl_up_sync(0xffffffffu, (int)head, o);
            if (lane >= o && !head) {
                fn = compose(fn, g);
                head = hd;
            }
        }
        const uint32_t out = fn & 0xffffu;
        uint32_t st = __shfl_up_sync(0xffffffffu, out, 1);
        if (lane == 0) st = carry;
        if (present && pred) {
            bool changed = false;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                const uint32_t xw = row_apply(w[r], (st >> r) & 1u, L == 0);
                changed |= (xw != w[r]);
                w[r] = xw;
            }
            if (changed) S.chg[x] = 1;
        }
        carry = __shfl_sync(0xffffffffu, out, 31);
        prev_present = (pm >> 31) & 1u;
        __syncwarp();
    }
}

#ifndef VF_XS_MINB
#define VF_XS_MINB 4  // <= 128 registers (1 lets the 4-chunk kernel take 162)
#endif
template <int NCH>
__global__ void __launch_bounds__(kXsWarps * 32, VF_XS_MINB)
    k_xrows_s(LevelInfo li, int L, const int32_t *__restrict__ map, const int32_t *__restrict__ nbr,
              uint8_t *__restrict__ masks, uint8_t *__restrict__ bflags, uint64_t *__restrict__ solid64) {
    extern __shared__ __align__(16) unsigned char s_raw[];
    const int lane = threadIdx.x & 31;
    XStage<NCH> &S = reinterpret_cast<XStage<NCH> *>(s_raw)[threadIdx.x >> 5];
    const int64_t gw = (int64_t)blockIdx.x * kXsWarps + (threadIdx.x >> 5);
    const int64_t nw = (int64_t)gridDim.x * kXsWarps;
    const int bx = li.bins[0], by = li.bins[1];
    const int64_t rows = (int64_t)by * li.bins[2];
    for (int64_t rw = gw; rw < rows; rw += nw) {
        const int j = (int)(rw % by), k = (int)(rw / by);
        if (!owns_row(li, j, k)) continue;
        const int32_t *row = map + rw * bx;
        int32_t ids[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) ids[c] = (32 * c + lane < bx) ? row[32 * c + lane] : -1;
        uint32_t anyp = 0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            S.id[32 * c + lane] = ids[c];
            S.chg[32 * c + lane] = 0;
            anyp |= __ballot_sync(0xffffffffu, ids[c] >= 0);
        }
        if (!anyp) continue;  // empty row
        __syncwarp();
        // masks + run-start codes, all loads in flight together
        uint4 mv[NCH][4];
        int32_t cpv[NCH], cmv[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int x = 32 * c + lane;
            const int32_t id = ids[c];
            cpv[c] = 0;
            cmv[c] = 0;
            if (id >= 0) {
                const uint4 *p = reinterpret_cast<const uint4 *>(masks + 64 * (int64_t)id);
#pragma unroll
                for (int q = 0; q < 4; ++q) mv[c][q] = p[q];
                if (!(x > 0 && S.id[x - 1] >= 0)) cpv[c] = nbr[27 * (int64_t)id + 2];
                if (L > 0 && !(x + 1 < bx && S.id[x + 1] >= 0)) cmv[c] = nbr[27 * (int64_t)id + 1];
            }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int x = 32 * c + lane;
            if (ids[c] >= 0) {
                uint32_t *w = S.m + 17 * x;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    w[4 * q] = mv[c][q].x; w[4 * q + 1] = mv[c][q].y;
                    w[4 * q + 2] = mv[c][q].z; w[4 * q + 3] = mv[c][q].w;
                }
                S.cp[x] = cpv[c];
                S.cm[x] = cmv[c];
            }
        }
        __syncwarp();
        xrow_pass_s<+1, NCH>(L, lane, bx, S);
        if (L > 0) xrow_pass_s<-1, NCH>(L, lane, bx, S);
        // finalize every block of the row and store the changed ones
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int x = 32 * c + lane;
            const int32_t id = ids[c];
            if (id < 0) continue;
            uint32_t w[16];
#pragma unroll
            for (int r = 0; r < 16; ++r) w[r] = S.m[17 * x + r];
            bool changed = S.chg[x] != 0;
            finalize_block(w, changed, bflags, solid64, id);
            if (changed) store_masks64(masks, id, w);
        }
        __syncwarp();
    }
}

// Hybrid for wide, sparse rows (B_L = 256): block ids and run-start codes are
// staged (all loads up front, empty 32-block chunks skipped without a load);
// masks stay in global memory, loaded per non-empty chunk as in k_xrows,
// with finalize fused into the last pass.
template <int NCH>
struct XHView {
    const int32_t *id, *cp, *cm;
};

template <int DIR, int NCH>
__device__ __forceinline__ void xrow_pass_hv(int L, int lane, int bx, const XHView<NCH> &S, uint32_t cmask,
                                            uint8_t *__restrict__ masks, bool finalize,
                                            uint8_t *__restrict__ bflags, uint64_t *__restrict__ solid64) {
    constexpr int trail = DIR > 0 ? 3 : 0;
    uint32_t carry = 0;
    bool prev_present = false;
#pragma unroll 1
    for (int c = 0; c < NCH; ++c) {
        const int x0 = 32 * c;
        // chunk of this pass: +x walks chunks 0.., -x walks x = bx-1-(x0+lane)
        const int cc = DIR > 0 ? c : (bx - 1 - x0) >> 5;
        const bool any = DIR > 0 ? ((cmask >> c) & 1u) : (((cmask >> cc) & 1u) || (x0 + 31 < bx && ((cmask >> ((bx - 1 - x0 - 31) >> 5)) & 1u)));
        if (x0 >= bx) break;
        if (!any) {
            prev_present = false;
            continue;
        }
        const int x = DIR > 0 ? x0 + lane : bx - 1 - (x0 + lane);
        const int32_t id = (x0 + lane < bx) ? S.id[x] : -1;
        const bool present = id >= 0;
        const uint32_t pm = __ballot_sync(0xffffffffu, present);
        if (pm == 0) {
            prev_present = false;
            continue;
        }
        const bool pred = lane > 0 ? ((pm >> (lane - 1)) & 1u) : prev_present;
        uint32_t w[16];
        uint32_t fn = 0;
        bool head = true;
        if (present) {
            load_masks64(masks, id, w);
            uint32_t A, B;
            row_fn(w, trail, A, B);
            fn = A | (B << 16);
            if (!pred) {
                const int32_t code = DIR > 0 ? S.cp[x] : S.cm[x];
                const uint32_t cb = (code == VF_NB_SOLID_NBR) ? A : B;
                fn = cb | (cb << 16);
            } else if (lane == 0) {
                fn = compose(fn, carry | (carry << 16));
            } else {
                head = false;
            }
        }
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t g = __shfl_up_sync(0xffffffffu, fn, o);
            const int hd = __shfl_up_sync(0xffffffffu, (int)head, o);
            if (lane >= o && !head) {
                fn = compose(fn, g);
                head = hd;
            }
        }
        const uint32_t out = fn & 0xffffu;
        uint32_t st = __shfl_up_sync(0xffffffffu, out, 1);
        if (lane == 0) st = carry;
        if (present) {
            bool changed = false;
            if (pred) {
#pragma unroll
                for (int r = 0; r < 16; ++r) {
                    const uint32_t xw = row_apply(w[r], (st >> r) & 1u, L == 0);
                    changed |= (xw != w[r]);
                    w[r] = xw;
                }
            }
            if (finalize) finalize_block(w, changed, bflags, solid64, id);
            if (changed) store_masks64(masks, id, w);
        }
        carry = __shfl_sync(0xffffffffu, out, 31);
        prev_present = (pm >> 31) & 1u;
    }
}

#ifndef VF_XH_MINB
#define VF_XH_MINB 8  // 64 registers: the max_ctas(8) grid is resident in one wave (measured)
#endif
template <int NCH>
__global__ void __launch_bounds__(kXsWarps * 32, VF_XH_MINB)
    k_xrows_h(LevelInfo li, int L, const int32_t *__restrict__ map, const int32_t *__restrict__ nbr,
              uint8_t *__restrict__ masks, uint8_t *__restrict__ bflags, uint64_t *__restrict__ solid64) {
    __shared__ int32_t s_id[kXsWarps][NCH * 32], s_cp[kXsWarps][NCH * 32], s_cm[kXsWarps][NCH * 32];
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kXsWarps + wi;
    const int64_t nw = (int64_t)gridDim.x * kXsWarps;
    const int bx = li.bins[0], by = li.bins[1];
    const int64_t rows = (int64_t)by * li.bins[2];
    for (int64_t rw = gw; rw < rows; rw += nw) {
        const int j = (int)(rw % by), k = (int)(rw / by);
        if (!owns_row(li, j, k)) continue;
        const int32_t *row = map + rw * bx;
        int32_t ids[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) ids[c] = (32 * c + lane < bx) ? row[32 * c + lane] : -1;
        uint32_t cmask = 0;
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            s_id[wi][32 * c + lane] = ids[c];
            cmask |= (__ballot_sync(0xffffffffu, ids[c] >= 0) ? 1u : 0u) << c;
        }
        if (!cmask) continue;
        __syncwarp();
        int32_t cpv[NCH], cmv[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            const int x = 32 * c + lane;
            const int32_t id = ids[c];
            cpv[c] = 0;
            cmv[c] = 0;
            if (id >= 0) {
                if (!(x > 0 && s_id[wi][x - 1] >= 0)) cpv[c] = nbr[27 * (int64_t)id + 2];
                if (L > 0 && !(x + 1 < bx && s_id[wi][x + 1] >= 0)) cmv[c] = nbr[27 * (int64_t)id + 1];
            }
        }
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
            s_cp[wi][32 * c + lane] = cpv[c];
            s_cm[wi][32 * c + lane] = cmv[c];
        }
        __syncwarp();
        XHView<NCH> V{s_id[wi], s_cp[wi], s_cm[wi]};
        xrow_pass_hv<+1, NCH>(L, lane, bx, V, cmask, masks, L == 0, bflags, solid64);
        if (L > 0) {
            __syncwarp();
            xrow_pass_hv<-1, NCH>(L, lane, bx, V, cmask, masks, true, bflags, solid64);
        }
        __syncwarp();
    }
}

template <int NCH>
static int launch_xrows_s(const LevelInfo &li, int L, const int32_t *map, vf_grid *g, cudaStream_t st) {
    const size_t smem = kXsWarps * sizeof(XStage<NCH>);
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_xrows_s<NCH>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = true;
    }
    const int64_t rows = (int64_t)li.bins[1] * li.bins[2];
    int64_t grid = (rows + kXsWarps - 1) / kXsWarps;
    const int64_t cap = max_ctas(NCH <= 2 ? 16 : (NCH <= 4 ? VF_GRID_XS4 : 4));
    if (grid > cap) grid = cap;
    k_xrows_s<NCH><<<(int)grid, kXsWarps * 32, smem, st>>>(li, L, map, g->d_nbr, g->d_masks, g->d_bflags,
                                                           g->d_solid64);
    return check_launch("k_xrows");
}

size_t propagate_level_workspace_size(const vf_config &cfg, int L) {
    const int64_t nb = (int64_t)(cfg.nb[0] << L) * (cfg.nb[1] << L) * (cfg.nb[2] << L);
    return ((size_t)nb * sizeof(int32_t) + 255) & ~(size_t)255;
}

int propagate_level_impl(const LevelInfo &li, vf_grid *g, int L, void *ws, size_t ws_bytes,
                         cudaStream_t st) {
    const int64_t nb = (int64_t)li.bins[0] * li.bins[1] * li.bins[2];
    if (ws_bytes < (size_t)nb * sizeof(int32_t)) return set_error(VF_EARG, "propagate workspace too small");
    int32_t *map = (int32_t *)ws;
    cudaMemsetAsync(map, 0xff, sizeof(int32_t) * (size_t)nb, st);
    kt_point("memset:level_map");
    k_level_map<<<max_ctas(8), 256, 0, st>>>(L, li, g->d_level_start, g->d_coords, map);
    int rc = check_launch("k_level_map");
    if (rc) return rc;
    const int bx = li.bins[0];
    if (!g_xrows_chunked) {
        if (bx <= 32) return launch_xrows_s<1>(li, L, map, g, st);
        if (bx <= 64) return launch_xrows_s<2>(li, L, map, g, st);
        if (bx <= 128) return launch_xrows_s<4>(li, L, map, g, st);
        // (8 chunks staged: 215 registers and 83 KB of shared memory per CTA --
        // slower next to the concurrent link enumeration; ids / codes only)
        if (bx <= 256) {
            const int64_t rows = (int64_t)li.bins[1] * li.bins[2];
            int64_t grid = (rows + kXsWarps - 1) / kXsWarps;
            if (grid > max_ctas(8)) grid = max_ctas(8);
            k_xrows_h<8><<<(int)grid, kXsWarps * 32, 0, st>>>(li, L, map, g->d_nbr, g->d_masks, g->d_bflags,
                                                              g->d_solid64);
            return check_launch("k_xrows");
        }
    }
    int64_t rows = (int64_t)li.bins[1] * li.bins[2];
    int64_t grid = (rows + kXrowWarps - 1) / kXrowWarps;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_xrows<<<(int)grid, kXrowWarps * 32, 0, st>>>(li, L, map, g->d_nbr, g->d_masks, g->d_bflags,
                                                   g->d_solid64);
    return check_launch("k_xrows");
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

extern "C" int vf_set_xrows_chunked(int on) {
    const int old = vf::g_xrows_chunked;
    if (on >= 0) vf::g_xrows_chunked = on ? 1 : 0;
    return old;
}
