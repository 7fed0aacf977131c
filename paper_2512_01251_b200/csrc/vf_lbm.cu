// vf_lbm.cu -- the LUT consumer: one D3Q27 BGK collide/stream step of one
// grid level with SBB / interpolated bounce-back (Bouzidi linear) wall links
// read from the cut-link LUT (SPEC.md:398-411 collide_stream_level,
// SPEC.md:392-397 equilibrium, SPEC.md:436-440 accumulate_forces;
// SURVEY.md §8(f) next #1) and the interface exchange between levels
// (§8(f) next #3; step_hierarchy in solver.py).  Oracle: oracle/lbm_oracle.c (same rules, FP64).
//
// State = post-collision populations, SoA f[q][cell] with cell = (block - s)
// * 64 + t over the level's blocks [s, e): a warp reads 32 consecutive cells
// of one block per population, so the 27 gathers of the pull stream stay
// within a block or its face neighbour (coalesced).  One thread per cell:
//   pull f_o(x) = f_o^post(x - c_o); across a block face through the 27
//   neighbour slots; wall link when x - c_o is SOLID (q_w = LUT[cmap[b]][q][t],
//   q = opp(o)); inlet / outlet / SBB on the domain faces;
//   moments, BGK relaxation to the second-order equilibrium, store.
// GHOST cells are held (interface exchange), SOLID cells untouched.  The
// momentum exchange of the wall links is reduced per block and accumulated
// in FP64.  Bytes per cell: 27 x 4 read + 27 x 4 written (+ 1 B mask, 108 +
// 216 B of neighbour ids / solid words per block): HBM-bound.
#include "vf_common.cuh"
#include "vf_internal.h"

namespace vf {

__constant__ float c_lw[27] = {8.f / 27, 2.f / 27, 2.f / 27, 2.f / 27, 2.f / 27, 2.f / 27, 2.f / 27,
                               1.f / 54, 1.f / 54, 1.f / 54, 1.f / 54, 1.f / 54, 1.f / 54, 1.f / 54,
                               1.f / 54, 1.f / 54, 1.f / 54, 1.f / 54, 1.f / 54, 1.f / 216, 1.f / 216,
                               1.f / 216, 1.f / 216, 1.f / 216, 1.f / 216, 1.f / 216, 1.f / 216};

__device__ __forceinline__ int lopp(int q) { return q == 0 ? 0 : ((q & 1) ? q + 1 : q - 1); }

// level cell of (block b, cell I,J,K) shifted by (dx,dy,dz) in {-1,0,1}^3
__device__ __forceinline__ int32_t cell_at(const int32_t *__restrict__ nbr, int32_t b, int I, int J,
                                           int K, int dx, int dy, int dz, int &t) {
    const int X = I + dx, Y = J + dy, Z = K + dz;
    const int ox = X < 0 ? -1 : (X > 3 ? 1 : 0), oy = Y < 0 ? -1 : (Y > 3 ? 1 : 0),
              oz = Z < 0 ? -1 : (Z > 3 ? 1 : 0);
    t = (X & 3) + 4 * (Y & 3) + 16 * (Z & 3);
    if (!(ox | oy | oz)) return b;
    return __ldg(nbr + 27 * (int64_t)b + slot_of(ox, oy, oz));
}

// A step is two passes over the level's blocks, split by cell.  A cell is
// SIMPLE when it is not GHOST and none of the 27 cells around it (itself
// included) is SOLID or outside the level / domain: its pull needs no
// boundary rule.  The simple set of a block is one 64-bit word, the
// 26-neighbour dilation (dil_x/y/z) of the "bad" words of the 27 blocks
// around it (solid64; every cell of a missing or outside neighbour is bad).
//   k_lbm_bulk    every block, its simple cells: 27 unconditional pulls
//                 through a per-CTA table (source neighbour code and cell of
//                 population o at cell t), BGK, store; SOLID / GHOST cells
//                 held (copied).  Blocks with any other cell are appended to
//                 a list.
//   k_lbm_special the listed blocks, their other cells only: domain faces (lateral SBB, inlet velocity
//                 bounce-back, outlet anti-bounce-back), wall links (SBB or
//                 Bouzidi linear IBB with q_w from the LUT) with the
//                 momentum exchange.
// The passes write disjoint cells from the same f_in, so they commute.
constexpr int kLbmWarps = 8;
#ifndef VF_LBM_MINB
#define VF_LBM_MINB 3  // 85 registers (with the staging prefetch; 4: 64 + 96 B spills, measured slower)
#endif
#ifndef VF_LBM_FUSED_MINB  // fused variant (-DVF_LBM_FUSED): measured slower
#define VF_LBM_FUSED_MINB 3
#endif
#ifndef VF_LBM_SPECIAL_MINB
#define VF_LBM_SPECIAL_MINB 3
#endif

// bad words of the 27 blocks around b (code (dx+1) + 3(dy+1) + 9(dz+1)) ->
// the simple cells of b (ghost: the block's GHOST cells)
// (codes in `skip` count as not bad)
__device__ __forceinline__ uint64_t simple_cells(const unsigned long long *bad, uint64_t ghost, uint32_t skip = 0) {
    uint64_t pl[3];
#pragma unroll
    for (int dz = 0; dz < 3; ++dz) {
        uint64_t col[3];
#pragma unroll
        for (int dy = 0; dy < 3; ++dy) {
            const int c = 3 * dy + 9 * dz;
            const uint64_t b0 = (skip >> c) & 1u ? 0ull : bad[c], b1 = (skip >> (c + 1)) & 1u ? 0ull : bad[c + 1],
                           b2 = (skip >> (c + 2)) & 1u ? 0ull : bad[c + 2];
            col[dy] = dil_x(b0, b1, b2);
        }
        pl[dz] = dil_y(col[0], col[1], col[2]);
    }
    return ~(dil_z(pl[0], pl[1], pl[2]) | ghost);
}

// stage the 27 neighbour ids (code order) and bad words of block b; returns
// the block's GHOST cells (bit t)
__device__ __forceinline__ uint64_t stage_block(int32_t s, int32_t e, int32_t b, int lane,
                                                const int32_t *__restrict__ nbr,
                                                const uint8_t *__restrict__ masks,
                                                const uint64_t *__restrict__ solid64, int32_t *nb,
                                                unsigned long long *bad) {
    if (lane < 27) {
        const int dx = lane % 3 - 1, dy = (lane / 3) % 3 - 1, dz = lane / 9 - 1;
        const int32_t v = (lane == 13) ? b : __ldg(nbr + 27 * (int64_t)b + slot_of(dx, dy, dz));
        nb[lane] = v;
        bad[lane] = (v >= s && v < e) ? __ldg(reinterpret_cast<const unsigned long long *>(solid64) + v) : ~0ull;
    }
    const bool g0 = masks[64 * (int64_t)b + lane] == VF_GHOST, g1 = masks[64 * (int64_t)b + lane + 32] == VF_GHOST;
    const uint64_t ghost = (uint64_t)__ballot_sync(0xffffffffu, g0) | ((uint64_t)__ballot_sync(0xffffffffu, g1) << 32);
    __syncwarp();
    return ghost;
}

// Codes whose neighbour lies outside the domain through a lateral face
// (lateral SBB: f_o(x) = f_opp(o)(x)) -- every outside face when the x faces
// are walls too, else those not through the x = 0 / x = l_x faces of an
// x-boundary block (inlet / outlet).  lane < 27 holds code `lane`'s id.
__device__ __forceinline__ uint32_t lateral_codes(int32_t v, int lane, int bx, int cells_x, int open_x) {
    const int dx = lane % 3 - 1;
    const bool xout = (dx < 0 && bx == 0) || (dx > 0 && 4 * bx + 4 >= cells_x);
    return __ballot_sync(0xffffffffu, lane < 27 && v == VF_NB_OUTSIDE && !(open_x && xout));
}
// the cells whose only boundary rule is the lateral SBB (not simple, not
// held): the complement of the dilation of the other bad words
__device__ __forceinline__ uint64_t lateral_cells(const unsigned long long *bad, uint64_t ghost, uint32_t lat,
                                                  uint64_t simple, uint64_t held) {
    return lat ? (simple_cells(bad, ghost, lat) & ~simple & ~held) : 0ull;
}

// source of population o at cell t: (neighbour code << 6) | cell
__host__ __device__ constexpr uint16_t pull_entry(int o, int t) {
    const int X = (t & 3) - c27(o, 0), Y = ((t >> 2) & 3) - c27(o, 1), Z = (t >> 4) - c27(o, 2);
    const int code = ((X >> 2) + 1) + 3 * ((Y >> 2) + 1) + 9 * ((Z >> 2) + 1);
    return (uint16_t)((code << 6) | ((X & 3) + 4 * (Y & 3) + 16 * (Z & 3)));
}
struct __align__(16) PullTable {
    uint16_t v[27 * 64];
};
constexpr PullTable make_pull_table() {
    PullTable p{};
    for (int i = 0; i < 27 * 64; ++i) p.v[i] = pull_entry(i >> 6, i & 63);
    return p;
}
// compile-time table in global memory, copied to shared memory per CTA
__device__ const __align__(16) PullTable g_pull = make_pull_table();

// BGK relaxation of the pulled populations of cell x to the second-order
// equilibrium, stored to fout
__device__ __forceinline__ void bgk_store(float *f, float omega, float *__restrict__ fout, int64_t n, int64_t x) {
    float rho = 0.f, u0 = 0.f, u1 = 0.f, u2 = 0.f;
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        rho += f[o];
        u0 += f[o] * c27(o, 0);
        u1 += f[o] * c27(o, 1);
        u2 += f[o] * c27(o, 2);
    }
    const float ir = 1.0f / rho;
    u0 *= ir; u1 *= ir; u2 *= ir;
    const float uu = 1.5f * (u0 * u0 + u1 * u1 + u2 * u2);
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        const float cu = c27(o, 0) * u0 + c27(o, 1) * u1 + c27(o, 2) * u2;
        const float feq = c_lw[o] * rho * (1.0f + 3.0f * cu + 4.5f * cu * cu - uu);
        fout[o * n + x] = f[o] + (feq - f[o]) * omega;
    }
}

__global__ void __launch_bounds__(kLbmWarps * 32, VF_LBM_MINB)
    k_lbm_bulk(int32_t s, int32_t e, int cells_x, int open_x, const int32_t *__restrict__ coords,
               const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
               const uint64_t *__restrict__ solid64, const float *__restrict__ fin, float *__restrict__ fout,
               float omega, int32_t *__restrict__ list, int32_t *__restrict__ n_list) {
    __shared__ __align__(16) uint16_t s_pull[27 * 64];
    __shared__ int32_t s_nb[kLbmWarps][27];
    __shared__ unsigned long long s_bad[kLbmWarps][27];
    for (int i = threadIdx.x; i < 27 * 64 / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(s_pull)[i] = reinterpret_cast<const uint4 *>(g_pull.v)[i];
    __syncthreads();
    const int64_t n = (int64_t)(e - s) * 64;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int nblk = e - s, stride = gridDim.x * kLbmWarps;
    // the next block's staging is prefetched into registers: its neighbour
    // ids and GHOST bits while this block starts, its solid words between
    // this block's two halves (their ids have arrived by then)
    int32_t nv = 0;
    unsigned long long nbad = 0ull;
    bool ng0 = false, ng1 = false;
    auto fetch_ids = [&](int lbn) {
        const int32_t bn = s + lbn;
        if (lane < 27) {
            const int dx = lane % 3 - 1, dy = (lane / 3) % 3 - 1, dz = lane / 9 - 1;
            nv = (lane == 13) ? bn : __ldg(nbr + 27 * (int64_t)bn + slot_of(dx, dy, dz));
        }
        ng0 = masks[64 * (int64_t)bn + lane] == VF_GHOST;
        ng1 = masks[64 * (int64_t)bn + lane + 32] == VF_GHOST;
    };
    auto fetch_bad = [&]() {
        if (lane < 27)
            nbad = (nv >= s && nv < e) ? __ldg(reinterpret_cast<const unsigned long long *>(solid64) + nv) : ~0ull;
    };
    int lb = blockIdx.x * kLbmWarps + w;
    if (lb < nblk) {
        fetch_ids(lb);
        fetch_bad();
    }
    for (; lb < nblk; lb += stride) {
        const int32_t b = s + lb;
        const int lbn = lb + stride;
        __syncwarp();
        if (lane < 27) {
            s_nb[w][lane] = nv;
            s_bad[w][lane] = nbad;
        }
        const uint64_t ghost = (uint64_t)__ballot_sync(0xffffffffu, ng0) | ((uint64_t)__ballot_sync(0xffffffffu, ng1) << 32);
        if (lbn < nblk) fetch_ids(lbn);  // in flight while this block is classified and its first half pulled
        __syncwarp();
        const uint64_t simple = simple_cells(s_bad[w], ghost);
        const uint64_t held = ghost | s_bad[w][13];  // GHOST / SOLID: f_out = f_in
        const int32_t v = lane < 27 ? s_nb[w][lane] : 0;
        uint32_t lat = 0;
        if (__any_sync(0xffffffffu, lane < 27 && v == VF_NB_OUTSIDE))  // a domain-face block
            lat = lateral_codes(v, lane, __ldg(coords + 4 * (int64_t)b), cells_x, open_x);
        const uint64_t sbb = lateral_cells(s_bad[w], ghost, lat, simple, held);
        if (lane < 27) s_nb[w][lane] = (v - s) * 64;  // pulls only reach level cells (or lateral SBB)
        __syncwarp();
        if ((simple | held | sbb) != ~0ull && lane == 0) list[atomicAdd(n_list, 1)] = lb;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            if (h == 1 && lbn < nblk) fetch_bad();
            const int t = lane + 32 * h;
            if (!((simple >> t) & 1ull)) continue;
            float f[27];
#pragma unroll
            for (int o = 0; o < 27; ++o) {
                const uint32_t p = s_pull[o * 64 + t];
                f[o] = __ldg(fin + o * n + (s_nb[w][p >> 6] + (int)(p & 63u)));
            }
            bgk_store(f, omega, fout, n, (int64_t)lb * 64 + t);
        }
        if (sbb) {  // warp-uniform: cells next to a lateral domain face only
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int t = lane + 32 * h;
                if (!((sbb >> t) & 1ull)) continue;
                const int64_t x = (int64_t)lb * 64 + t;
                float f[27];
#pragma unroll
                for (int o = 0; o < 27; ++o) {
                    const uint32_t p = s_pull[o * 64 + t];
                    const int q = o == 0 ? 0 : ((o & 1) ? o + 1 : o - 1);
                    f[o] = (lat >> (p >> 6)) & 1u ? __ldg(fin + q * n + x)
                                                  : __ldg(fin + o * n + (s_nb[w][p >> 6] + (int)(p & 63u)));
                }
                bgk_store(f, omega, fout, n, x);
            }
        }
        if (held) {  // warp-uniform
#pragma unroll 1
            for (int h = 0; h < 2; ++h) {
                const int t = lane + 32 * h;
                if (!((held >> t) & 1ull)) continue;
                const int64_t x = (int64_t)lb * 64 + t;
#pragma unroll
                for (int q = 0; q < 27; ++q) fout[q * n + x] = __ldg(fin + q * n + x);
            }
        }
    }
}

// the special cells of block b (staged: nb ids, sol words, ghost), packed
// onto the lanes (k-th set bit of spec); wall momentum exchange into F
__device__ __forceinline__ void special_cells(int32_t s, int32_t e, int cells_x, int32_t b, int lb, int lane,
                                              uint64_t ghost, uint64_t spec, const int32_t *nb,
                                              const unsigned long long *sol, const uint16_t *pull,
                                              const int32_t *__restrict__ coords, const int32_t *__restrict__ cmap,
                                              const float *__restrict__ lengths, const float *__restrict__ fin,
                                              float *__restrict__ fout, const vf_flow &flow, float &Fx, float &Fy,
                                              float &Fz) {
    const int64_t n = (int64_t)(e - s) * 64;
    const float omega = 1.0f / (float)flow.tau;
    const float uin[3] = {(float)flow.u_in[0], (float)flow.u_in[1], (float)flow.u_in[2]};
    const uint64_t held = ghost | sol[13];
    const int bx = __ldg(coords + 4 * (int64_t)b);
    const int32_t slot = flow.ibb ? cmap[b] : -1;
    // the block's special cells, packed onto the lanes (k-th set bit)
    const uint32_t lo = (uint32_t)spec, hi = (uint32_t)(spec >> 32);
    const int nlo = __popc(lo), cnt = nlo + __popc(hi);
#pragma unroll 1
    for (int k0 = 0; k0 < cnt; k0 += 32) {
        const int k = k0 + lane;
        if (k >= cnt) continue;
        const int t = k < nlo ? (int)__fns(lo, 0, k + 1) : 32 + (int)__fns(hi, 0, k - nlo + 1);
        const int64_t x = (int64_t)lb * 64 + t;
        if ((held >> t) & 1ull) {  // SOLID / GHOST: held
#pragma unroll
            for (int q = 0; q < 27; ++q) fout[q * n + x] = fin[q * n + x];
            continue;
        }
        const int I = t & 3;
        // outlet cells (x = l_x face): velocity of x for the anti-bounce-back
        float v0 = 0.f, v1 = 0.f, v2 = 0.f;
        if (flow.open_x && 4 * bx + I == cells_x - 1) {
            float rx = 0.f;
#pragma unroll
            for (int q = 0; q < 27; ++q) {
                const float v = fin[q * n + x];
                rx += v;
                v0 += v * c27(q, 0);
                v1 += v * c27(q, 1);
                v2 += v * c27(q, 2);
            }
            v0 /= rx; v1 /= rx; v2 /= rx;
        }
        float f[27];
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            const uint32_t p = pull[o * 64 + t];
            const int code = (int)(p >> 6), ty = (int)(p & 63u);
            const int32_t y = nb[code];
            if (!((sol[code] >> ty) & 1ull)) {  // a level cell that is not SOLID
                f[o] = fin[o * n + (int64_t)(y - s) * 64 + ty];
                continue;
            }
            const int q = o == 0 ? 0 : ((o & 1) ? o + 1 : o - 1);
            const float fq = fin[q * n + x];
            float v = fq;  // SBB: lateral faces, SBB walls
            if (y == VF_NB_OUTSIDE) {
                const int gx = 4 * bx + I - c27(o, 0);
                if (flow.open_x && gx < 0) {  // inlet: velocity bounce-back, rho_w = 1
                    v -= 6.0f * c_lw[q] * (c27(q, 0) * uin[0] + c27(q, 1) * uin[1] + c27(q, 2) * uin[2]);
                } else if (flow.open_x && gx >= cells_x) {  // outlet: anti-bounce-back, rho_w = 1
                    const float cq = c27(q, 0) * v0 + c27(q, 1) * v1 + c27(q, 2) * v2;
                    v = -fq + 2.0f * c_lw[q] * (1.0f + 4.5f * cq * cq - 1.5f * (v0 * v0 + v1 * v1 + v2 * v2));
                }
            } else {  // wall link x -> y (SOLID cell, or a missing block next to ghosts)
                const float qw = slot >= 0 ? lengths[((int64_t)slot * 27 + q) * 64 + t] : -1.0f;
                if (qw > 0.0f && qw < 0.5f) {
                    // second node behind x: x + c_o = x - c_q (the source of population q)
                    const uint32_t p2 = pull[q * 64 + t];
                    const int code2 = (int)(p2 >> 6), tz = (int)(p2 & 63u);
                    if (!((sol[code2] >> tz) & 1ull))
                        v = 2.0f * qw * fq + (1.0f - 2.0f * qw) *
                                                 fin[q * n + (int64_t)(nb[code2] - s) * 64 + tz];
                } else if (qw >= 0.5f) {
                    v = fq / (2.0f * qw) + (2.0f * qw - 1.0f) / (2.0f * qw) * fin[o * n + x];
                }
                Fx += (fq + v) * c27(q, 0);
                Fy += (fq + v) * c27(q, 1);
                Fz += (fq + v) * c27(q, 2);
            }
            f[o] = v;
        }
        bgk_store(f, omega, fout, n, x);
    }
}

// per-block force partial: a fixed lane tree, stored at the block's local
// id -- independent of which warp took the block
__device__ __forceinline__ void block_force(double *part, int lb, int lane, float Fx, float Fy, float Fz) {
    __syncwarp();
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Fx += __shfl_xor_sync(0xffffffffu, Fx, off);
        Fy += __shfl_xor_sync(0xffffffffu, Fy, off);
        Fz += __shfl_xor_sync(0xffffffffu, Fz, off);
    }
    if (lane == 0) {
        part[3 * (int64_t)lb + 0] = (double)Fx;
        part[3 * (int64_t)lb + 1] = (double)Fy;
        part[3 * (int64_t)lb + 2] = (double)Fz;
    }
}

__global__ void __launch_bounds__(kLbmWarps * 32, VF_LBM_SPECIAL_MINB)
    k_lbm_special(int32_t s, int32_t e, int cells_x, const int32_t *__restrict__ coords,
                  const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
                  const uint64_t *__restrict__ solid64, const int32_t *__restrict__ cmap,
                  const float *__restrict__ lengths, const float *__restrict__ fin,
                  float *__restrict__ fout, vf_flow flow, const int32_t *__restrict__ list,
                  const int32_t *__restrict__ n_list, double *__restrict__ part) {
    __shared__ __align__(16) uint16_t s_pull[27 * 64];
    __shared__ int32_t s_nb[kLbmWarps][27];
    __shared__ unsigned long long s_sol[kLbmWarps][27];
    for (int i = threadIdx.x; i < 27 * 64 / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(s_pull)[i] = reinterpret_cast<const uint4 *>(g_pull.v)[i];
    __syncthreads();
    const int nitems = *n_list;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int it = blockIdx.x * kLbmWarps + w; it < nitems; it += gridDim.x * kLbmWarps) {
        float Fx = 0.f, Fy = 0.f, Fz = 0.f;  // this block's wall momentum exchange
        const int lb = list[it];
        const int32_t b = s + lb;
        __syncwarp();
        const uint64_t ghost = stage_block(s, e, b, lane, nbr, masks, solid64, s_nb[w], s_sol[w]);
        // the cells of this pass: neither simple, lateral-SBB-only nor held
        // (the bulk pass's)
        const uint64_t simple = simple_cells(s_sol[w], ghost), held = ghost | s_sol[w][13];
        const int32_t v = lane < 27 ? s_nb[w][lane] : 0;
        uint32_t lat = 0;
        if (__any_sync(0xffffffffu, lane < 27 && v == VF_NB_OUTSIDE))
            lat = lateral_codes(v, lane, __ldg(coords + 4 * (int64_t)b), cells_x, flow.open_x);
        const uint64_t spec = ~(simple | held | lateral_cells(s_sol[w], ghost, lat, simple, held));
        special_cells(s, e, cells_x, b, lb, lane, ghost, spec, s_nb[w], s_sol[w], s_pull, coords, cmap, lengths,
                      fin, fout, flow, Fx, Fy, Fz);
        if (part) block_force(part, lb, lane, Fx, Fy, Fz);
    }
}

// fused step: every block's simple cells (fast pulls), then its special
// cells (the general path) in the same warp
__global__ void __launch_bounds__(kLbmWarps * 32, VF_LBM_FUSED_MINB)
    k_lbm_cells(int32_t s, int32_t e, int cells_x, const int32_t *__restrict__ coords,
                const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
                const uint64_t *__restrict__ solid64, const int32_t *__restrict__ cmap,
                const float *__restrict__ lengths, const float *__restrict__ fin, float *__restrict__ fout,
                vf_flow flow, double *__restrict__ part) {
    __shared__ __align__(16) uint16_t s_pull[27 * 64];
    __shared__ int32_t s_nb[kLbmWarps][27], s_off[kLbmWarps][27];
    __shared__ unsigned long long s_sol[kLbmWarps][27];
    for (int i = threadIdx.x; i < 27 * 64 / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(s_pull)[i] = reinterpret_cast<const uint4 *>(g_pull.v)[i];
    __syncthreads();
    const int64_t n = (int64_t)(e - s) * 64;
    const float omega = 1.0f / (float)flow.tau;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int lb = blockIdx.x * kLbmWarps + w; lb < e - s; lb += gridDim.x * kLbmWarps) {
        const int32_t b = s + lb;
        __syncwarp();
        const uint64_t ghost = stage_block(s, e, b, lane, nbr, masks, solid64, s_nb[w], s_sol[w]);
        const uint64_t simple = simple_cells(s_sol[w], ghost);
        if (lane < 27) s_off[w][lane] = (s_nb[w][lane] - s) * 64;  // used for level cells only
        __syncwarp();
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            if (!((simple >> t) & 1ull)) continue;
            float f[27];
#pragma unroll
            for (int o = 0; o < 27; ++o) {
                const uint32_t p = s_pull[o * 64 + t];
                f[o] = __ldg(fin + o * n + (s_off[w][p >> 6] + (int)(p & 63u)));
            }
            bgk_store(f, omega, fout, n, (int64_t)lb * 64 + t);
        }
        if (simple != ~0ull) {  // warp-uniform
            float Fx = 0.f, Fy = 0.f, Fz = 0.f;
            special_cells(s, e, cells_x, b, lb, lane, ghost, ~simple, s_nb[w], s_sol[w], s_pull, coords, cmap,
                          lengths, fin, fout, flow, Fx, Fy, Fz);
            if (part) block_force(part, lb, lane, Fx, Fy, Fz);
        }
    }
}

// d_force += sum over the level's blocks of the per-block partials, in block
// order with a fixed reduction tree (identical force series
// across runs; the special-block list order depends on atomics)
__global__ void __launch_bounds__(1024) k_lbm_force_reduce(int32_t nb, const double *__restrict__ part,
                                                           double *__restrict__ d_force) {
    __shared__ double s_r[3][1024];
    double a[3] = {0.0, 0.0, 0.0};
    for (int32_t b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
        for (int c = 0; c < 3; ++c) a[c] += part[3 * (int64_t)b + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) s_r[c][threadIdx.x] = a[c];
    __syncthreads();
    for (int o = 512; o > 0; o >>= 1) {
        if ((int)threadIdx.x < o)
#pragma unroll
            for (int c = 0; c < 3; ++c) s_r[c][threadIdx.x] += s_r[c][threadIdx.x + o];
        __syncthreads();
    }
    if (threadIdx.x < 3) d_force[threadIdx.x] += s_r[threadIdx.x][0];
}

// equilibrium initialisation of the level's fluid cells (SOLID cells zero)
__global__ void k_lbm_init(int32_t s, int32_t e, const uint8_t *__restrict__ masks, float rho,
                           float u0, float u1, float u2, float *__restrict__ f) {
    const int64_t n = (int64_t)(e - s) * 64;
    const float uu = 1.5f * (u0 * u0 + u1 * u1 + u2 * u2);
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const bool solid = masks[64 * (int64_t)s + x] == VF_SOLID;
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            const float cu = c27(o, 0) * u0 + c27(o, 1) * u1 + c27(o, 2) * u2;
            f[o * n + x] = solid ? 0.0f : c_lw[o] * rho * (1.0f + 3.0f * cu + 4.5f * cu * cu - uu);
        }
    }
}

// ---- multi-level interface exchange --
// Cell-centred 2:1 layout: fine global cell g (per axis, level L+1) lies in
// coarse cell G = g >> 1 at offset s/4 coarse cells, s = +1 for odd g, -1
// for even g.  Fine <- coarse fills the GHOST cells of level L+1 (A14) by
// tensor-product interpolation of the coarse post-collision populations,
// blended in time, f^ = sum_k w_k ((1 - theta) f_old + theta f_new)(G + s k):
//   order 3 (cubic Lagrange, nodes k = -1, 0, 1, 2 at x = 1/4):
//            w = (-7, 105, 35, -5) / 128,
//   order 1 (linear, k = 0, 1): w = (3, 1) / 4,
// falling back 3 -> 1 -> 0 (the coarse cell G itself) when a stencil cell is
// outside the level (negative neighbour code) or SOLID; a ghost with no
// usable G is held.  The non-equilibrium part is then rescaled,
// f = feq(rho^, u^) + alpha (f^ - feq(rho^, u^)) (alpha = 1: f = f^).
// Coarse <- fine (k_lbm_restrict) averages the 8 children of every coarse
// cell of a refined block that is neither SOLID, INTERFACE nor GHOST and
// whose children hold no GHOST cell, over the non-SOLID children, with the
// inverse rescale beta.  Weights are dyadic (exact in FP32); sums in FP32.
__constant__ float c_w3[4] = {-7.0f / 128, 105.0f / 128, 35.0f / 128, -5.0f / 128};

// rescale of the non-equilibrium part (in place on f[27]); a == 1: identity
__device__ __forceinline__ void neq_rescale(float *f, float a) {
    if (a == 1.0f) return;
    float rho = 0.f, u0 = 0.f, u1 = 0.f, u2 = 0.f;
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        rho += f[o];
        u0 += f[o] * c27(o, 0);
        u1 += f[o] * c27(o, 1);
        u2 += f[o] * c27(o, 2);
    }
    if (!(rho > 0.0f)) return;
    const float ir = 1.0f / rho;
    u0 *= ir; u1 *= ir; u2 *= ir;
    const float uu = 1.5f * (u0 * u0 + u1 * u1 + u2 * u2);
#pragma unroll
    for (int o = 0; o < 27; ++o) {
        const float cu = c27(o, 0) * u0 + c27(o, 1) * u1 + c27(o, 2) * u2;
        const float feq = c_lw[o] * rho * (1.0f + 3.0f * cu + 4.5f * cu * cu - uu);
        f[o] = feq + a * (f[o] - feq);
    }
}

__global__ void k_lbm_parents(int32_t n_blocks, const int32_t *__restrict__ child, int32_t *__restrict__ parent) {
    for (int32_t b = blockIdx.x * blockDim.x + threadIdx.x; b < n_blocks; b += gridDim.x * blockDim.x) {
        const int32_t c = child[b];
        if (c >= 0)
#pragma unroll
            for (int o = 0; o < 8; ++o) parent[c + o] = b;
    }
}

// CTA per sibling group: the fine level is made of groups of 8 children of
// one coarse parent P (ids first child + octant), warp w <-> child octant w.
// Every stencil of the group (cubic: +-2 coarse cells around a fine cell's
// coarse cell) lies in the 8x8x8 coarse cells around P, box index
// (lx + 2) + 8 (ly + 2) + 64 (lz + 2) for P-local cell l.  Their level-local
// ids (or -1: outside the level / SOLID) are staged once per group, with a
// bit plane per box z (bit x + 8 y: usable) for the per-cell order test.
// Per round of kFillQ populations the CTA stages the 512 time-blended coarse
// values and interpolates the whole group separably: x (fine X 0..7 of the
// group x box rows y, z: 512 outputs), y (fine X, Y x box z: 512), then z for
// the ghost cells -- two outputs per thread per pass, taps in ascending
// coarse index so the separable passes and the per-cell fallback (a stencil
// cell missing: cubic -> linear -> the coarse cell itself) sum identically.
// A thread's x parity in pass 1 is tid & 1, its y parity in pass 2
// (tid >> 3) & 1 and its cells' z parity (lane >> 4) & 1: the tap weights
// are registers.
constexpr int kFillQ = 9;  // populations per round (3 rounds)
#ifndef VF_FILL_MINB
#define VF_FILL_MINB 2
#endif

__device__ __forceinline__ float axis_w(int ord, int k) {
    return ord == 3 ? c_w3[k] : (ord == 1 ? (k ? 0.25f : 0.75f) : 1.0f);
}
__host__ __device__ constexpr int ntaps(int ord) { return ord == 3 ? 4 : (ord == 1 ? 2 : 1); }
// first tap relative to the coarse cell of a fine cell with odd (pos) or
// even index; weight of the j-th tap in ascending order
__host__ __device__ constexpr int tap0(int ord, bool pos) {
    return ord == 3 ? (pos ? -1 : -2) : (ord == 1 ? (pos ? 0 : -1) : 0);
}
__device__ __forceinline__ float wtap(int ord, bool pos, int j) {
    return axis_w(ord, pos ? j : ntaps(ord) - 1 - j);
}
// stencil of order ord starting at box cell (x0, y0, z0) entirely usable
__device__ __forceinline__ bool stencil_ok(const unsigned long long *ok, int ord, int x0, int y0, int z0) {
    const int nt = ntaps(ord);
    const uint64_t m = nt == 4 ? 0x0F0F0F0Full : (nt == 2 ? 0x0303ull : 1ull);
    for (int k = 0; k < nt; ++k)
        if (((ok[z0 + k] >> (x0 + 8 * y0)) & m) != m) return false;
    return true;
}

template <int ORD, bool BLEND>
__global__ void __launch_bounds__(256, VF_FILL_MINB)
    k_lbm_fill_ghosts(int32_t sf, int32_t ef, int32_t sc, int32_t ec, const int32_t *__restrict__ nbr,
                      const int32_t *__restrict__ child, const uint8_t *__restrict__ masks,
                      const int32_t *__restrict__ parent, const float *__restrict__ fold,
                      const float *__restrict__ fnew, float theta, float alpha, float *__restrict__ ff) {
    constexpr int NT = ntaps(ORD);
    __shared__ int32_t s_pn[27];
    __shared__ int32_t s_c[512];
    __shared__ unsigned long long s_ok[8];
    __shared__ float s_a[kFillQ][512];  // staged values, then pass-2 outputs
    __shared__ float s_b[kFillQ][512];  // pass-1 outputs
    const int64_t nf = (int64_t)(ef - sf) * 64, nc = (int64_t)(ec - sc) * 64;
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int ox = w & 1, oy = (w >> 1) & 1, oz = w >> 2;
    const float th0 = 1.0f - theta;
    const bool p1 = tid & 1, p2 = (tid >> 3) & 1, p3 = (lane >> 4) & 1;
    float W1[NT], W2[NT], W3[NT];
#pragma unroll
    for (int j = 0; j < NT; ++j) {
        W1[j] = wtap(ORD, p1, j);
        W2[j] = wtap(ORD, p2, j);
        W3[j] = wtap(ORD, p3, j);
    }
    // pass 1: s_b[idx] = sum_k W1[k] s_a[i1 + k], idx = tid + 256 i
    const int i1 = (((tid & 7) >> 1) + 2 + tap0(ORD, p1)) + 8 * ((tid >> 3) & 7) + 64 * (tid >> 6);
    // pass 2: s_a[idx] = sum_k W2[k] s_b[i2 + 8 k]
    const int i2 = (tid & 7) + 8 * ((((tid >> 3) & 7) >> 1) + 2 + tap0(ORD, p2)) + 64 * (tid >> 6);
    // pass 3 (cell t = lane + 32 h of child w): sum_k W3[k] s_a[i3 + 64 (h + k)]
    const int i3 = (4 * ox + (lane & 3)) + 8 * (4 * oy + ((lane >> 2) & 3)) + 64 * (2 * oz + 2 + tap0(ORD, p3));
    const int ngroups = (ef - sf) >> 3;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int32_t b0 = sf + 8 * g, b = b0 + w;
        const bool g0 = masks[64 * (int64_t)b + lane] == VF_GHOST;
        const bool g1 = masks[64 * (int64_t)b + lane + 32] == VF_GHOST;
        const int32_t P = parent[b0];
        const bool ok = P >= sc && P < ec && child[P] == b0;  // uniform over the CTA
        if (!__syncthreads_or(g0 || g1) || !ok) continue;
        if (tid < 27) {
            const int dx = tid % 3 - 1, dy = (tid / 3) % 3 - 1, dz = tid / 9 - 1;
            s_pn[tid] = tid == 13 ? P : __ldg(nbr + 27 * (int64_t)P + slot_of(dx, dy, dz));
        }
        __syncthreads();
#pragma unroll
        for (int i = 0; i < 2; ++i) {
            const int r = tid + 256 * i;
            const int lx = (r & 7) - 2, ly = ((r >> 3) & 7) - 2, lz = (r >> 6) - 2;
            const int32_t Y = s_pn[((lx >> 2) + 1) + 3 * ((ly >> 2) + 1) + 9 * ((lz >> 2) + 1)];
            int32_t c = -1;
            if (Y >= sc && Y < ec) {
                const int tt = (lx & 3) + 4 * (ly & 3) + 16 * (lz & 3);
                if (masks[64 * (int64_t)Y + tt] != VF_SOLID) c = (Y - sc) * 64 + tt;
            }
            s_c[r] = c;
            const uint32_t bal = __ballot_sync(0xffffffffu, c >= 0);
            if (lane == 0) reinterpret_cast<uint32_t *>(s_ok)[w + 8 * i] = bal;
        }
        __syncthreads();
        // order of each owned ghost cell (ORD unless a stencil cell is missing)
        int ord[2], cb[2];  // cb: box index of the first tap at order ord
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            ord[h] = -1;
            cb[h] = 0;
            if (!(h ? g1 : g0)) continue;
            const int t = lane + 32 * h;
            const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
            const int gx = 2 * ox + (I >> 1) + 2, gy = 2 * oy + (J >> 1) + 2, gz = 2 * oz + (K >> 1) + 2;
            const bool qx = I & 1, qy = J & 1, qz = K & 1;
            int o = ORD;
            if (o == 3 && !stencil_ok(s_ok, 3, gx + tap0(3, qx), gy + tap0(3, qy), gz + tap0(3, qz))) o = 1;
            if (o == 1 && !stencil_ok(s_ok, 1, gx + tap0(1, qx), gy + tap0(1, qy), gz + tap0(1, qz))) o = 0;
            if (o == 0 && !stencil_ok(s_ok, 0, gx, gy, gz)) o = -1;  // held
            ord[h] = o;
            if (o >= 0) cb[h] = (gx + tap0(o, qx)) + 8 * (gy + tap0(o, qy)) + 64 * (gz + tap0(o, qz));
        }
        const int64_t xf = (int64_t)(b - sf) * 64;
        const int32_t c0 = s_c[tid], c1 = s_c[tid + 256];
#pragma unroll 1
        for (int q0 = 0; q0 < 27; q0 += kFillQ) {
            float v[kFillQ][2];
#pragma unroll
            for (int j = 0; j < kFillQ; ++j) {
                const int64_t a = (int64_t)(q0 + j) * nc;
                v[j][0] = v[j][1] = 0.0f;
                if (c0 >= 0) v[j][0] = BLEND ? th0 * __ldg(fold + a + c0) + theta * __ldg(fnew + a + c0) : __ldg(fold + a + c0);
                if (c1 >= 0) v[j][1] = BLEND ? th0 * __ldg(fold + a + c1) + theta * __ldg(fnew + a + c1) : __ldg(fold + a + c1);
            }
            __syncthreads();  // the previous round's pass 3 has read s_a
#pragma unroll
            for (int j = 0; j < kFillQ; ++j) {
                s_a[j][tid] = v[j][0];
                s_a[j][tid + 256] = v[j][1];
            }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kFillQ; ++j)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float *p = s_a[j] + i1 + 256 * i;
                    float a = 0.0f;
#pragma unroll
                    for (int k = 0; k < NT; ++k) a += W1[k] * p[k];
                    s_b[j][tid + 256 * i] = a;
                }
            __syncthreads();
#pragma unroll
            for (int j = 0; j < kFillQ; ++j)
#pragma unroll
                for (int i = 0; i < 2; ++i) {
                    const float *p = s_b[j] + i2 + 256 * i;
                    float a = 0.0f;
#pragma unroll
                    for (int k = 0; k < NT; ++k) a += W2[k] * p[8 * k];
                    s_a[j][tid + 256 * i] = a;
                }
            __syncthreads();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (ord[h] != ORD) continue;  // held, or a fallback cell (below)
#pragma unroll 3
                for (int j = 0; j < kFillQ; ++j) {
                    const float *p = s_a[j] + i3 + 64 * h;
                    float acc = 0.0f;
#pragma unroll
                    for (int k = 0; k < NT; ++k) acc += W3[k] * p[64 * k];
                    ff[(int64_t)(q0 + j) * nf + xf + lane + 32 * h] = acc;
                }
            }
        }
        // fallback cells: their own tensor product from the coarse values
        // (rare: a stencil cell outside the level or SOLID)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int o = ord[h];
            if (o < 0 || o == ORD) continue;
            const int t = lane + 32 * h;
            const bool qx = t & 1, qy = (t >> 2) & 1, qz = (t >> 4) & 1;
            const int nt = ntaps(o);
            for (int q = 0; q < 27; ++q) {
                float acc = 0.0f;
                for (int kz = 0; kz < nt; ++kz) {
                    float ay = 0.0f;
                    for (int ky = 0; ky < nt; ++ky) {
                        float ax = 0.0f;
                        for (int kx = 0; kx < nt; ++kx) {
                            const int32_t c = s_c[cb[h] + kx + 8 * ky + 64 * kz];
                            const int64_t a = (int64_t)q * nc + c;
                            const float val = BLEND ? th0 * __ldg(fold + a) + theta * __ldg(fnew + a) : __ldg(fold + a);
                            ax += wtap(o, qx, kx) * val;
                        }
                        ay += wtap(o, qy, ky) * ax;
                    }
                    acc += wtap(o, qz, kz) * ay;
                }
                ff[(int64_t)q * nf + xf + t] = acc;
            }
        }
        if (alpha != 1.0f) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (ord[h] < 0) continue;
                const int64_t x = xf + lane + 32 * h;
                float f[27];
#pragma unroll
                for (int q = 0; q < 27; ++q) f[q] = ff[(int64_t)q * nf + x];
                neq_rescale(f, alpha);
#pragma unroll
                for (int q = 0; q < 27; ++q) ff[(int64_t)q * nf + x] = f[q];
            }
        }
        __syncthreads();  // s_c / s_ok / s_a of this group are done
    }
}

// CTA per sibling group of the fine level (its parent P = parent[first
// child]); thread (t, r) = (tid & 63, tid >> 6) takes coarse cell t of P and
// populations r, r + 4, ...: the 8 children x <= 7 populations are loaded in
// one round (SOLID children contribute +0, summed in child order), the
// moments for the rescale are reduced over the 4 population quarters in a
// fixed order through shared memory.
__global__ void __launch_bounds__(256, 3) k_lbm_restrict(int32_t sc, int32_t ec, int32_t sf, int32_t ef,
                                                         const int32_t *__restrict__ child,
                                                         const int32_t *__restrict__ parent,
                                                         const uint8_t *__restrict__ masks,
                                                         const float *__restrict__ ff, float beta,
                                                         float *__restrict__ fc) {
    __shared__ float s_m[4][4][64];  // [quarter][rho, m_x, m_y, m_z][cell]
    const int64_t nf = (int64_t)(ef - sf) * 64, nc = (int64_t)(ec - sc) * 64;
    const int t = threadIdx.x & 63, r = threadIdx.x >> 6;
    const int ngroups = (ef - sf) >> 3;
    for (int g = blockIdx.x; g < ngroups; g += gridDim.x) {
        const int32_t c0 = sf + 8 * g;
        const int32_t P = __ldg(parent + c0);
        if (P < sc || P >= ec || __ldg(child + P) != c0) continue;  // uniform over the CTA
        const uint8_t m = masks[64 * (int64_t)P + t];
        const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
        const int32_t C = c0 + (I >> 1) + 2 * (J >> 1) + 4 * (K >> 1);
        const int base = 2 * (I & 1) + 8 * (J & 1) + 32 * (K & 1);  // first child cell
        uint32_t use = 0;
        bool ghost = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint8_t mf = masks[64 * (int64_t)C + base + (k & 1) + 4 * ((k >> 1) & 1) + 16 * (k >> 2)];
            ghost |= mf == VF_GHOST;
            if (mf != VF_SOLID) use |= 1u << k;
        }
        const bool act = !(m == VF_SOLID || m == VF_INTERFACE || m == VF_GHOST || ghost || !use);
        float f[7];
        const float *src = ff + (int64_t)(C - sf) * 64 + base;
        if (act) {
            const float inv = 1.0f / (float)__popc(use);
#pragma unroll
            for (int j = 0; j < 7; ++j) f[j] = 0.0f;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int o = (k & 1) + 4 * ((k >> 1) & 1) + 16 * (k >> 2);
                const bool u = (use >> k) & 1u;
#pragma unroll
                for (int j = 0; j < 7; ++j) {
                    const int q = r + 4 * j;
                    if (q < 27) {
                        const float v = __ldg(src + (int64_t)q * nf + o);
                        f[j] += u ? v : 0.0f;
                    }
                }
            }
#pragma unroll
            for (int j = 0; j < 7; ++j) f[j] *= inv;
        }
        if (beta != 1.0f) {  // uniform
            float m4[4] = {0.f, 0.f, 0.f, 0.f};
            if (act)
#pragma unroll
                for (int j = 0; j < 7; ++j) {
                    const int q = r + 4 * j;
                    if (q < 27) {
                        m4[0] += f[j];
                        m4[1] += f[j] * c27(q, 0);
                        m4[2] += f[j] * c27(q, 1);
                        m4[3] += f[j] * c27(q, 2);
                    }
                }
#pragma unroll
            for (int c = 0; c < 4; ++c) s_m[r][c][t] = m4[c];
            __syncthreads();
            if (act) {
                float M[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) M[c] = (s_m[0][c][t] + s_m[1][c][t]) + (s_m[2][c][t] + s_m[3][c][t]);
                if (M[0] > 0.0f) {
                    const float ir = 1.0f / M[0];
                    const float u0 = M[1] * ir, u1 = M[2] * ir, u2 = M[3] * ir;
                    const float uu = 1.5f * (u0 * u0 + u1 * u1 + u2 * u2);
#pragma unroll
                    for (int j = 0; j < 7; ++j) {
                        const int q = r + 4 * j;
                        if (q < 27) {
                            const float cu = c27(q, 0) * u0 + c27(q, 1) * u1 + c27(q, 2) * u2;
                            const float feq = c_lw[q] * M[0] * (1.0f + 3.0f * cu + 4.5f * cu * cu - uu);
                            f[j] = feq + beta * (f[j] - feq);
                        }
                    }
                }
            }
            __syncthreads();
        }
        if (act) {
            const int64_t x = (int64_t)(P - sc) * 64 + t;
#pragma unroll
            for (int j = 0; j < 7; ++j) {
                const int q = r + 4 * j;
                if (q < 27) fc[(int64_t)q * nc + x] = f[j];
            }
        }
    }
}

}  // namespace vf

using namespace vf;

extern "C" {

int vf_lbm_init(const vf_grid *g, int32_t s, int32_t e, double rho, const double *u, float *f,
                void *stream) {
    if (!g || !f || !u || s < 0 || e < s || e > g->capacity)
        return set_error(VF_EARG, "vf_lbm_init: bad argument");
    if (e == s) return VF_OK;
    int64_t grid = ((int64_t)(e - s) * 64 + 255) / 256;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_lbm_init<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(s, e, g->d_masks, (float)rho, (float)u[0],
                                                             (float)u[1], (float)u[2], f);
    return check_launch("k_lbm_init");
}

int vf_lbm_parents(const vf_grid *g, int32_t n_blocks, int32_t *d_parent, void *stream) {
    if (!g || !d_parent || n_blocks < 0 || n_blocks > g->capacity)
        return set_error(VF_EARG, "vf_lbm_parents: bad argument");
    cudaStream_t st = (cudaStream_t)stream;
    cudaMemsetAsync(d_parent, 0xff, sizeof(int32_t) * (size_t)n_blocks, st);
    if (n_blocks == 0) return VF_OK;
    k_lbm_parents<<<max_ctas(4), 256, 0, st>>>(n_blocks, g->d_child, d_parent);
    return check_launch("k_lbm_parents");
}

int vf_lbm_fill_ghosts(const vf_grid *g, int32_t sf, int32_t ef, int32_t sc, int32_t ec, const int32_t *d_parent,
                       const float *fc_old, const float *fc_new, double theta, double alpha, int order, float *ff,
                       void *stream) {
    if (!g || !d_parent || !fc_old || !ff || sf < 0 || ef < sf || ef > g->capacity || sc < 0 || ec < sc ||
        ec > g->capacity || !(theta >= 0.0 && theta <= 1.0) || (theta > 0.0 && !fc_new) ||
        !(order == 0 || order == 1 || order == 3))
        return set_error(VF_EARG, "vf_lbm_fill_ghosts: bad argument");
    if ((ef - sf) % 8) return set_error(VF_EARG, "vf_lbm_fill_ghosts: the fine range must be whole sibling groups (a level >= 1)");
    if (ef == sf || ec == sc) return VF_OK;
    int64_t grid = (ef - sf) / 8;
    if (grid > max_ctas(VF_FILL_MINB)) grid = max_ctas(VF_FILL_MINB);
    cudaStream_t st = (cudaStream_t)stream;
    const float *fn = fc_new ? fc_new : fc_old;
#define VF_FILL_LAUNCH(O, B)                                                                                   \
    k_lbm_fill_ghosts<O, B><<<(int)grid, 256, 0, st>>>(sf, ef, sc, ec, g->d_nbr, g->d_child, g->d_masks, d_parent, \
                                                       fc_old, fn, (float)theta, (float)alpha, ff)
    const bool blend = theta != 0.0;
    if (order == 3) { if (blend) VF_FILL_LAUNCH(3, true); else VF_FILL_LAUNCH(3, false); }
    else if (order == 1) { if (blend) VF_FILL_LAUNCH(1, true); else VF_FILL_LAUNCH(1, false); }
    else { if (blend) VF_FILL_LAUNCH(0, true); else VF_FILL_LAUNCH(0, false); }
#undef VF_FILL_LAUNCH
    return check_launch("k_lbm_fill_ghosts");
}

int vf_lbm_restrict(const vf_grid *g, int32_t sc, int32_t ec, int32_t sf, int32_t ef, const int32_t *d_parent,
                    const float *ff, double beta, float *fc, void *stream) {
    if (!g || !d_parent || !ff || !fc || sf < 0 || ef < sf || ef > g->capacity || sc < 0 || ec < sc ||
        ec > g->capacity)
        return set_error(VF_EARG, "vf_lbm_restrict: bad argument");
    if ((ef - sf) % 8) return set_error(VF_EARG, "vf_lbm_restrict: the fine range must be whole sibling groups (a level >= 1)");
    if (ef == sf || ec == sc) return VF_OK;
    int64_t grid = (ef - sf) / 8;
    if (grid > max_ctas(3)) grid = max_ctas(3);
    k_lbm_restrict<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(sc, ec, sf, ef, g->d_child, d_parent, g->d_masks, ff,
                                                                 (float)beta, fc);
    return check_launch("k_lbm_restrict");
}

int vf_lbm_step(const vf_config *cfg, const vf_grid *g, int level, int32_t s, int32_t e,
                const int32_t *cmap, const float *lengths, const float *fin, float *fout,
                const vf_flow *flow, double *d_force, int32_t *d_scratch, void *stream) {
    if (!cfg || !g || !fin || !fout || !flow || !d_scratch || fin == fout || s < 0 || e < s ||
        e > g->capacity || level < 0 || level >= VF_MAX_LEVELS || !(flow->tau > 0.5) ||
        (flow->ibb && (!cmap || !lengths)))
        return set_error(VF_EARG, "vf_lbm_step: bad argument (tau must exceed 1/2)");
    if (e == s) return VF_OK;
    cudaStream_t st = (cudaStream_t)stream;
    const int cells_x = 4 * (cfg->nb[0] << level);
    int32_t *n_list = d_scratch, *list = d_scratch + 1;
    // per-block force partials after the special-block list, 8-byte aligned
    double *part = d_force ? reinterpret_cast<double *>(d_scratch + ((e - s + 2 + 1) & ~1)) : nullptr;
#ifndef VF_LBM_FUSED
    cudaMemsetAsync(n_list, 0, sizeof(int32_t), st);
    kt_point("memset:lbm_list");
#endif
    if (part) {
        cudaMemsetAsync(part, 0, sizeof(double) * 3 * (size_t)(e - s), st);
        kt_point("memset:lbm_part");
    }
    int rc;
#ifndef VF_LBM_FUSED
    int64_t grid = ((int64_t)(e - s) + kLbmWarps - 1) / kLbmWarps;
    if (grid > max_ctas(VF_LBM_MINB)) grid = max_ctas(VF_LBM_MINB);
    k_lbm_bulk<<<(int)grid, kLbmWarps * 32, 0, st>>>(s, e, cells_x, flow->open_x, g->d_coords, g->d_nbr, g->d_masks,
                                                     g->d_solid64, fin, fout, 1.0f / (float)flow->tau, list, n_list);
    rc = check_launch("k_lbm_bulk");
    if (rc) return rc;
    int64_t grid2 = ((int64_t)(e - s) + kLbmWarps - 1) / kLbmWarps;
    if (grid2 > max_ctas(VF_LBM_SPECIAL_MINB)) grid2 = max_ctas(VF_LBM_SPECIAL_MINB);
    k_lbm_special<<<(int)grid2, kLbmWarps * 32, 0, st>>>(s, e, cells_x, g->d_coords, g->d_nbr, g->d_masks,
                                                         g->d_solid64, cmap, lengths, fin, fout, *flow, list,
                                                         n_list, part);
    rc = check_launch("k_lbm_special");
#else
    (void)list;
    int64_t grid = ((int64_t)(e - s) + kLbmWarps - 1) / kLbmWarps;
    if (grid > max_ctas(VF_LBM_FUSED_MINB)) grid = max_ctas(VF_LBM_FUSED_MINB);
    k_lbm_cells<<<(int)grid, kLbmWarps * 32, 0, st>>>(s, e, cells_x, g->d_coords, g->d_nbr, g->d_masks,
                                                      g->d_solid64, cmap, lengths, fin, fout, *flow, part);
    rc = check_launch("k_lbm_cells");
#endif
    if (rc || !d_force) return rc;
    k_lbm_force_reduce<<<1, 1024, 0, st>>>(e - s, part, d_force);
    return check_launch("k_lbm_force_reduce");
}

}  // extern "C"
