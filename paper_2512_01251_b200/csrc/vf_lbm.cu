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
// momentum exchange of the wall links is reduced per warp and accumulated in
// FP64.  Bytes per fluid cell: 27 x 4 read + 27 x 4 written (+ 64 B masks
// per block): HBM-bound.
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

// Warp per block (two 32-cell halves): the block's 27 neighbour ids, their
// solid64 words (finalize; bit t = cell t SOLID) and the block's x index are
// staged in per-warp shared memory, indexed by direction code
// (dx+1) + 3(dy+1) + 9(dz+1), so a pulled population costs one shared-memory
// lookup and one global load that is coalesced within a block.  Domain faces
// (lateral SBB, inlet velocity bounce-back, outlet anti-bounce-back) are
// resolved inline.  WALLS = false is the bulk pass over every block: a wall
// link gets a provisional SBB value and its block is appended to the wall
// list; WALLS = true re-runs the listed blocks with the wall rule (SBB or
// Bouzidi linear IBB with q_w from the LUT) and the momentum exchange, and
// overwrites those cells (same f_in, so the two passes commute).
constexpr int kLbmWarps = 8;
#ifndef VF_LBM_MINB
#define VF_LBM_MINB 3
#endif

template <bool WALLS>
__global__ void __launch_bounds__(kLbmWarps * 32, VF_LBM_MINB)
    k_lbm_cells(int32_t s, int32_t e, int cells_x, const int32_t *__restrict__ coords,
                const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
                const uint64_t *__restrict__ solid64, const int32_t *__restrict__ cmap,
                const float *__restrict__ lengths, const float *__restrict__ fin,
                float *__restrict__ fout, vf_flow flow, int32_t *__restrict__ wall_list,
                int32_t *__restrict__ n_wall, double *__restrict__ part) {
    __shared__ int32_t s_nb[kLbmWarps][27];
    __shared__ unsigned long long s_sol[kLbmWarps][27];
    const int64_t n = (int64_t)(e - s) * 64;
    const int nitems = WALLS ? *n_wall : e - s;
    const float omega = 1.0f / (float)flow.tau;
    const float uin[3] = {(float)flow.u_in[0], (float)flow.u_in[1], (float)flow.u_in[2]};
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int it = blockIdx.x * kLbmWarps + w; it < nitems; it += gridDim.x * kLbmWarps) {
        float Fx = 0.f, Fy = 0.f, Fz = 0.f;  // this block's wall momentum exchange
        const int lb = WALLS ? wall_list[it] : it;
        const int32_t b = s + lb;
        __syncwarp();
        if (lane < 27) {
            const int dx = lane % 3 - 1, dy = (lane / 3) % 3 - 1, dz = lane / 9 - 1;
            const int32_t v = (lane == 13) ? b : __ldg(nbr + 27 * (int64_t)b + slot_of(dx, dy, dz));
            s_nb[w][lane] = v;
            s_sol[w][lane] = (v >= s && v < e)
                                 ? __ldg(reinterpret_cast<const unsigned long long *>(solid64) + v)
                                 : ~0ull;
        }
        const int bx = __ldg(coords + 4 * (int64_t)b);
        const int32_t slot = (WALLS && flow.ibb) ? cmap[b] : -1;
        __syncwarp();
        bool wall_blk = false;
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
            const int64_t x = (int64_t)lb * 64 + t;
            const uint8_t m = masks[64 * (int64_t)b + t];
            if (m == VF_SOLID || m == VF_GHOST) {
                if (!WALLS) {
#pragma unroll
                    for (int q = 0; q < 27; ++q) fout[q * n + x] = fin[q * n + x];
                }
                continue;
            }
            // outlet cells (x = l_x face): velocity of x for the anti-bounce-back
            float v0 = 0.f, v1 = 0.f, v2 = 0.f;
            if (flow.open_x && 4 * bx + I == cells_x - 1) {
                float rx = 0.f;
#pragma unroll
                for (int k = 0; k < 27; ++k) {
                    const float v = fin[k * n + x];
                    rx += v;
                    v0 += v * c27(k, 0);
                    v1 += v * c27(k, 1);
                    v2 += v * c27(k, 2);
                }
                v0 /= rx; v1 /= rx; v2 /= rx;
            }
            float f[27];
            bool wall = false;
#pragma unroll
            for (int o = 0; o < 27; ++o) {
                const int X = I - c27(o, 0), Y = J - c27(o, 1), Z = K - c27(o, 2);
                const int code = ((X >> 2) + 1) + 3 * ((Y >> 2) + 1) + 9 * ((Z >> 2) + 1);
                const int ty = (X & 3) + 4 * (Y & 3) + 16 * (Z & 3);
                const int32_t y = s_nb[w][code];
                if (!((s_sol[w][code] >> ty) & 1ull)) {  // a level cell that is not SOLID
                    f[o] = fin[o * n + (int64_t)(y - s) * 64 + ty];
                    continue;
                }
                const int q = o == 0 ? 0 : ((o & 1) ? o + 1 : o - 1);
                const float fq = fin[q * n + x];
                float v = fq;  // SBB: lateral faces, SBB walls (provisional in the bulk pass)
                if (y == VF_NB_OUTSIDE) {
                    const int gx = 4 * bx + X;
                    if (flow.open_x && gx < 0) {  // inlet: velocity bounce-back, rho_w = 1
                        v -= 6.0f * c_lw[q] * (c27(q, 0) * uin[0] + c27(q, 1) * uin[1] + c27(q, 2) * uin[2]);
                    } else if (flow.open_x && gx >= cells_x) {  // outlet: anti-bounce-back, rho_w = 1
                        const float cq = c27(q, 0) * v0 + c27(q, 1) * v1 + c27(q, 2) * v2;
                        v = -fq + 2.0f * c_lw[q] * (1.0f + 4.5f * cq * cq - 1.5f * (v0 * v0 + v1 * v1 + v2 * v2));
                    }
                } else {  // wall link x -> y (SOLID cell, or a missing block next to ghosts)
                    wall = true;
                    if (WALLS) {
                        const float qw = slot >= 0 ? lengths[((int64_t)slot * 27 + q) * 64 + t] : -1.0f;
                        if (qw > 0.0f && qw < 0.5f) {
                            // second node behind x: x + c_o = x - c_q
                            const int X2 = I + c27(o, 0), Y2 = J + c27(o, 1), Z2 = K + c27(o, 2);
                            const int code2 = ((X2 >> 2) + 1) + 3 * ((Y2 >> 2) + 1) + 9 * ((Z2 >> 2) + 1);
                            const int tz = (X2 & 3) + 4 * (Y2 & 3) + 16 * (Z2 & 3);
                            if (!((s_sol[w][code2] >> tz) & 1ull))
                                v = 2.0f * qw * fq + (1.0f - 2.0f * qw) *
                                                         fin[q * n + (int64_t)(s_nb[w][code2] - s) * 64 + tz];
                        } else if (qw >= 0.5f) {
                            v = fq / (2.0f * qw) + (2.0f * qw - 1.0f) / (2.0f * qw) * fin[o * n + x];
                        }
                        Fx += (fq + v) * c27(q, 0);
                        Fy += (fq + v) * c27(q, 1);
                        Fz += (fq + v) * c27(q, 2);
                    }
                }
                f[o] = v;
            }
            wall_blk |= wall;
            if (WALLS && !wall) continue;  // the bulk pass's value is exact
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
        if (!WALLS && __any_sync(0xffffffffu, wall_blk) && lane == 0)
            wall_list[atomicAdd(n_wall, 1)] = lb;
        if (WALLS && part) {
            // per-block partial: a fixed lane tree, stored at the block's
            // local id -- independent of which warp took the block
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
    }
}

// d_force += sum over the level's blocks of the per-block partials, in block
// order with a fixed reduction tree (identical force series
// across runs; the wall-block list order depends on atomics)
__global__ void __launch_bounds__(256) k_lbm_force_reduce(int32_t nb, const double *__restrict__ part,
                                                          double *__restrict__ d_force) {
    __shared__ double s_r[3][256];
    double a[3] = {0.0, 0.0, 0.0};
    for (int32_t b = threadIdx.x; b < nb; b += blockDim.x)
#pragma unroll
        for (int c = 0; c < 3; ++c) a[c] += part[3 * (int64_t)b + c];
#pragma unroll
    for (int c = 0; c < 3; ++c) s_r[c][threadIdx.x] = a[c];
    __syncthreads();
    for (int o = 128; o > 0; o >>= 1) {
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

// Warp per fine block: the block's 64 cells lie in 2x2x2 coarse cells, so
// every stencil (cubic: +-2 coarse cells) lies in the 6x6x6 coarse cells
// around them.  Their level-local ids (or -1: outside the level / SOLID) are
// staged once; then per population the 216 time-blended coarse values are
// staged and each lane interpolates its (<= 2) ghost cells separably
// (x, then y, then z).  The interpolated populations go to ff and are then
// rescaled in place by their owning lane.
constexpr int kFillWarps = 8;
#ifndef VF_FILL_Q
#define VF_FILL_Q 3
#endif
#ifndef VF_FILL_MINB
#define VF_FILL_MINB 2  // <= 128 registers: 2 CTAs per SM (measured best; 1 -> 188 registers, 3 -> 80)
#endif
constexpr int kFillQ = VF_FILL_Q;  // populations staged per load round (27 = 9 x 3)

__device__ __forceinline__ float axis_w(int ord, int k) {
    return ord == 3 ? c_w3[k] : (ord == 1 ? (k ? 0.25f : 0.75f) : 1.0f);
}

__global__ void __launch_bounds__(kFillWarps * 32, VF_FILL_MINB)
    k_lbm_fill_ghosts(int32_t sf, int32_t ef, int32_t sc, int32_t ec, const int32_t *__restrict__ coords,
                      const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
                      const int32_t *__restrict__ parent, const float *__restrict__ fold,
                      const float *__restrict__ fnew, float theta, float alpha, int order,
                      float *__restrict__ ff) {
    __shared__ int32_t s_c[kFillWarps][216];
    __shared__ float s_vq[kFillWarps][kFillQ][216];  // kFillQ populations staged per round
    __shared__ float s_t1[kFillWarps][144], s_t2[kFillWarps][96];
    const int64_t nf = (int64_t)(ef - sf) * 64, nc = (int64_t)(ec - sc) * 64;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const float th0 = 1.0f - theta;
    for (int32_t b = sf + blockIdx.x * kFillWarps + w; b < ef; b += gridDim.x * kFillWarps) {
        const bool g0 = masks[64 * (int64_t)b + lane] == VF_GHOST;
        const bool g1 = masks[64 * (int64_t)b + lane + 32] == VF_GHOST;
        if (!__any_sync(0xffffffffu, g0 || g1)) continue;
        const int32_t P = parent[b];
        if (P < sc || P >= ec) continue;  // warp-uniform
        int R0[3];  // the fine block's first coarse cell, relative to P
#pragma unroll
        for (int d = 0; d < 3; ++d) R0[d] = 2 * coords[4 * (int64_t)b + d] - 4 * coords[4 * (int64_t)P + d];
        // staged coarse cells: local (R0 - 2 + rx, ...), r = rx + 6 ry + 36 rz
        for (int r = lane; r < 216; r += 32) {
            const int lx = R0[0] - 2 + r % 6, ly = R0[1] - 2 + (r / 6) % 6, lz = R0[2] - 2 + r / 36;
            const int ox = lx < 0 ? -1 : (lx > 3 ? 1 : 0), oy = ly < 0 ? -1 : (ly > 3 ? 1 : 0),
                      oz = lz < 0 ? -1 : (lz > 3 ? 1 : 0);
            const int32_t Y = (ox | oy | oz) ? __ldg(nbr + 27 * (int64_t)P + slot_of(ox, oy, oz)) : P;
            int32_t c = -1;
            if (Y >= sc && Y < ec) {
                const int tt = (lx & 3) + 4 * (ly & 3) + 16 * (lz & 3);
                if (masks[64 * (int64_t)Y + tt] != VF_SOLID) c = (Y - sc) * 64 + tt;
            }
            s_c[w][r] = c;
        }
        __syncwarp();
        // per owned ghost cell: staged base index, axis steps, order
        int base[2], st[2][3], ord[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = lane + 32 * h;
            ord[h] = -1;
            base[h] = 0;
            st[h][0] = st[h][1] = st[h][2] = 0;
            if (!(h ? g1 : g0)) continue;
            const int I[3] = {t & 3, (t >> 2) & 3, t >> 4};
            int bx[3];
#pragma unroll
            for (int d = 0; d < 3; ++d) {
                bx[d] = (I[d] >> 1) + 2;  // G relative to the staged box
                st[h][d] = (I[d] & 1) ? 1 : -1;  // fine cell 4c + I: odd iff I odd
            }
            const int sx = st[h][0], sy = 6 * st[h][1], sz = 36 * st[h][2];
            base[h] = bx[0] + 6 * bx[1] + 36 * bx[2];
            int o = order >= 3 ? 3 : (order >= 1 ? 1 : 0);
            if (o == 3) {
                for (int k = 0; k < 64 && o == 3; ++k)
                    if (s_c[w][base[h] + sx * ((k & 3) - 1) + sy * (((k >> 2) & 3) - 1) + sz * ((k >> 4) - 1)] < 0) o = 1;
            }
            if (o == 1) {
                for (int k = 0; k < 8 && o == 1; ++k)
                    if (s_c[w][base[h] + sx * (k & 1) + sy * ((k >> 1) & 1) + sz * (k >> 2)] < 0) o = 0;
            }
            if (o == 0 && s_c[w][base[h]] < 0) o = -1;  // held
            ord[h] = o;
            st[h][1] *= 6;
            st[h][2] *= 36;
        }
#pragma unroll 1
        for (int q0 = 0; q0 < 27; q0 += kFillQ) {
          __syncwarp();
          // kFillQ x 7 independent loads per lane in flight (216 = 6 x 32 + 24)
          {
            float v[kFillQ][7];
#pragma unroll
            for (int j = 0; j < kFillQ; ++j)
#pragma unroll
                for (int i = 0; i < 7; ++i) {
                    const int r = lane + 32 * i;
                    const int32_t c = r < 216 ? s_c[w][r] : -1;
                    v[j][i] = 0.0f;
                    if (c >= 0) {
                        const int64_t a = (int64_t)(q0 + j) * nc + c;
                        v[j][i] = theta == 0.0f ? __ldg(fold + a) : th0 * __ldg(fold + a) + theta * __ldg(fnew + a);
                    }
                }
#pragma unroll
            for (int j = 0; j < kFillQ; ++j)
#pragma unroll
                for (int i = 0; i < 7; ++i)
                    if (lane + 32 * i < 216) s_vq[w][j][lane + 32 * i] = v[j][i];
          }
          __syncwarp();
#pragma unroll 1
          for (int j = 0; j < kFillQ; ++j) {
            const int q = q0 + j;
            const float *sv = s_vq[w][j];
            __syncwarp();
            // separable passes at the requested order for the whole block
            // (x: 4 x 6 x 6, y: 4 x 4 x 6, z: 4 x 4 x 4); same association as
            // the per-cell sum below, so a cell's value does not depend on
            // which path computed it
            const int og = order >= 3 ? 3 : (order >= 1 ? 1 : 0);
            const int ng = og == 3 ? 4 : (og == 1 ? 2 : 1), kg = og == 3 ? -1 : 0;
            for (int e = lane; e < 144; e += 32) {  // (fx, ry, rz)
                const int fx = e & 3, ry = (e >> 2) % 6, rz = (e >> 2) / 6;
                const int G = (fx >> 1) + 2, sg = (fx & 1) ? 1 : -1;
                float a = 0.0f;
                for (int k = 0; k < ng; ++k) a += axis_w(og, k) * sv[G + sg * (k + kg) + 6 * ry + 36 * rz];
                s_t1[w][e] = a;
            }
            __syncwarp();
            for (int e = lane; e < 96; e += 32) {  // (fx, fy, rz)
                const int fx = e & 3, fy = (e >> 2) & 3, rz = e >> 4;
                const int G = (fy >> 1) + 2, sg = (fy & 1) ? 1 : -1;
                float a = 0.0f;
                for (int k = 0; k < ng; ++k) a += axis_w(og, k) * s_t1[w][fx + 4 * (G + sg * (k + kg)) + 24 * rz];
                s_t2[w][e] = a;
            }
            __syncwarp();
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int o = ord[h];
                if (o < 0) continue;
                const int t = lane + 32 * h;
                float acc = 0.0f;
                if (o == og) {
                    const int fz = t >> 4, G = (fz >> 1) + 2, sg = (fz & 1) ? 1 : -1;
                    for (int k = 0; k < ng; ++k) acc += axis_w(og, k) * s_t2[w][(t & 15) + 16 * (G + sg * (k + kg))];
                } else {  // fallback order of this cell (a stencil cell is missing)
                    const int n = o == 3 ? 4 : (o == 1 ? 2 : 1), k0 = o == 3 ? -1 : 0;
                    for (int kz = 0; kz < n; ++kz) {
                        float ay = 0.0f;
                        for (int ky = 0; ky < n; ++ky) {
                            float ax = 0.0f;
                            const int row = base[h] + st[h][1] * (ky + k0) + st[h][2] * (kz + k0);
                            for (int kx = 0; kx < n; ++kx) ax += axis_w(o, kx) * sv[row + st[h][0] * (kx + k0)];
                            ay += axis_w(o, ky) * ax;
                        }
                        acc += axis_w(o, kz) * ay;
                    }
                }
                ff[(int64_t)q * nf + (int64_t)(b - sf) * 64 + t] = acc;
            }
          }
        }
        if (alpha != 1.0f) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (ord[h] < 0) continue;
                const int64_t x = (int64_t)(b - sf) * 64 + lane + 32 * h;
                float f[27];
#pragma unroll
                for (int q = 0; q < 27; ++q) f[q] = ff[(int64_t)q * nf + x];
                neq_rescale(f, alpha);
#pragma unroll
                for (int q = 0; q < 27; ++q) ff[(int64_t)q * nf + x] = f[q];
            }
        }
    }
}

__global__ void k_lbm_restrict(int32_t sc, int32_t ec, int32_t sf, int32_t ef, const int32_t *__restrict__ child,
                               const uint8_t *__restrict__ masks, const float *__restrict__ ff, float beta,
                               float *__restrict__ fc) {
    const int64_t nf = (int64_t)(ef - sf) * 64, nc = (int64_t)(ec - sc) * 64;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < nc; x += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = sc + (int32_t)(x >> 6);
        const int t = (int)(x & 63);
        const int32_t c0 = child[b];
        if (c0 < 0) continue;
        const uint8_t m = masks[64 * (int64_t)b + t];
        if (m == VF_SOLID || m == VF_INTERFACE || m == VF_GHOST) continue;
        const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
        const int32_t C = c0 + (I >> 1) + 2 * (J >> 1) + 4 * (K >> 1);
        if (C < sf || C >= ef) continue;
        int fine[8], n = 0;
        bool ghost = false;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int tt = (2 * (I & 1) + (k & 1)) + 4 * (2 * (J & 1) + ((k >> 1) & 1)) + 16 * (2 * (K & 1) + (k >> 2));
            const uint8_t mf = masks[64 * (int64_t)C + tt];
            ghost |= mf == VF_GHOST;
            if (mf != VF_SOLID) fine[n++] = (C - sf) * 64 + tt;
        }
        if (ghost || n == 0) continue;
        const float inv = 1.0f / (float)n;
        float f[27];
#pragma unroll
        for (int q = 0; q < 27; ++q) {
            float acc = 0.0f;
            for (int k = 0; k < n; ++k) acc += ff[(int64_t)q * nf + fine[k]];
            f[q] = acc * inv;
        }
        neq_rescale(f, beta);
#pragma unroll
        for (int q = 0; q < 27; ++q) fc[(int64_t)q * nc + x] = f[q];
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
    if (ef == sf || ec == sc) return VF_OK;
    int64_t grid = ((int64_t)(ef - sf) + kFillWarps - 1) / kFillWarps;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_lbm_fill_ghosts<<<(int)grid, kFillWarps * 32, 0, (cudaStream_t)stream>>>(
        sf, ef, sc, ec, g->d_coords, g->d_nbr, g->d_masks, d_parent, fc_old, fc_new ? fc_new : fc_old,
        (float)theta, (float)alpha, order, ff);
    return check_launch("k_lbm_fill_ghosts");
}

int vf_lbm_restrict(const vf_grid *g, int32_t sc, int32_t ec, int32_t sf, int32_t ef, const float *ff, double beta,
                    float *fc, void *stream) {
    if (!g || !ff || !fc || sf < 0 || ef < sf || ef > g->capacity || sc < 0 || ec < sc || ec > g->capacity)
        return set_error(VF_EARG, "vf_lbm_restrict: bad argument");
    if (ef == sf || ec == sc) return VF_OK;
    int64_t grid = ((int64_t)(ec - sc) * 64 + 255) / 256;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_lbm_restrict<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(sc, ec, sf, ef, g->d_child, g->d_masks, ff,
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
    int32_t *n_wall = d_scratch, *wall_list = d_scratch + 1;
    // per-block force partials after the wall list, 8-byte aligned
    double *part = d_force ? reinterpret_cast<double *>(d_scratch + ((e - s + 2 + 1) & ~1)) : nullptr;
    cudaMemsetAsync(n_wall, 0, sizeof(int32_t), st);
    if (part) cudaMemsetAsync(part, 0, sizeof(double) * 3 * (size_t)(e - s), st);
    int64_t grid = ((int64_t)(e - s) + kLbmWarps - 1) / kLbmWarps;
    if (grid > max_ctas(VF_LBM_MINB)) grid = max_ctas(VF_LBM_MINB);
    k_lbm_cells<false><<<(int)grid, kLbmWarps * 32, 0, st>>>(
        s, e, cells_x, g->d_coords, g->d_nbr, g->d_masks, g->d_solid64, cmap, lengths, fin, fout, *flow,
        wall_list, n_wall, nullptr);
    int rc = check_launch("k_lbm_cells");
    if (rc) return rc;
    k_lbm_cells<true><<<max_ctas(2), kLbmWarps * 32, 0, st>>>(
        s, e, cells_x, g->d_coords, g->d_nbr, g->d_masks, g->d_solid64, cmap, lengths, fin, fout, *flow,
        wall_list, n_wall, part);
    int rc2 = check_launch("k_lbm_walls");
    if (rc2 || !d_force) return rc2;
    k_lbm_force_reduce<<<1, 256, 0, st>>>(e - s, part, d_force);
    return check_launch("k_lbm_force_reduce");
}

}  // extern "C"
