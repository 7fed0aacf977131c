// vf_lbm.cu -- the LUT consumer: one D3Q27 BGK collide/stream step of one
// grid level with SBB / interpolated bounce-back (Bouzidi linear) wall links
// read from the cut-link LUT (SPEC.md:398-411 collide_stream_level,
// SPEC.md:392-397 equilibrium, SPEC.md:436-440 accumulate_forces;
// SURVEY.md §8(f) next #1).  Oracle: oracle/lbm_oracle.c (same rules, FP64).
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

// wall links (SOLID y: SBB / Bouzidi linear IBB with the LUT q_w) and domain
// faces (inlet velocity bounce-back, outlet anti-bounce-back, lateral SBB) of
// one cell; f[o] is NaN for the populations to resolve
__device__ __noinline__ void resolve_links(float *f, int64_t x, int64_t n, int32_t b, int t,
                                           int32_t s, int32_t e, int cells_x,
                                           const int32_t *__restrict__ coords,
                                           const int32_t *__restrict__ nbr,
                                           const uint8_t *__restrict__ masks,
                                           const int32_t *__restrict__ cmap,
                                           const float *__restrict__ lengths,
                                           const float *__restrict__ fin, const vf_flow &flow,
                                           const float *uin, float &Fx, float &Fy, float &Fz) {
    const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
    // moments of x (outlet anti-bounce-back)
    float rx = 0.f, u0 = 0.f, u1 = 0.f, u2 = 0.f;
    for (int q = 0; q < 27; ++q) {
        const float v = fin[q * n + x];
        rx += v;
        u0 += v * c27(q, 0);
        u1 += v * c27(q, 1);
        u2 += v * c27(q, 2);
    }
    const float ux[3] = {u0 / rx, u1 / rx, u2 / rx};
    const int32_t slot = flow.ibb ? cmap[b] : -1;
    for (int o = 0; o < 27; ++o) {
        if (!isnan(f[o])) continue;
        const int q = lopp(o);
        int ty;
        const int32_t y = cell_at(nbr, b, I, J, K, -c27(o, 0), -c27(o, 1), -c27(o, 2), ty);
        const float fq = fin[q * n + x];
        const float cqx = (float)c27(q, 0), cqy = (float)c27(q, 1), cqz = (float)c27(q, 2);
        if (y == VF_NB_OUTSIDE) {  // domain face
            const int gx = 4 * coords[4 * (int64_t)b] + I - c27(o, 0);
            if (!flow.open_x) {
                f[o] = fq;  // closed box: SBB on every face
            } else if (gx < 0) {  // inlet: velocity bounce-back, rho_w = 1
                f[o] = fq - 6.0f * c_lw[q] * (cqx * uin[0] + cqy * uin[1] + cqz * uin[2]);
            } else if (gx >= cells_x) {  // outlet: anti-bounce-back, rho_w = 1
                const float cq = cqx * ux[0] + cqy * ux[1] + cqz * ux[2];
                const float uu = ux[0] * ux[0] + ux[1] * ux[1] + ux[2] * ux[2];
                f[o] = -fq + 2.0f * c_lw[q] * (1.0f + 4.5f * cq * cq - 1.5f * uu);
            } else {
                f[o] = fq;  // lateral faces: SBB
            }
            continue;
        }
        // wall link x -> y (SOLID cell): Bouzidi linear with the LUT q_w
        const float qw = slot >= 0 ? lengths[((int64_t)slot * 27 + q) * 64 + t] : -1.0f;
        float fo;
        if (!(qw > 0.0f)) {
            fo = fq;  // SBB
        } else if (qw < 0.5f) {
            int tz;
            const int32_t z = cell_at(nbr, b, I, J, K, c27(o, 0), c27(o, 1), c27(o, 2), tz);
            if (z >= s && z < e && masks[64 * (int64_t)z + tz] != VF_SOLID)
                fo = 2.0f * qw * fq + (1.0f - 2.0f * qw) * fin[q * n + (int64_t)(z - s) * 64 + tz];
            else
                fo = fq;
        } else {
            fo = fq / (2.0f * qw) + (2.0f * qw - 1.0f) / (2.0f * qw) * fin[o * n + x];
        }
        f[o] = fo;
        Fx += (fq + fo) * cqx;
        Fy += (fq + fo) * cqy;
        Fz += (fq + fo) * cqz;
    }
}

__global__ void __launch_bounds__(256, 3)
    k_lbm_step(int32_t s, int32_t e, int cells_x, const int32_t *__restrict__ coords,
               const int32_t *__restrict__ nbr, const uint8_t *__restrict__ masks,
               const int32_t *__restrict__ cmap, const float *__restrict__ lengths,
               const float *__restrict__ fin, float *__restrict__ fout, vf_flow flow,
               double *__restrict__ d_force) {
    const int64_t n = (int64_t)(e - s) * 64;
    const float omega = 1.0f / (float)flow.tau;
    const float uin[3] = {(float)flow.u_in[0], (float)flow.u_in[1], (float)flow.u_in[2]};
    float Fx = 0.f, Fy = 0.f, Fz = 0.f;
    for (int64_t x = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; x < n;
         x += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = s + (int32_t)(x >> 6);
        const int t = (int)(x & 63);
        const uint8_t m = masks[64 * (int64_t)b + t];
        if (m == VF_SOLID || m == VF_GHOST) {
#pragma unroll
            for (int q = 0; q < 27; ++q) fout[q * n + x] = fin[q * n + x];
            continue;
        }
        const int I = t & 3, J = (t >> 2) & 3, K = t >> 4;
        float f[27];
        bool wall_any = false, outside_any = false;
#pragma unroll
        for (int o = 0; o < 27; ++o) {
            int ty;
            const int32_t y = cell_at(nbr, b, I, J, K, -c27(o, 0), -c27(o, 1), -c27(o, 2), ty);
            if (y >= s && y < e && masks[64 * (int64_t)y + ty] != VF_SOLID) {
                f[o] = fin[o * n + (int64_t)(y - s) * 64 + ty];
            } else {
                f[o] = __int_as_float(0x7fc00000);  // resolved below (rare)
                if (y == VF_NB_OUTSIDE) outside_any = true;
                else wall_any = true;
            }
        }
        if (outside_any || wall_any) {  // rare: resolved out of line on a local copy
            float fl[27];
#pragma unroll
            for (int o = 0; o < 27; ++o) fl[o] = f[o];
            resolve_links(fl, x, n, b, t, s, e, cells_x, coords, nbr, masks, cmap, lengths, fin,
                          flow, uin, Fx, Fy, Fz);
#pragma unroll
            for (int o = 0; o < 27; ++o) f[o] = fl[o];
        }
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
    if (d_force) {
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Fx += __shfl_xor_sync(0xffffffffu, Fx, off);
            Fy += __shfl_xor_sync(0xffffffffu, Fy, off);
            Fz += __shfl_xor_sync(0xffffffffu, Fz, off);
        }
        if ((threadIdx.x & 31) == 0 && (Fx != 0.f || Fy != 0.f || Fz != 0.f)) {
            atomicAdd(d_force + 0, (double)Fx);
            atomicAdd(d_force + 1, (double)Fy);
            atomicAdd(d_force + 2, (double)Fz);
        }
    }
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

int vf_lbm_step(const vf_config *cfg, const vf_grid *g, int level, int32_t s, int32_t e,
                const int32_t *cmap, const float *lengths, const float *fin, float *fout,
                const vf_flow *flow, double *d_force, void *stream) {
    if (!cfg || !g || !fin || !fout || !flow || fin == fout || s < 0 || e < s || e > g->capacity ||
        level < 0 || level >= VF_MAX_LEVELS || !(flow->tau > 0.5) || (flow->ibb && (!cmap || !lengths)))
        return set_error(VF_EARG, "vf_lbm_step: bad argument (tau must exceed 1/2)");
    if (e == s) return VF_OK;
    const int cells_x = 4 * (cfg->nb[0] << level);
    int64_t grid = ((int64_t)(e - s) * 64 + 255) / 256;
    if (grid > max_ctas(8)) grid = max_ctas(8);
    k_lbm_step<<<(int)grid, 256, 0, (cudaStream_t)stream>>>(s, e, cells_x, g->d_coords, g->d_nbr,
                                                             g->d_masks, cmap, lengths, fin, fout,
                                                             *flow, d_force);
    return check_launch("k_lbm_step");
}

}  // extern "C"
