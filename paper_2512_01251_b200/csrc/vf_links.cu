// vf_links.cu -- boundary cells, boundary tables and the cut-link LUT
// (SPEC.md:319-345).
//
//   K-bnd    one CTA (64 threads = cells) per finest-level block that is solid
//            or touches a solid block; direct neighbour reads through the A15
//            index maps (the paper's faster "direct" variant).
//            Single pass: pass 1 only tests "== SOLID" and pass 2 only turns
//            FLUID into BOUNDARY, so fusing the two kernels of PAPER.md:941 is
//            race-free in outcome.
//   K-tab    contraction map = exclusive scan of (count > 0) over the finest
//            level in ascending block id (pin A16).
//   (link lengths: vf_linklen.cu)
#include <math.h>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

// 26-neighbour dilation of the SOLID cells: dil_x / dil_y / dil_z
// (vf_common.cuh); BOUNDARY = FLUID & D.
// thread per finest-level block: 27 solid64 words -> dilation -> FLUID cells
// of the block's masks that the dilation covers become BOUNDARY
#ifndef VF_BOUNDARY_MINB
#define VF_BOUNDARY_MINB 3
#endif
__global__ void __launch_bounds__(256, VF_BOUNDARY_MINB)
    k_boundary(LevelInfo li, int L, const int32_t *__restrict__ level_start,
               const int32_t *__restrict__ nbr, const int32_t *__restrict__ coords,
               uint8_t *__restrict__ bflags, uint8_t *__restrict__ masks,
               const uint64_t *__restrict__ solid64, int32_t *__restrict__ bcount) {
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < e;
         b += (int64_t)gridDim.x * blockDim.x) {
        if (li.shard_count > 1) {  // multi-GPU: blocks of other ranks are theirs
            const int4 c = reinterpret_cast<const int4 *>(coords)[b];
            if (!owns_row(li, c.y, c.z)) continue;
        }
        // solid64 (exchanged between ranks) rather than the neighbours' masks,
        // which may belong to another rank; missing neighbours contribute 0
        uint64_t S[27];
        uint64_t any = 0;
#pragma unroll
        for (int q = 0; q < 27; ++q) {
            const int32_t v = q == 0 ? (int32_t)b : __ldg(nbr + 27 * b + q);
            S[q] = v >= 0 ? __ldg(reinterpret_cast<const unsigned long long *>(solid64) + v) : 0ull;
            any |= S[q];
        }
        int cnt = 0;
        if (any) {  // candidate (A18): the block or a neighbour has a SOLID cell
            uint64_t pl[3];
#pragma unroll
            for (int oz = -1; oz <= 1; ++oz) {
                uint64_t col[3];
#pragma unroll
                for (int oy = -1; oy <= 1; ++oy)
                    col[oy + 1] = dil_x(S[slot_of(-1, oy, oz)], S[slot_of(0, oy, oz)], S[slot_of(1, oy, oz)]);
                pl[oz + 1] = dil_y(col[0], col[1], col[2]);
            }
            const uint64_t D = dil_z(pl[0], pl[1], pl[2]);
            uint32_t w[16];
            const uint4 *mp = reinterpret_cast<const uint4 *>(masks + 64 * b);
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const uint4 u = mp[k];
                w[4 * k] = u.x; w[4 * k + 1] = u.y; w[4 * k + 2] = u.z; w[4 * k + 3] = u.w;
            }
            bool changed = false;
#pragma unroll
            for (int r = 0; r < 16; ++r) {
                uint32_t x = w[r];
#pragma unroll
                for (int I = 0; I < 4; ++I) {
                    if (((x >> (8 * I)) & 0xffu) == VF_FLUID && ((D >> (4 * r + I)) & 1ull)) {
                        x |= (uint32_t)VF_BOUNDARY << (8 * I);
                        ++cnt;
                    }
                }
                changed |= x != w[r];
                w[r] = x;
            }
            if (changed) {
                uint4 *mo = reinterpret_cast<uint4 *>(masks + 64 * b);
#pragma unroll
                for (int k = 0; k < 4; ++k) mo[k] = make_uint4(w[4 * k], w[4 * k + 1], w[4 * k + 2], w[4 * k + 3]);
            }
        }
        bcount[b] = cnt;
        const uint8_t f = bflags[b];
        bflags[b] = (uint8_t)(cnt > 0 ? (f | VF_BF_BOUNDARY) : (f & ~VF_BF_BOUNDARY));
    }
}

int boundary_impl(const vf_config &cfg, vf_grid *g, int32_t *bcount, cudaStream_t st) {
    const int L = g->n_levels - 1;
    cudaMemsetAsync(bcount, 0, sizeof(int32_t) * (size_t)g->capacity, st);
    kt_point("memset:bcount");
    k_boundary<<<wave_ctas(k_boundary, 256), 256, 0, st>>>(make_level(cfg, L), L, g->d_level_start,
                                                       g->d_nbr, g->d_coords, g->d_bflags,
                                                       g->d_masks, g->d_solid64, bcount);
    return check_launch("k_boundary");
}

// ---------------------------------------------------------------------------
// tables

struct LoadBnd {
    const int32_t *level_start;
    int L;
    const int32_t *bcount;
    __device__ int operator()(int64_t i) const { return bcount[level_start[L] + i] > 0 ? 1 : 0; }
};
struct EmitCmap {
    const int32_t *level_start;
    int L;
    int32_t *cmap;
    int32_t *inv;  // nullable: slot -> block
    __device__ void operator()(int64_t i, int v, int ex) const {
        const int32_t b = level_start[L] + (int32_t)i;
        cmap[b] = v ? ex : -1;
        if (v && inv) inv[ex] = b;
    }
};

size_t tables_workspace_size(int32_t capacity) {
    return 256 + ((scan_workspace_bytes(capacity) + 255) & ~(size_t)255);
}

int tables_impl(vf_grid *g, const int32_t *bcount, int32_t *cmap, int32_t *d_n_b, void *ws,
                size_t ws_bytes, cudaStream_t st, int32_t *inv) {
    if (ws_bytes < tables_workspace_size(g->capacity)) return set_error(VF_EARG, "tables workspace too small");
    const int L = g->n_levels - 1;
    void *scan_ws = (char *)ws + 256;
    // non-finest blocks are never mapped
    cudaMemsetAsync(cmap, 0xff, sizeof(int32_t) * (size_t)g->capacity, st);
    kt_point("memset:cmap");
    cudaError_t ce = scan_launch_fn(LoadBnd{g->d_level_start, L, bcount}, EmitCmap{g->d_level_start, L, cmap, inv},
                                    g->capacity, ScanLevelN{g->d_level_start, L}, d_n_b, scan_ws, st);
    return ce == cudaSuccess ? VF_OK : set_cuda_error(ce, "tables scan");
}

}  // namespace vf
