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

constexpr int kBndWarps = 8;

// warp per finest-level block: the 27 neighbour ids decide candidacy (the
// block or a neighbour is solid); a 6x6x6 shared-memory halo of SOLID bits is
// gathered once, then every FLUID cell ORs its 26 halo neighbours (constant
// offsets).  Reads of concurrently re-marked cells see FLUID or BOUNDARY,
// both "not SOLID", so the fused single pass equals PAPER.md:941's two passes.
__global__ void __launch_bounds__(kBndWarps * 32)
    k_boundary(LevelInfo li, int L, const int32_t *__restrict__ level_start,
               const int32_t *__restrict__ nbr, const int32_t *__restrict__ coords,
               uint8_t *__restrict__ bflags, uint8_t *__restrict__ masks,
               const uint64_t *__restrict__ solid64, int32_t *__restrict__ bcount) {
    __shared__ uint8_t s_halo[kBndWarps][216];
    __shared__ uint64_t s_sol[kBndWarps][27];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t gw = (int64_t)blockIdx.x * kBndWarps + w, nw = (int64_t)gridDim.x * kBndWarps;
    const int32_t s = level_start[L], e = level_start[L + 1];
    for (int64_t b = s + gw; b < e; b += nw) {
        if (li.shard_count > 1) {  // multi-GPU: blocks of other ranks are theirs
            const int4 c = reinterpret_cast<const int4 *>(coords)[b];
            if (!owns_row(li, c.y, c.z)) continue;
        }
        int32_t myn = -1;
        if (lane < 27) myn = (lane == 0) ? (int32_t)b : nbr[27 * b + lane];
        // solid64 (exchanged between ranks) rather than the masks of
        // neighbours, which may belong to another rank
        const uint64_t sm = (lane < 27 && myn >= 0) ? solid64[myn] : 0ull;
        if (!__any_sync(0xffffffffu, sm != 0)) {  // not a candidate (A18): no boundary cell
            if (lane == 0) {
                bcount[b] = 0;
                bflags[b] = (uint8_t)(bflags[b] & ~VF_BF_BOUNDARY);
            }
            continue;
        }
        if (lane < 27) s_sol[w][lane] = sm;
        __syncwarp();
        for (int h = lane; h < 216; h += 32) {
            const int hx = h % 6 - 1, hy = (h / 6) % 6 - 1, hz = h / 36 - 1;
            const int ox = hx < 0 ? -1 : (hx > 3 ? 1 : 0);
            const int oy = hy < 0 ? -1 : (hy > 3 ? 1 : 0);
            const int oz = hz < 0 ? -1 : (hz > 3 ? 1 : 0);
            const uint64_t nsm = s_sol[w][slot_of(ox, oy, oz)];
            s_halo[w][h] = (uint8_t)((nsm >> ((hx & 3) + 4 * (hy & 3) + 16 * (hz & 3))) & 1ull);
        }
        __syncwarp();
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < 2; ++k) {
            const int c = lane + 32 * k;
            const int I = c & 3, J = (c >> 2) & 3, K = c >> 4;
            if (masks[64 * b + c] != VF_FLUID) continue;
            const uint8_t *hp = &s_halo[w][(I + 1) + 6 * (J + 1) + 36 * (K + 1)];
            uint32_t any = 0;
#pragma unroll
            for (int dz = -1; dz <= 1; ++dz)
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy)
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx)
                        if (dx || dy || dz) any |= hp[dx + 6 * dy + 36 * dz];
            if (any) {
                masks[64 * b + c] = VF_BOUNDARY;
                ++cnt;
            }
        }
        cnt = warp_sum(cnt);
        if (lane == 0) {
            bcount[b] = cnt;
            const uint8_t f = bflags[b];
            bflags[b] = (uint8_t)(cnt > 0 ? (f | VF_BF_BOUNDARY) : (f & ~VF_BF_BOUNDARY));
        }
        __syncwarp();
    }
}

int boundary_impl(const vf_config &cfg, vf_grid *g, int32_t *bcount, cudaStream_t st) {
    const int L = g->n_levels - 1;
    cudaMemsetAsync(bcount, 0, sizeof(int32_t) * (size_t)g->capacity, st);
    k_boundary<<<max_ctas(8), kBndWarps * 32, 0, st>>>(make_level(cfg, L), L, g->d_level_start,
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
    __device__ void operator()(int64_t i, int v, int ex) const {
        cmap[level_start[L] + i] = v ? ex : -1;
    }
};

__global__ void k_level_count2(int L, const int32_t *__restrict__ level_start, int32_t *__restrict__ out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *out = level_start[L + 1] - level_start[L];
}

size_t tables_workspace_size(int32_t capacity) {
    return 256 + ((scan_workspace_bytes(capacity) + 255) & ~(size_t)255);
}

int tables_impl(vf_grid *g, const int32_t *bcount, int32_t *cmap, int32_t *d_n_b, void *ws,
                size_t ws_bytes, cudaStream_t st) {
    if (ws_bytes < tables_workspace_size(g->capacity)) return set_error(VF_EARG, "tables workspace too small");
    const int L = g->n_levels - 1;
    int32_t *scal = (int32_t *)ws;
    void *scan_ws = (char *)ws + 256;
    // non-finest blocks are never mapped
    cudaMemsetAsync(cmap, 0xff, sizeof(int32_t) * (size_t)g->capacity, st);
    k_level_count2<<<1, 32, 0, st>>>(L, g->d_level_start, scal);
    int rc = check_launch("k_level_count2");
    if (rc) return rc;
    cudaError_t ce = scan_launch(LoadBnd{g->d_level_start, L, bcount}, EmitCmap{g->d_level_start, L, cmap},
                                 g->capacity, scal, d_n_b, scan_ws, st);
    return ce == cudaSuccess ? VF_OK : set_cuda_error(ce, "tables scan");
}

}  // namespace vf
