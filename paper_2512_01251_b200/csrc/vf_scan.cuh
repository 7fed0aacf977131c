// vf_scan.cuh -- single-pass exclusive prefix scan with decoupled look-back.
//
// Used for every "stream compaction / scatter" step of the pipeline
// (face filtering, bin offsets = Thrust steps 5-9 of PAPER.md:477-479,
// child-id allocation, contraction map).  The element count may be
// device-resident (d_n), so a level never needs a host round trip: CTAs
// whose dynamic tile id lies beyond ceil(n/TILE) exit immediately.
//
//   Load(i)  -> int   value of element i (only called for i < n)
//   Emit(i, v, excl)  called for every i < n with its exclusive prefix
//   d_total          receives the sum (written by the last tile)
//
// Workspace: (tiles + 1) uint64 status words, zeroed by scan_launch.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace vf {

#ifndef VF_SCAN_MINB
#define VF_SCAN_MINB 6  // <= 40 registers: 48 warps per SM (measured best; 1 lets the compiler take 96)
#endif
constexpr int kScanThreads = 256;
#ifndef VF_SCAN_ITEMS
#define VF_SCAN_ITEMS 16
#endif
constexpr int kScanItems = VF_SCAN_ITEMS;
constexpr int kScanTile = kScanThreads * kScanItems;  // 4096

constexpr uint64_t kFlagAgg = 1ull << 32;
constexpr uint64_t kFlagPre = 2ull << 32;

__device__ __forceinline__ uint64_t ld_volatile_u64(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_volatile_u64(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// warp-wide sum (all lanes receive the total)
__device__ __forceinline__ int warp_sum_scan(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// element count: device-resident value, or the static bound
struct ScanN {
    const int32_t *d_n;
    int64_t n_static;
    __device__ int64_t operator()() const { return d_n ? (int64_t)(*d_n) : n_static; }
};
// element count of a level: level_start[L+1] - level_start[L] (device-resident)
struct ScanLevelN {
    const int32_t *level_start;
    int L;
    __device__ int64_t operator()() const { return (int64_t)level_start[L + 1] - level_start[L]; }
};
struct ScanNoEpi {
    __device__ void operator()(int) const {}
};

// Epi(total) runs once, on the thread that publishes the total (after every
// element's prefix is known to that thread's tile; other tiles may still be
// emitting, so Epi must not depend on Emit's outputs)
template <typename Load, typename Emit, typename NFn = ScanN, typename Epi = ScanNoEpi>
__global__ void __launch_bounds__(kScanThreads, VF_SCAN_MINB)
    scan_kernel(Load load, Emit emit, NFn nfn, int32_t *__restrict__ d_total,
                uint64_t *__restrict__ status, Epi epi = Epi()) {
    __shared__ int s_warp[kScanThreads / 32];
    __shared__ int s_tile;
    __shared__ int s_prefix;
    __shared__ int s_tile_agg;
    // tile staged through shared memory: loads and emits in warp-striped
    // (coalesced) order, the scan over 16 consecutive items per thread
    __shared__ int s_v[kScanTile + kScanTile / 32];
    const int64_t n = nfn();
    const int64_t n_tiles = (n + kScanTile - 1) / kScanTile;
    uint32_t *counter = reinterpret_cast<uint32_t *>(status);
    if (threadIdx.x == 0) s_tile = (int)atomicAdd(counter, 1u);
    __syncthreads();
    const int64_t tile = s_tile;
    if (n == 0) {
        if (tile == 0 && threadIdx.x == 0) {
            if (d_total) *d_total = 0;
            epi(0);
        }
        return;
    }
    if (tile >= n_tiles) return;
    uint64_t *tstat = status + 1;

    const int64_t tbase = tile * kScanTile;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int j = k * kScanThreads + threadIdx.x;
        const int64_t i = tbase + j;
        s_v[j + (j >> 5)] = (i < n) ? load(i) : 0;
    }
    __syncthreads();
    int vals[kScanItems];
    int tsum = 0;
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int j = threadIdx.x * kScanItems + k;
        vals[k] = s_v[j + (j >> 5)];
        tsum += vals[k];
    }
    // block-wide exclusive scan of the per-thread sums
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    if (warp == 0) {
        int w = (lane < kScanThreads / 32) ? s_warp[lane] : 0;
        int wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, wi, o);
            if (lane >= o) wi += y;
        }
        if (lane < kScanThreads / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
        const int agg = __shfl_sync(0xffffffffu, wi, kScanThreads / 32 - 1);
        // decoupled look-back (warp 0)
        int prefix = 0;
        if (tile == 0) {
            if (lane == 0) st_volatile_u64(&tstat[0], kFlagPre | (uint32_t)agg);
        } else {
            if (lane == 0) st_volatile_u64(&tstat[tile], kFlagAgg | (uint32_t)agg);
            int64_t pred = tile - 1;
            while (true) {
                const int64_t idx = pred - lane;
                uint64_t s;
                if (idx >= 0) {
                    do { s = ld_volatile_u64(&tstat[idx]); } while ((s >> 32) == 0);
                } else {
                    s = kFlagPre;  // virtual tile with prefix 0
                }
                const uint32_t pre_mask = __ballot_sync(0xffffffffu, (s >> 32) == 2);
                int v = (int)(uint32_t)(s & 0xffffffffu);
                if (pre_mask) {
                    const int first = __ffs(pre_mask) - 1;
                    if (lane > first) v = 0;
                    prefix += warp_sum_scan(v);
                    break;
                }
                prefix += warp_sum_scan(v);
                pred -= 32;
            }
            if (lane == 0) st_volatile_u64(&tstat[tile], kFlagPre | (uint32_t)(prefix + agg));
        }
        if (lane == 0) {
            s_prefix = prefix;
            s_tile_agg = agg;
            if (tile == n_tiles - 1) {
                if (d_total) *d_total = prefix + agg;
                epi(prefix + agg);
            }
        }
    }
    __syncthreads();
    int run = s_prefix + s_warp[warp] + incl - tsum;
    // exclusive prefixes back to shared memory (over the values: each
    // thread rewrites only its own 16 slots), then emit in striped order
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int j = threadIdx.x * kScanItems + k;
        s_v[j + (j >> 5)] = run;
        run += vals[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kScanItems; ++k) {
        const int j = k * kScanThreads + threadIdx.x;
        const int64_t i = tbase + j;
        if (i < n) {
            const int ex = s_v[j + (j >> 5)];
            const int jn = j + 1;
            // the value is the next exclusive prefix minus this one (the
            // tile's last item: the tile aggregate)
            const int nx = (j + 1 < kScanTile) ? s_v[jn + (jn >> 5)] : (s_prefix + s_tile_agg);
            emit(i, nx - ex, ex);
        }
    }
}

inline size_t scan_workspace_bytes(int64_t n_bound) {
    const int64_t tiles = (n_bound + kScanTile - 1) / kScanTile;
    return (size_t)(tiles + 2) * sizeof(uint64_t);
}

// n_bound bounds the device count (grid size); nfn gives the count on device
template <typename Load, typename Emit, typename NFn, typename Epi = ScanNoEpi>
cudaError_t scan_launch_fn(Load load, Emit emit, int64_t n_bound, NFn nfn, int32_t *d_total,
                           void *ws, cudaStream_t st, Epi epi = Epi()) {
    const int64_t tiles = (n_bound + kScanTile - 1) / kScanTile;
    cudaError_t e = cudaMemsetAsync(ws, 0, scan_workspace_bytes(n_bound), st);
    if (e != cudaSuccess) return e;
    const int64_t grid = tiles > 0 ? tiles : 1;
    scan_kernel<<<(unsigned)grid, kScanThreads, 0, st>>>(load, emit, nfn, d_total,
                                                        reinterpret_cast<uint64_t *>(ws), epi);
    return cudaGetLastError();
}

template <typename Load, typename Emit>
cudaError_t scan_launch(Load load, Emit emit, int64_t n_bound, const int32_t *d_n,
                        int32_t *d_total, void *ws, cudaStream_t st) {
    return scan_launch_fn(load, emit, n_bound, ScanN{d_n, n_bound}, d_total, ws, st);
}

}  // namespace vf
