// vf_bins.cu -- spatial-bin hierarchy build.
//
//   K-ind   face-parallel ray indicators, 1D (x-rows) or MD (13 rep. dirs)
//           (Alg. 1, pins SURVEY A6)
//   K-scan  compaction of kept faces (decoupled look-back, vf_scan.cuh)
//   K-pairs face-parallel bin candidates vs the dx-expanded bin box, written
//           into a per-face slot row (cap N_lim asserted) and, in the fused
//           build, histogrammed straight into the dense per-bin counts
//           (Alg. 2, pins A5)
//   K-scan  counts -> offsets (replaces Thrust steps 3-9)
//   K-scat  counting-sort scatter of face ids into their bin slices
//   K-sort  per-bin ascending face-id order (deterministic BinLevel,
//           SPEC.md:154,178) -- thread per bin for short slices, CTA per bin
//           for long ones.
#include <math.h>

#include <algorithm>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

// --------------------------------------------------------------------------
// K-ind

// row index range whose centres can lie in [A, B]: j in [ceil(A/dx - 1/2),
// floor(B/dx - 1/2)], widened by a relative 1e-9 (>> rounding).  Rows outside
// fail the SAT's exact box-axis comparison, so this is a superset (A6).
__device__ __forceinline__ bool tight_rows(double A, double B, double dx, int n, int &a, int &b) {
    const double fa = ceil(VF_DDIV(A, dx) - 0.5 - 1e-9);
    const double fb = floor(VF_DDIV(B, dx) - 0.5 + 1e-9);
    const double ca = fmax(fa, 0.0), cb = fmin(fb, (double)(n - 1));
    if (ca > cb) return false;
    a = (int)ca;
    b = (int)cb;
    return true;
}

// candidate x-rows of a face: centres within eps of its y/z extent.
// inv_dx is exact for power-of-two dx (else the range is widened by a row).
__device__ __forceinline__ bool face_rows(const double *v, const LevelInfo &li, double inv_dx,
                                          int widen, int &ja, int &jb, int &ka, int &kb) {
    const double eps = li.eps;
    const double ylo = fmin(fmin(v[1], v[4]), v[7]), yhi = fmax(fmax(v[1], v[4]), v[7]);
    const double zlo = fmin(fmin(v[2], v[5]), v[8]), zhi = fmax(fmax(v[2], v[5]), v[8]);
    // j in [ceil((lo-eps)/dx - 1/2), floor((hi+eps)/dx - 1/2)] (+- 1e-9 relative)
    const double fja = ceil((ylo - eps) * inv_dx - 0.5 - 1e-9) - widen;
    const double fjb = floor((yhi + eps) * inv_dx - 0.5 + 1e-9) + widen;
    const double fka = ceil((zlo - eps) * inv_dx - 0.5 - 1e-9) - widen;
    const double fkb = floor((zhi + eps) * inv_dx - 0.5 + 1e-9) + widen;
    const double cja = fmax(fja, 0.0), cjb = fmin(fjb, (double)(li.cells[1] - 1));
    const double cka = fmax(fka, 0.0), ckb = fmin(fkb, (double)(li.cells[2] - 1));
    if (cja > cjb || cka > ckb) return false;
    ja = (int)cja; jb = (int)cjb; ka = (int)cka; kb = (int)ckb;
    if (li.shard_count <= 1) return true;
    for (int k = ka; k <= kb; ++k)  // multi-GPU: does any candidate row belong to us?
        for (int j = ja; j <= jb; ++j)
            if (owns_row(li, j >> 2, k >> 2)) return true;
    return false;
}

// exact row tests of one face (rare path, run warp-converged from the queue)
__device__ __noinline__ bool indicator_rows(const double *__restrict__ faces, int64_t f,
                                            const LevelInfo &li, double inv_dx, int widen) {
    double v[9], n[3];
    load_face(faces, f, v, n);
    int ja, jb, ka, kb;
    if (!face_rows(v, li, inv_dx, widen, ja, jb, ka, kb)) return false;
    const double dx = li.dx, eps = li.eps;
    SatFace sf;
    sat_face_init(sf, v);
    for (int k = ka; k <= kb; ++k) {
        const double z = node_c(k, dx);
        for (int j = ja; j <= jb; ++j) {
            if (!owns_row(li, j >> 2, k >> 2)) continue;  // multi-GPU: rows of other ranks
            const double y = node_c(j, dx);
            if (sat_exact(sf, 0.0, VF_DSUB(y, eps), VF_DSUB(z, eps), li.len[0], VF_DADD(y, eps),
                          VF_DADD(z, eps)))
                return true;
        }
    }
    return false;
}

// 1D indicators (Alg. 1 axis-only, pin A6): a streaming pass over all faces
// computes the candidate row ranges (most faces have none at coarse levels);
// faces with rows enter a per-warp queue that is drained 32 at a time through
// the exact SAT, so the FP64 path runs warp-converged.
constexpr int kIndWarps = 8;

__global__ void __launch_bounds__(kIndWarps * 32, 3)
    k_indicators_1d(LevelInfo li, double inv_dx, int widen, const double *__restrict__ faces,
                    int64_t F, uint8_t *__restrict__ out) {
    __shared__ int64_t s_q[kIndWarps][64];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int64_t first = ((int64_t)blockIdx.x * kIndWarps + w) * 32;
    const int64_t stride = (int64_t)gridDim.x * kIndWarps * 32;
    int qn = 0;
    for (int64_t base = first; base < F; base += stride) {
        const int64_t f = base + lane;
        bool has = false;
        if (f < F) {
            double v[9], n[3];
            load_face(faces, f, v, n);
            int ja, jb, ka, kb;
            has = !(fabs(n[0]) < li.eps_par) && face_rows(v, li, inv_dx, widen, ja, jb, ka, kb);
            if (!has) out[f] = 0;
        }
        const uint32_t m = __ballot_sync(0xffffffffu, has);
        if (has) s_q[w][qn + __popc(m & ((1u << lane) - 1u))] = f;
        qn += __popc(m);
        __syncwarp();
        if (qn >= 32) {
            const int64_t g = s_q[w][qn - 32 + lane];
            __syncwarp();
            out[g] = (uint8_t)indicator_rows(faces, g, li, inv_dx, widen);
            qn -= 32;
        }
        __syncwarp();
    }
    if (lane < qn) {
        const int64_t g = s_q[w][lane];
        out[g] = (uint8_t)indicator_rows(faces, g, li, inv_dx, widen);
    }
}

#ifndef VF_IND_MINB
#define VF_IND_MINB 2  // 120 registers, no spills (3: 80 + 128 B stack)
#endif
// All levels in ONE pass over the face records (the per-level kernel reads
// the 96 B/face records once per level): bit L of out[f] is the 1D indicator
// of face f at level L.  Candidate rows are decided by the FP32 row
// classifier (vf_common.cuh); only undecided rows run the exact SAT.  Same
// predicate as indicator_rows, row for row.
// The face records reach the warps through shared memory: a warp takes 32
// consecutive faces (3 KB) at a time and prefetches its next 32 with
// cp.async (16 B per lane-copy, L2 only) while it classifies the current
// ones, so the record stream keeps flowing through the long, divergent row
// loops (double-buffered per warp; no block barriers).
constexpr int kIndFaceD2 = kFaceStride / 2;  // double2 per face record
__device__ __forceinline__ void ind_prefetch(const double *__restrict__ faces, int64_t F, int64_t c, double2 *dst,
                                             int lane) {
    const int64_t f0 = c * 32;
    const int64_t nf = F - f0 < 32 ? F - f0 : 32;
    const double2 *src = reinterpret_cast<const double2 *>(faces + f0 * kFaceStride);
    for (int i = lane; i < nf * kIndFaceD2; i += 32) {
        const unsigned d = (unsigned)__cvta_generic_to_shared(dst + i);
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(d), "l"(src + i) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

__global__ void __launch_bounds__(256, VF_IND_MINB)
    k_indicators_all(LevelSet ls, const double *__restrict__ faces, int64_t F,
                     uint16_t *__restrict__ out) {
    __shared__ double2 s_rec[8][2][32 * kIndFaceD2];  // per warp: two 32-face buffers (48 KB)
    const int lane = threadIdx.x & 31, wi = threadIdx.x >> 5;
    const int64_t nchunk = (F + 31) / 32, cstride = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t c = (int64_t)blockIdx.x * (blockDim.x >> 5) + wi;
    if (c < nchunk) ind_prefetch(faces, F, c, s_rec[wi][0], lane);
    for (int buf = 0; c < nchunk; c += cstride, buf ^= 1) {
        if (c + cstride < nchunk) {
            ind_prefetch(faces, F, c + cstride, s_rec[wi][buf ^ 1], lane);
            asm volatile("cp.async.wait_group 1;" ::: "memory");
        } else {
            asm volatile("cp.async.wait_group 0;" ::: "memory");
        }
        __syncwarp();
        const int64_t f = c * 32 + lane;
        double v[9], n[3];
        if (f < F) {
            const double2 *p = s_rec[wi][buf] + lane * kIndFaceD2;
            const double2 a = p[0], b = p[1], cc = p[2], d = p[3], e = p[4], g = p[5];
            v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = cc.x; v[5] = cc.y;
            v[6] = d.x; v[7] = d.y; v[8] = e.x;
            n[0] = e.y; n[1] = g.x; n[2] = g.y;
        }
        __syncwarp();  // the buffer is refilled two chunks later
        if (f >= F) continue;
        uint32_t bits = 0;
        if (!(fabs(n[0]) < ls.li[0].eps_par)) {
            const double xlo = fmin(fmin(v[0], v[3]), v[6]), xhi = fmax(fmax(v[0], v[3]), v[6]);
            // level-independent part of the row classifier (row_class_init):
            // the yz edge functions, their lengths, orientation, fast-accept
            // eligibility; per level only the margins change with dx
            const float a1 = (float)(v[4] - v[1]), b1 = (float)(v[5] - v[2]);
            const float a2 = (float)(v[7] - v[1]), b2 = (float)(v[8] - v[2]);
            const float cr = a1 * b2 - b1 * a2;
            const float ext = fmaxf(fmaxf(fabsf(a1), fabsf(b1)), fmaxf(fabsf(a2), fabsf(b2)));
            const float e1a = a2 - a1, e1b = b2 - b1;
            const float l0 = sqrtf(a1 * a1 + b1 * b1), l1 = sqrtf(e1a * e1a + e1b * e1b), l2 = sqrtf(a2 * a2 + b2 * b2);
            const float sg = cr >= 0.0f ? 1.0f : -1.0f;
            const double tx = 1e-6 * ls.li[0].len[0];
            const bool acc = fabs(n[0]) >= 1e-3 && xlo > tx && xhi < ls.li[0].len[0] - tx && cr != 0.0f;
            // candidate row ranges in FP32 from the face's y/z extent in
            // finest-level cells (power-of-two dx: exact level scaling; the
            // 0.01-cell padding covers the FP32 rounding, extra rows are
            // rejected by the row test itself -- same bits as face_rows)
            const int Lf = ls.n - 1;
            const double invf = ls.inv_dx[Lf], eps0 = ls.li[0].eps;
            const float ya = (float)((fmin(fmin(v[1], v[4]), v[7]) - eps0) * invf);
            const float yb = (float)((fmax(fmax(v[1], v[4]), v[7]) + eps0) * invf);
            const float za = (float)((fmin(fmin(v[2], v[5]), v[8]) - eps0) * invf);
            const float zb = (float)((fmax(fmax(v[2], v[5]), v[8]) + eps0) * invf);
            for (int L = 0; L < ls.n; ++L) {
                const LevelInfo &li = ls.li[L];
                int ja, jb, ka, kb;
                if (ls.widen[L] == 0 && li.eps == eps0 && li.shard_count <= 1) {
                    const float sc = ldexpf(1.0f, L - Lf);
                    ja = max((int)ceilf(ya * sc - 0.5f - 0.01f), 0);
                    jb = min((int)floorf(yb * sc - 0.5f + 0.01f), li.cells[1] - 1);
                    ka = max((int)ceilf(za * sc - 0.5f - 0.01f), 0);
                    kb = min((int)floorf(zb * sc - 0.5f + 0.01f), li.cells[2] - 1);
                    if (ja > jb || ka > kb) continue;
                } else if (!face_rows(v, li, ls.inv_dx[L], ls.widen[L], ja, jb, ka, kb)) {
                    continue;
                }
                const double dx = li.dx, eps = li.eps;
                RowClass rc;
                {  // = row_class_init(rc, v, n, xlo, xhi, dx, eps, li.len[0])
                    const float tol = 1e-5f * (ext + (float)dx) + 6.0f * (float)eps;
                    const float ab = 4e-6f * (ext + (float)dx) * (ext + (float)dx);
                    rc.yz = make_float4(a1, b1, a2, b2);
                    rc.tol = make_float4(tol * l0 + ab, tol * l1 + ab, tol * l2 + ab, acc ? sg : 2.0f * sg);
                }
                bool hit = false;
                for (int k = ka; k <= kb && !hit; ++k) {
                    const double z = node_c(k, dx);
                    for (int j = ja; j <= jb; ++j) {
                        if (!owns_row(li, j >> 2, k >> 2)) continue;
                        const double y = node_c(j, dx);
                        const int cls = row_class(rc, (float)VF_DSUB(y, v[1]), (float)VF_DSUB(z, v[2]));
                        if (cls == 0) continue;
                        if (cls == 1 || row_sat_exact_f(faces, f, y, z, eps, li.len[0])) {
                            hit = true;
                            break;
                        }
                    }
                }
                if (hit) bits |= 1u << L;
            }
        }
        out[f] = (uint16_t)bits;
    }
}

// The kept faces of every level appended to that level's compact_map from the
// indicator bits (2 B/face, instead of a compaction scan over F per level).
// A warp owns a contiguous segment of 1024 faces: pass 1 counts the kept
// faces per level (ballots), one atomic per level reserves the warp's slots,
// pass 2 re-reads the bits (L1) and writes the face ids.  No shared memory,
// no barriers.  The maps are unordered across warps -- the embed's pair
// lists and block bins are order-free (the voxelizer breaks ties by face id).
constexpr int kMapSeg = 1024;

__global__ void __launch_bounds__(256)
    k_bits_to_maps(const uint16_t *__restrict__ bits_in, int64_t F, int nL, int32_t *__restrict__ maps,
                   int64_t map_stride, int32_t *__restrict__ n_maps) {
    const int lane = threadIdx.x & 31;
    const int64_t nseg = (F + kMapSeg - 1) / kMapSeg;
    for (int64_t sg = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); sg < nseg;
         sg += (int64_t)gridDim.x * (blockDim.x >> 5)) {
        const int64_t f0 = sg * kMapSeg;
        uint32_t cnt[VF_MAX_LEVELS];
#pragma unroll
        for (int L = 0; L < VF_MAX_LEVELS; ++L) cnt[L] = 0;
        for (int i = 0; i < kMapSeg; i += 32) {
            const int64_t f = f0 + i + lane;
            const uint32_t bits = f < F ? __ldg(bits_in + f) : 0u;
#pragma unroll
            for (int L = 0; L < VF_MAX_LEVELS; ++L)
                if (L < nL) cnt[L] += __popc(__ballot_sync(0xffffffffu, (bits >> L) & 1u));
        }
        uint32_t base[VF_MAX_LEVELS];
#pragma unroll
        for (int L = 0; L < VF_MAX_LEVELS; ++L) {
            int b = 0;
            if (L < nL && lane == 0 && cnt[L]) b = atomicAdd(&n_maps[L], (int)cnt[L]);
            base[L] = (uint32_t)__shfl_sync(0xffffffffu, b, 0);
        }
        for (int i = 0; i < kMapSeg; i += 32) {
            const int64_t f = f0 + i + lane;
            const uint32_t bits = f < F ? __ldg(bits_in + f) : 0u;
#pragma unroll
            for (int L = 0; L < VF_MAX_LEVELS; ++L) {
                if (L >= nL) break;
                const uint32_t m = __ballot_sync(0xffffffffu, (bits >> L) & 1u);
                if ((bits >> L) & 1u) maps[L * map_stride + base[L] + __popc(m & ((1u << lane) - 1u))] = (int32_t)f;
                base[L] += __popc(m);
            }
        }
    }
}

int launch_indicators_all(const vf_config &cfg, const double *faces, int64_t F, uint16_t *out,
                          int32_t *maps, int64_t map_stride, int32_t *n_maps, cudaStream_t st) {
    if (F <= 0) return VF_OK;
    LevelSet ls;
    ls.n = cfg.l_max;
    for (int L = 0; L < cfg.l_max; ++L) {
        ls.li[L] = make_level(cfg, L);
        int ex = 0;
        ls.widen[L] = (frexp(ls.li[L].dx, &ex) == 0.5) ? 0 : 1;  // 1/dx exact for 2^-k
        ls.inv_dx[L] = 1.0 / ls.li[L].dx;
    }
    int64_t g = (F + 255) / 256;
    if (g > max_ctas(8)) g = max_ctas(8);
    k_indicators_all<<<(int)g, 256, 0, st>>>(ls, faces, F, out);
    int rc = check_launch("k_indicators_all");
    if (rc || !maps) return rc;
    cudaMemsetAsync(n_maps, 0, sizeof(int32_t) * cfg.l_max, st);
    kt_point("memset:n_maps");
    int64_t gm = ((F + kMapSeg - 1) / kMapSeg + 7) / 8;
    if (gm > max_ctas(8)) gm = max_ctas(8);
    k_bits_to_maps<<<(int)(gm < 1 ? 1 : gm), 256, 0, st>>>(out, F, cfg.l_max, maps, map_stride, n_maps);
    return check_launch("k_bits_to_maps");
}

__device__ bool indicator_md(const double *v, const double *n, const LevelInfo &li) {
    SatFace f;
    sat_face_init(f, v);
    const double dx = li.dx, eps = li.eps;
    int a[3], b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        double fa = floor(VF_DDIV(f.lo[d], dx)) - 1.0, fb = floor(VF_DDIV(f.hi[d], dx)) + 1.0;
        fa = fmax(fa, 0.0);
        fb = fmin(fb, (double)(li.cells[d] - 1));
        if (fa > fb) return false;
        a[d] = (int)fa;
        b[d] = (int)fb;
    }
    for (int q = 1; q < 27; q += 2) {
        const double c0 = c27(q, 0), c1 = c27(q, 1), c2 = c27(q, 2);
        const double cn = __dsqrt_rn(VF_DADD(VF_DADD(VF_DMUL(c0, c0), VF_DMUL(c1, c1)), VF_DMUL(c2, c2)));
        const double den = VF_DADD(VF_DADD(VF_DMUL(c0, n[0]), VF_DMUL(c1, n[1])), VF_DMUL(c2, n[2]));
        if (fabs(den) < VF_DMUL(li.eps_par, cn)) continue;
        for (int k = a[2]; k <= b[2]; ++k) {
            const double z = node_c(k, dx);
            for (int j = a[1]; j <= b[1]; ++j) {
                const double y = node_c(j, dx);
                for (int i = a[0]; i <= b[0]; ++i) {
                    const double x = node_c(i, dx);
                    const double d = VF_DDIV(plane_num(v, n, x, y, z), den);
                    const double xi = VF_DADD(x, VF_DMUL(d, c0));
                    const double yi = VF_DADD(y, VF_DMUL(d, c1));
                    const double zi = VF_DADD(z, VF_DMUL(d, c2));
                    if (sat_exact(f, VF_DSUB(xi, eps), VF_DSUB(yi, eps), VF_DSUB(zi, eps),
                                  VF_DADD(xi, eps), VF_DADD(yi, eps), VF_DADD(zi, eps)))
                        return true;
                }
            }
        }
    }
    return false;
}

// min 3 CTAs/SM (<= 85 registers): the face scan is memory bound and the SAT
// path (the only register-hungry part) runs for few faces
template <int MODE>
__global__ void __launch_bounds__(256, 3)
    k_indicators(LevelInfo li, const double *__restrict__ faces, int64_t F,
                 uint8_t *__restrict__ out) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F;
         f += (int64_t)gridDim.x * blockDim.x) {
        double v[9], n[3];
        load_face(faces, f, v, n);
        out[f] = (uint8_t)indicator_md(v, n, li);
    }
}

// --------------------------------------------------------------------------
// K-pairs

// exact SAT of one candidate bin box (the classifier's undecided case): the
// face is re-read (L1) and the SAT set up here, out of line, so the hot loop
// of k_pairs does not carry the SatFace registers
static __device__ __noinline__ bool bin_sat_exact_f(const double *__restrict__ faces, int64_t f,
                                                    double mx, double my, double mz, double Mx,
                                                    double My, double Mz) {
    double v[9], n[3];
    load_face(faces, f, v, n);
    SatFace sf;
    sat_face_init(sf, v);
    return sat_exact(sf, mx, my, mz, Mx, My, Mz);
}

// Alg. 2 literally: every candidate bin through the exact SAT (faces with
// more than 32 candidate bins along an axis -- long slivers)
static __device__ __noinline__ int face_pairs_generic(const double *__restrict__ faces, int64_t fid,
                                                      const LevelInfo &li, int nlim, int32_t *slot,
                                                      int32_t *counts) {
    double v[9], n[3];
    load_face(faces, fid, v, n);
    SatFace f;
    sat_face_init(f, v);
    const double dx = li.dx, h = li.h;
    int a[3], b[3];
    for (int d = 0; d < 3; ++d) {
        const double s = VF_DDIV((double)li.bins[d], li.len[d]);
        a[d] = (int)fmax(floor(VF_DMUL(f.lo[d], s)) - 1.0, 0.0);
        b[d] = (int)fmin(floor(VF_DMUL(f.hi[d], s)) + 1.0, (double)(li.bins[d] - 1));
    }
    int cnt = 0;
    for (int bk = a[2]; bk <= b[2]; ++bk) {
        const double mz = VF_DSUB(VF_DMUL((double)bk, h), dx), Mz = VF_DADD(VF_DMUL((double)(bk + 1), h), dx);
        for (int bj = a[1]; bj <= b[1]; ++bj) {
            if (!owns_row(li, bj, bk)) continue;
            const double my = VF_DSUB(VF_DMUL((double)bj, h), dx), My = VF_DADD(VF_DMUL((double)(bj + 1), h), dx);
            for (int bi = a[0]; bi <= b[0]; ++bi) {
                const double mx = VF_DSUB(VF_DMUL((double)bi, h), dx), Mx = VF_DADD(VF_DMUL((double)(bi + 1), h), dx);
                if (sat_exact(f, mx, my, mz, Mx, My, Mz)) {
                    if (cnt >= nlim) return -1;
                    slot[cnt++] = bi + li.bins[0] * (bj + li.bins[1] * bk);
                }
            }
        }
    }
    if (counts)
        for (int k = 0; k < cnt; ++k) atomicAdd(&counts[slot[k]], 1);
    return cnt;
}

// FP32 classifier of the SAT of a face against one (Delta x-expanded) bin
// box: 1 = the reference SAT (geometry.py:441-500) certainly accepts, 0 =
// certainly rejects, 2 = undecided (run the exact SAT).  Face-local frame:
// u2, u3 = FP32(v2 - v1), FP32(v3 - v1) (v1 at the origin); (cx, cy, cz) =
// FP32(box centre - v1), (rx, ry, rz) the half widths.
// The SAT is the conjunction of per-axis tests; the box axes are decided
// exactly by the caller.  For each of the 9 edge axes e of the planes yz, xy,
// zx and for the plane-cut test the separation s (box-centre projection vs
// the triangle's projection widened by the box's) is evaluated in FP32:
//   edge axes: |s_32 - s_ref| <= 2 W |de|_1 + FP32 rounding + the reference's
//     own FP64 rounding (<= 6u C |e|_1), with |de| <= 2.4e-7 E the FP32
//     rounding of the local axis; tau_e = |e|_1 (4e-6 W + Ct) + 4e-6 E W
//     (W: largest local |coordinate| + box half width, E: largest edge
//     component, Ct = 1e-14 C, C >= every |absolute coordinate|);
//   plane: |n_32 - n_ref| <= 8.3e-7 E^2 per component, the reference's pn
//     rounding <= 8u E^2; tau_p = E^2 (4e-5 W + 6 Ct).
// An axis whose reference components are exactly zero (edge parallel to the
// plane's normal axis: bit in `zero`) never separates and is skipped.  Sure
// separation on one axis => the reference rejects; sure overlap on every
// axis => it accepts (every per-axis outcome agrees with the reference's).
__device__ __forceinline__ int bin_class(const float *u2, const float *u3, float cx, float cy,
                                         float cz, float rx, float ry, float rz, float E, float W,
                                         float Ct, uint32_t zero) {
    const float c[3] = {cx, cy, cz}, r[3] = {rx, ry, rz};
    bool sure = true;
#pragma unroll
    for (int pl = 0; pl < 3; ++pl) {
        const int A = pl == 0 ? 1 : (pl == 1 ? 0 : 2), B = pl == 0 ? 2 : (pl == 1 ? 1 : 0);
        const float a2 = u2[A], b2 = u2[B], a3 = u3[A], b3 = u3[B];
#pragma unroll
        for (int e = 0; e < 3; ++e) {
            if ((zero >> (3 * pl + e)) & 1u) continue;
            // edge j -> j+1: (e_x, e_y) = (b_{j+1} - b_j, a_j - a_{j+1}), v1 = 0
            const float ex = e == 0 ? b2 : (e == 1 ? b3 - b2 : -b3);
            const float ey = e == 0 ? -a2 : (e == 1 ? a2 - a3 : a3);
            const float t2 = a2 * ex + b2 * ey, t3 = a3 * ex + b3 * ey;
            const float lo = fminf(0.0f, fminf(t2, t3)) - (r[A] * fabsf(ex) + r[B] * fabsf(ey));
            const float hi = fmaxf(0.0f, fmaxf(t2, t3)) + (r[A] * fabsf(ex) + r[B] * fabsf(ey));
            const float p = c[A] * ex + c[B] * ey;
            const float tau = (fabsf(ex) + fabsf(ey)) * (4e-6f * W + Ct) + 4e-6f * E * W;
            if (p < lo - tau || p > hi + tau) return 0;
            if (p < lo + tau || p > hi - tau) sure = false;
        }
    }
    const float nx = u2[1] * u3[2] - u2[2] * u3[1];
    const float ny = u2[2] * u3[0] - u2[0] * u3[2];
    const float nz = u2[0] * u3[1] - u2[1] * u3[0];
    const float Rn = rx * fabsf(nx) + ry * fabsf(ny) + rz * fabsf(nz);
    const float pn = fabsf(nx * cx + ny * cy + nz * cz);
    const float taup = E * E * (4e-5f * W + 6.0f * Ct);
    if (pn > Rn + taup) return 0;
    if (pn > Rn - taup) sure = false;
    return sure ? 1 : 2;
}

// Candidate bins of one face (Alg. 2, pins A5); returns the count or -1 on
// cap violation.  Every candidate bin I_min-1..I_max+1 is decided exactly as
// the reference SAT (geometry.py:441-500) decides it, but the FP64 SAT only
// runs where its outcome is not certain:
//   * box axes: the SAT's three box-axis tests are exact comparisons of the
//     face extent with the bin box [I h - dx, (I+1) h + dx]; they are
//     separable, so each axis' candidate range is pruned to the bins that
//     pass them (bit masks, same FP64 box bounds as the SAT call);
//   * a vertex strictly inside the box by mg = 1e-10 C (C >= every |coord|
//     of face and box) in all three axes: the SAT accepts.  Each of the 9
//     edge axes projects that vertex into the box's projection with slack
//     mg (|e_x| + |e_y|) >> the FP64 rounding of the projections (~6u C);
//     the plane-cut test has (d + d1) >= mg |n|_1 and (d + d2) <= -mg |n|_1
//     up to ~6u |n|_1 C for the plane's anchor v1.  For v2 / v3 the computed
//     normal misses them by |dn . e| <= 24u E^3 (E: largest edge
//     component), so they are used only when the face is well conditioned,
//     |n|_1 >= 1e-3 E^2 (FP32 estimate >= 2e-3 E^2), where mg |n|_1 >=
//     1e-13 E^3 dominates;
//   * the FP32 classifier bin_class; its undecided band: the exact SAT.
// The accepted set -- hence the pairs, their x-fastest order and the cap
// check -- is identical to testing every candidate with the SAT.
__device__ __forceinline__ int face_pairs(const double *__restrict__ faces, int64_t fid, const double *v,
                          const LevelInfo &li, int nlim, int32_t *slot,
                          int32_t *counts /* nullable: fused histogram */) {
    double lo[3], hi[3];
    double C = fmax(fmax(li.len[0], li.len[1]), li.len[2]) + li.h;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        lo[d] = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
        hi[d] = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
        if (hi[d] < 0.0 || lo[d] > li.len[d]) return 0;  // outside domain
        C = fmax(C, fmax(fabs(lo[d]), fabs(hi[d])));
    }
    const double mg = 1e-10 * C;
    // face-local FP32 frame (bin_class) and the conditioning of the plane
    // test for v2 / v3
    float u2[3], u3[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        u2[d] = (float)(v[3 + d] - v[d]);
        u3[d] = (float)(v[6 + d] - v[d]);
    }
    const float E = fmaxf(fmaxf(fmaxf(fabsf(u2[0]), fabsf(u2[1])), fmaxf(fabsf(u2[2]), fabsf(u3[0]))),
                          fmaxf(fabsf(u3[1]), fabsf(u3[2])));
    bool cond;
    {
        const float nx = u2[1] * u3[2] - u2[2] * u3[1], ny = u2[2] * u3[0] - u2[0] * u3[2],
                    nz = u2[0] * u3[1] - u2[1] * u3[0];
        cond = fabsf(nx) + fabsf(ny) + fabsf(nz) >= 2e-3f * E * E;
    }
    // edge axes whose reference components are exactly zero (never separate)
    uint32_t zero = 0;
    {
        const int A[3] = {1, 0, 2}, B[3] = {2, 1, 0};
#pragma unroll
        for (int pl = 0; pl < 3; ++pl)
#pragma unroll
            for (int e = 0; e < 3; ++e) {
                const int j = e, k = (e + 1) % 3;
                if (v[3 * j + A[pl]] == v[3 * k + A[pl]] && v[3 * j + B[pl]] == v[3 * k + B[pl]])
                    zero |= 1u << (3 * pl + e);
            }
    }
    const float Ct = (float)(1e-14 * C);
    const double dx = li.dx, h = li.h;
    const float rh = (float)(0.5 * h + dx);
    int a[3], b[3];
    uint32_t pass[3], in[3][3];  // per axis: box-axis pass bits; per vertex: inside-with-margin bits
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double s = VF_DDIV((double)li.bins[d], li.len[d]);
        double fa = floor(VF_DMUL(lo[d], s)) - 1.0, fb = floor(VF_DMUL(hi[d], s)) + 1.0;
        fa = fmax(fa, 0.0);
        fb = fmin(fb, (double)(li.bins[d] - 1));
        if (fa > fb) return 0;
        a[d] = (int)fa;
        b[d] = (int)fb;
        if (b[d] - a[d] >= 32) return face_pairs_generic(faces, fid, li, nlim, slot, counts);
        pass[d] = 0;
        in[0][d] = in[1][d] = in[2][d] = 0;
        for (int I = a[d]; I <= b[d]; ++I) {
            const double m = VF_DSUB(VF_DMUL((double)I, h), dx), M = VF_DADD(VF_DMUL((double)(I + 1), h), dx);
            const uint32_t bit = 1u << (I - a[d]);
            if (!(hi[d] < m || M < lo[d])) pass[d] |= bit;
            const double ml = m + mg, Ml = M - mg;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (ml < v[3 * k + d] && v[3 * k + d] < Ml) in[k][d] |= bit;
        }
    }
    // W: largest local |coordinate| (vertices, candidate box centres) + box half width
    float W = E;
#pragma unroll
    for (int d = 0; d < 3; ++d)
        W = fmaxf(W, fmaxf(fabsf((float)(((double)a[d] + 0.5) * h - v[d])),
                           fabsf((float)(((double)b[d] + 0.5) * h - v[d]))));
    W += rh * 1.0001f;
    const int64_t nbx = li.bins[0], nby = li.bins[1];
    int cnt = 0;
    for (uint32_t mz = pass[2]; mz; mz &= mz - 1) {
        const int oz = __ffs(mz) - 1, bk = a[2] + oz;
        const double bz0 = VF_DSUB(VF_DMUL((double)bk, h), dx), bz1 = VF_DADD(VF_DMUL((double)(bk + 1), h), dx);
        const float cz = (float)(0.5 * (bz0 + bz1) - v[2]), rz = (float)(0.5 * (bz1 - bz0));
        for (uint32_t my = pass[1]; my; my &= my - 1) {
            const int oy = __ffs(my) - 1, bj = a[1] + oy;
            if (!owns_row(li, bj, bk)) continue;  // multi-GPU: bins of other ranks
            const double by0 = VF_DSUB(VF_DMUL((double)bj, h), dx), by1 = VF_DADD(VF_DMUL((double)(bj + 1), h), dx);
            const float cy = (float)(0.5 * (by0 + by1) - v[1]), ry = (float)(0.5 * (by1 - by0));
            // vertices inside (y, z) of this bin, per x bit
            uint32_t fx = 0;
#pragma unroll
            for (int k = 0; k < 3; ++k)
                if (((in[k][1] >> oy) & (in[k][2] >> oz) & 1u) && (k == 0 || cond)) fx |= in[k][0];
            for (uint32_t mx = pass[0]; mx; mx &= mx - 1) {
                const int ox = __ffs(mx) - 1, bi = a[0] + ox;
                bool acc = (fx >> ox) & 1u;
                if (!acc) {
                    const double bx0 = VF_DSUB(VF_DMUL((double)bi, h), dx), bx1 = VF_DADD(VF_DMUL((double)(bi + 1), h), dx);
                    const int cls = bin_class(u2, u3, (float)(0.5 * (bx0 + bx1) - v[0]), cy, cz,
                                              (float)(0.5 * (bx1 - bx0)), ry, rz, E, W, Ct, zero);
                    acc = cls == 1 || (cls == 2 && bin_sat_exact_f(faces, fid, bx0, by0, bz0, bx1, by1, bz1));
                }
                if (acc) {
                    if (cnt >= nlim) return -1;  // no histogram entry was made yet
                    slot[cnt++] = (int32_t)(bi + nbx * (bj + nby * (int64_t)bk));
                }
            }
        }
    }
    // histogram only once the face is known to respect N_lim: a capped face
    // contributes nothing, so the bin slices stay consistent with the scatter
    if (counts)
        for (int k = 0; k < cnt; ++k) atomicAdd(&counts[slot[k]], 1);
    return cnt;
}

// K-pairs: thread per kept face (face_pairs).  A warp-flattened variant
// ((face, candidate bin) work spread over the lanes, per-face 64-bit accept
// masks in shared memory) was measured slower on the B200: the candidate
// decode and the shared 64-bit atomics cost more than the idle lanes.
#ifndef VF_PAIRS_MINB
#define VF_PAIRS_MINB 4
#endif
constexpr int kPairThreads = 128;
__global__ void __launch_bounds__(kPairThreads, VF_PAIRS_MINB)
    k_pairs(LevelInfo li, int nlim, const double *__restrict__ faces,
            const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map, int64_t n_static,
            int32_t *__restrict__ slots, int32_t *__restrict__ slot_cnt,
            int32_t *__restrict__ counts, int32_t *__restrict__ d_status) {
    const int64_t n = d_n_map ? (int64_t)*d_n_map : n_static;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int64_t f = map ? (int64_t)map[m] : m;
        double v[9], nn[3];
        load_face(faces, f, v, nn);
        int c = face_pairs(faces, f, v, li, nlim, slots + m * nlim, counts);
        if (c < 0) {
            latch_status(d_status, VF_ENLIM);
            c = 0;
        }
        slot_cnt[m] = c;
    }
}

// Embed pairs (block-indexed bins): the same accepted (bin, face) set as
// k_pairs, appended compactly to one (bin, face) list -- one global slot
// reservation per warp -- instead of a per-face row of N_lim slots: the
// reserved memory is the list capacity, not F * N_lim.  The per-face slots
// are staged in shared memory (row stride N_lim + 1: no bank conflicts).
// Capacity overflow latches VF_ECAPACITY with the required count in
// status[3] (the engine re-sizes and reruns).
__global__ void __launch_bounds__(kPairThreads, VF_PAIRS_MINB)
    k_pairs_append(LevelInfo li, int nlim, const double *__restrict__ faces,
                   const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map,
                   int64_t n_static, int2 *__restrict__ pairs, int32_t *__restrict__ d_n_pairs,
                   int64_t cap, int32_t *__restrict__ d_status) {
    extern __shared__ int32_t s_slots[];
    int32_t *slot = s_slots + threadIdx.x * (nlim + 1);
    const int lane = threadIdx.x & 31;
    const int64_t n = d_n_map ? (int64_t)*d_n_map : n_static;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t m0 = blockIdx.x * (int64_t)blockDim.x + (threadIdx.x & ~31); m0 < n; m0 += stride) {
        const int64_t m = m0 + lane;
        int c = 0;
        int32_t f = 0;
        if (m < n) {
            f = map ? map[m] : (int32_t)m;
            double v[9], nn[3];
            load_face(faces, f, v, nn);
            c = face_pairs(faces, f, v, li, nlim, slot, nullptr);
            if (c < 0) {
                latch_status(d_status, VF_ENLIM);
                c = 0;
            }
        }
        int inc = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int t = __shfl_up_sync(0xffffffffu, inc, o);
            if (lane >= o) inc += t;
        }
        const int total = __shfl_sync(0xffffffffu, inc, 31);
        int base = 0;
        if (lane == 31 && total) base = atomicAdd(d_n_pairs, total);
        base = __shfl_sync(0xffffffffu, base, 31);
        const int64_t p0 = (int64_t)base + inc - c;
        if (p0 + c > cap) {
            latch_status(d_status, VF_ECAPACITY);
            atomicMax(d_status + 3, (int32_t)min(p0 + c, (int64_t)0x7fffffff));
        }
        for (int k = 0; k < c; ++k)
            if (p0 + k < cap) pairs[p0 + k] = make_int2(slot[k], f);
    }
}

int pairs_append_impl(const LevelInfo &li, int nlim, const double *faces, int64_t F,
                      const int32_t *map, const int32_t *d_n_map, int2 *pairs, int32_t *d_n_pairs,
                      int64_t cap, int32_t *d_status, cudaStream_t st) {
    // the pair's bin key is the flat int32 index I + B_x (J + B_y K)
    if ((int64_t)li.bins[0] * li.bins[1] * li.bins[2] > 0x7fffffffll)
        return set_error(VF_EARG, "embed: more than 2^31 bins at the finest level (deeper than the pair key allows)");
    const size_t smem = (size_t)kPairThreads * (nlim + 1) * sizeof(int32_t);
    static size_t attr = 0;
    if (smem > attr) {
        cudaFuncSetAttribute(k_pairs_append, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        attr = smem;
    }
    cudaMemsetAsync(d_n_pairs, 0, sizeof(int32_t), st);
    kt_point("memset:n_pairs");
    int64_t g = (F + kPairThreads - 1) / kPairThreads;
    if (g > max_ctas(VF_GRID_PAIRS * 2)) g = max_ctas(VF_GRID_PAIRS * 2);
    k_pairs_append<<<(int)(g < 1 ? 1 : g), kPairThreads, smem, st>>>(li, nlim, faces, map, d_n_map, F, pairs,
                                                                     d_n_pairs, cap, d_status);
    return check_launch("k_pairs");
}

// Bins matched to blocks (pin A4): the voxelizer of level L
// reads the bin of each level-L block only, so the embed groups the pairs by
// level-L BLOCK instead of by bin.  A pair's bin key (I, J, K) is the block
// key; the block is found by descending the forest from the root block
// (I, J, K) >> L through the child links (child ids are parent-first + octant,
// ox + 2 oy + 4 oz, vf_forest.cu) -- no dense B_L^3 map, no hash table.
// Pairs whose bin holds no level-L block are dropped (never read).
// K1: pair -> level-local block u, per-block pair counts, the nonempty blocks
__global__ void __launch_bounds__(256)
    k_pair_blocks(int L, int bx, int by, int3 nb0, const int2 *__restrict__ pairs,
                  const int32_t *__restrict__ d_n_pairs, int64_t cap,
                  const int32_t *__restrict__ level_start, const int32_t *__restrict__ child,
                  int32_t *__restrict__ blk, int32_t *__restrict__ cnt, int32_t *__restrict__ ne,
                  int32_t *__restrict__ d_n_ne) {
    const int64_t n = min((int64_t)*d_n_pairs, cap);
    const int32_t s = level_start[L], n_used = level_start[VF_MAX_LEVELS];
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t key = pairs[p].x;
        const int bi = key % bx, r = key / bx, bj = r % by, bk = r / by;
        const int32_t b = block_of_key(L, bi, bj, bk, nb0, child, n_used);
        int32_t u = -1;
        if (b >= 0) {
            u = b - s;
            if (atomicAdd(&cnt[u], 1) == 0) ne[atomicAdd(d_n_ne, 1)] = u;
        }
        blk[p] = u;
    }
}

struct LoadCnt {
    const int32_t *p;
    __device__ int operator()(int64_t i) const { return p[i]; }
};
struct EmitBase {
    int32_t *base, *cur;
    __device__ void operator()(int64_t i, int, int ex) const {
        base[i] = ex;
        cur[i] = ex;
    }
};

// K3: counting-sort scatter of the face ids into their block's slice
__global__ void __launch_bounds__(256)
    k_pair_scatter(const int2 *__restrict__ pairs, const int32_t *__restrict__ d_n_pairs, int64_t cap,
                   const int32_t *__restrict__ blk, int32_t *__restrict__ cur,
                   int32_t *__restrict__ face_ids) {
    const int64_t n = min((int64_t)*d_n_pairs, cap);
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t u = blk[p];
        if (u >= 0) face_ids[atomicAdd(&cur[u], 1)] = pairs[p].y;
    }
}

int block_bins_impl(const LevelInfo &li, int L, vf_grid *g, const int2 *pairs,
                    const int32_t *d_n_pairs, int64_t cap, const BlockBins &bb, cudaStream_t st) {
    const int3 nb0 = make_int3(li.bins[0] >> L, li.bins[1] >> L, li.bins[2] >> L);
    cudaMemsetAsync(bb.d_n_ne, 0, sizeof(int32_t), st);
    kt_point("memset:n_ne");
    k_pair_blocks<<<max_ctas(8), 256, 0, st>>>(L, li.bins[0], li.bins[1], nb0, pairs, d_n_pairs, cap,
                                               g->d_level_start, g->d_child, bb.blk, bb.cnt, bb.ne,
                                               bb.d_n_ne);
    int rc = check_launch("k_pair_blocks");
    if (rc) return rc;
    // grid bound: the level's blocks <= its bins (coarse levels: a few tiles)
    const int64_t nbound = std::min((int64_t)g->capacity, (int64_t)li.bins[0] * li.bins[1] * li.bins[2]);
    cudaError_t e = scan_launch_fn(LoadCnt{bb.cnt}, EmitBase{bb.base, bb.cur}, nbound,
                                   ScanLevelN{g->d_level_start, L}, bb.d_total, bb.scan_ws, st);
    kt_point("scan_kernel");
    if (e != cudaSuccess) return set_cuda_error(e, "block bins scan");
    k_pair_scatter<<<max_ctas(8), 256, 0, st>>>(pairs, d_n_pairs, cap, bb.blk, bb.cur, bb.face_ids);
    return check_launch("k_pair_scatter");
}

// pair list in face-major order (API compute_bin_pairs)
__global__ void k_pairs_emit(int nlim, const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map,
                             int64_t n_static, const int32_t *__restrict__ slots,
                             const int32_t *__restrict__ slot_cnt, const int32_t *__restrict__ pos,
                             int32_t *__restrict__ pair_bin, int32_t *__restrict__ pair_face,
                             int64_t pair_cap, int32_t *__restrict__ d_status) {
    const int64_t n = d_n_map ? (int64_t)*d_n_map : n_static;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = map ? map[m] : (int32_t)m;
        const int c = slot_cnt[m];
        const int64_t p0 = pos[m];
        for (int k = 0; k < c; ++k) {
            if (p0 + k >= pair_cap) { latch_status(d_status, VF_ECAPACITY); break; }
            pair_bin[p0 + k] = slots[m * nlim + k];
            pair_face[p0 + k] = f;
        }
    }
}

// --------------------------------------------------------------------------
// counting sort

__global__ void k_hist_pairs(const int32_t *__restrict__ pair_bin, const int32_t *__restrict__ d_n,
                             int32_t *__restrict__ counts) {
    const int64_t n = *d_n;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x)
        atomicAdd(&counts[pair_bin[p]], 1);
}

// scatter from slots: counts[] is used as a down-counting cursor and is
// restored by k_bin_sort (counts[b] = offsets[b+1]-offsets[b]).
__global__ void __launch_bounds__(256)
    k_scatter_slots(int nlim, const int32_t *__restrict__ map, const int32_t *__restrict__ d_n_map,
                    int64_t n_static, const int32_t *__restrict__ slots,
                    const int32_t *__restrict__ slot_cnt, const int32_t *__restrict__ offsets,
                    int32_t *__restrict__ counts, int32_t *__restrict__ face_ids,
                    int64_t cap, int32_t *__restrict__ d_status) {
    const int64_t n = d_n_map ? (int64_t)*d_n_map : n_static;
    for (int64_t m = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; m < n;
         m += (int64_t)gridDim.x * blockDim.x) {
        const int32_t f = map ? map[m] : (int32_t)m;
        const int c = slot_cnt[m];
        for (int k = 0; k < c; ++k) {
            const int32_t b = slots[m * nlim + k];
            const int64_t p = (int64_t)offsets[b] + atomicSub(&counts[b], 1) - 1;
            if (p < cap) face_ids[p] = f;
            else latch_status(d_status, VF_ECAPACITY);
        }
    }
}

__global__ void k_scatter_pairs(const int32_t *__restrict__ pair_bin, const int32_t *__restrict__ pair_face,
                                const int32_t *__restrict__ d_n, const int32_t *__restrict__ offsets,
                                int32_t *__restrict__ counts, int32_t *__restrict__ face_ids) {
    const int64_t n = *d_n;
    for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < n;
         p += (int64_t)gridDim.x * blockDim.x) {
        const int32_t b = pair_bin[p];
        const int64_t q = (int64_t)offsets[b] + atomicSub(&counts[b], 1) - 1;
        face_ids[q] = pair_face[p];
    }
}

constexpr int kSmallBin = 24;

// restore counts, sort short bins in place (thread per bin), queue long bins
__global__ void __launch_bounds__(256)
    k_bin_sort_small(int64_t n_bins, const int32_t *__restrict__ offsets,
                     const int32_t *__restrict__ d_total, int32_t *__restrict__ counts,
                     int32_t *__restrict__ face_ids, int32_t *__restrict__ large_list,
                     int32_t *__restrict__ d_n_large) {
    const int64_t total = *d_total;
    for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < n_bins;
         b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t off = offsets[b];
        const int64_t end = (b + 1 < n_bins) ? (int64_t)offsets[b + 1] : total;
        const int cnt = (int)(end - off);
        counts[b] = cnt;
        if (cnt <= 1) continue;
        if (cnt > kSmallBin) {
            const int k = atomicAdd(d_n_large, 1);
            large_list[k] = (int32_t)b;
            continue;
        }
        int32_t a[kSmallBin];
        for (int i = 0; i < cnt; ++i) a[i] = face_ids[off + i];
        for (int i = 1; i < cnt; ++i) {  // insertion sort
            const int32_t x = a[i];
            int j = i - 1;
            while (j >= 0 && a[j] > x) { a[j + 1] = a[j]; --j; }
            a[j + 1] = x;
        }
        for (int i = 0; i < cnt; ++i) face_ids[off + i] = a[i];
    }
}

constexpr int kLargeSmem = 12288;  // ints staged in shared memory

// CTA per long bin: rank sort (face ids within a bin are distinct)
__global__ void __launch_bounds__(256)
    k_bin_sort_large(const int32_t *__restrict__ large_list, const int32_t *__restrict__ d_n_large,
                     const int32_t *__restrict__ offsets, const int32_t *__restrict__ counts,
                     int32_t *__restrict__ face_ids, int32_t *__restrict__ scratch) {
    extern __shared__ int32_t s_ids[];
    const int n_large = *d_n_large;
    for (int w = blockIdx.x; w < n_large; w += gridDim.x) {
        const int32_t b = large_list[w];
        const int64_t off = offsets[b];
        const int cnt = counts[b];
        const bool in_smem = cnt <= kLargeSmem;
        const int32_t *src = in_smem ? s_ids : scratch + off;
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int32_t x = face_ids[off + i];
            if (in_smem) s_ids[i] = x;
            else scratch[off + i] = x;
        }
        __syncthreads();
        if (!in_smem) __threadfence_block();
        for (int i = threadIdx.x; i < cnt; i += blockDim.x) {
            const int32_t x = src[i];
            int r = 0;
            for (int j = 0; j < cnt; ++j) r += (src[j] < x);
            face_ids[off + r] = x;
        }
        __syncthreads();
    }
}

// --------------------------------------------------------------------------
// host side

static inline int grid_for(int64_t n, int threads, int max_ctas) {
    int64_t g = (n + threads - 1) / threads;
    if (g < 1) g = 1;
    if (g > max_ctas) g = max_ctas;
    return (int)g;
}

int launch_indicators(const LevelInfo &li, int mode, const double *faces, int64_t F,
                      uint8_t *out, cudaStream_t st) {
    if (F <= 0) return VF_OK;
    if (mode == 0) {
        int ex = 0;
        const int widen = (frexp(li.dx, &ex) == 0.5) ? 0 : 1;  // 1/dx exact for 2^-k
        k_indicators_1d<<<grid_for((F + 31) / 32, kIndWarps, max_ctas(6)), kIndWarps * 32, 0, st>>>(
            li, 1.0 / li.dx, widen, faces, F, out);
    } else {
        k_indicators<1><<<grid_for(F, 256, max_ctas(8)), 256, 0, st>>>(li, faces, F, out);
    }
    return check_launch("k_indicators");
}

struct LoadU8 {
    const uint8_t *p;
    __device__ int operator()(int64_t i) const { return p[i] ? 1 : 0; }
};
struct EmitCompact {
    int32_t *map;
    __device__ void operator()(int64_t i, int v, int ex) const {
        if (v) map[ex] = (int32_t)i;
    }
};
struct LoadBit {
    const uint16_t *p;
    int L;
    __device__ int operator()(int64_t i) const { return (p[i] >> L) & 1; }
};
struct LoadI32 {
    const int32_t *p;
    __device__ int operator()(int64_t i) const { return p[i]; }
};
struct EmitOffsets {
    int32_t *out;
    __device__ void operator()(int64_t i, int, int ex) const { out[i] = ex; }
};

int launch_compact(const uint8_t *ind, int64_t n, int32_t *map, int32_t *d_count, void *ws,
                   cudaStream_t st) {
    cudaError_t e = scan_launch(LoadU8{ind}, EmitCompact{map}, n, nullptr, d_count, ws, st);
    kt_point("scan_kernel");
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "compact scan");
}

int launch_compact_bits(const uint16_t *bits, int L, int64_t n, int32_t *map, int32_t *d_count,
                        void *ws, cudaStream_t st) {
    cudaError_t e = scan_launch(LoadBit{bits, L}, EmitCompact{map}, n, nullptr, d_count, ws, st);
    kt_point("scan_kernel");
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "compact scan (bits)");
}

int launch_exclusive_scan(const int32_t *in, int64_t n_bound, const int32_t *d_n, int32_t *out,
                          int32_t *d_total, void *ws, cudaStream_t st) {
    cudaError_t e = scan_launch(LoadI32{in}, EmitOffsets{out}, n_bound, d_n, d_total, ws, st);
    kt_point("scan_kernel");
    return e == cudaSuccess ? VF_OK : set_cuda_error(e, "exclusive scan");
}

// workspace layout of one bin build
struct BinsWs {
    uint8_t *ind;        // [F]
    int32_t *slot_cnt;   // [F]
    int32_t *pos;        // [F]
    int32_t *slots;      // [F*nlim]
    int32_t *large;      // [n_bins]
    int32_t *scalars;    // [8]: 0 n_large, 1 n_pairs
    void *scan_ws;       // scan status words
    size_t scan_bytes;
};

static size_t align_up(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t bins_ws_layout(int64_t F, int nlim, int64_t n_bins, char *base, BinsWs *w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        char *p = base ? base + off : nullptr;
        off += align_up(bytes);
        return p;
    };
    const int64_t scan_n = (F * nlim > n_bins ? F * nlim : n_bins) + 1;
    BinsWs t;
    t.ind = (uint8_t *)take((size_t)F + 1);
    t.slot_cnt = (int32_t *)take(sizeof(int32_t) * ((size_t)F + 1));
    t.pos = (int32_t *)take(sizeof(int32_t) * ((size_t)F + 1));
    t.slots = (int32_t *)take(sizeof(int32_t) * ((size_t)F * nlim + 1));
    t.large = (int32_t *)take(sizeof(int32_t) * ((size_t)n_bins + 1));
    t.scalars = (int32_t *)take(sizeof(int32_t) * 8);
    t.scan_bytes = scan_workspace_bytes(scan_n);
    t.scan_ws = take(t.scan_bytes);
    if (w) *w = t;
    return off;
}

size_t bins_workspace_size(int64_t F, int nlim, int64_t n_bins) {
    return bins_ws_layout(F, nlim, n_bins, nullptr, nullptr);
}

// indicators -> compact -> pairs(+hist) -> offsets -> scatter -> sort
int build_bins_impl(const LevelInfo &li, int nlim, const double *faces, int64_t F, int mode,
                    int use_filter, vf_bins *bins, int32_t *d_status, void *ws, size_t ws_bytes,
                    cudaStream_t st, const uint16_t *ind_bits, bool sorted) {
    const int64_t n_bins = (int64_t)li.bins[0] * li.bins[1] * li.bins[2];
    BinsWs w;
    if (bins_ws_layout(F, nlim, n_bins, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "bins workspace too small");
    int rc;
    const int32_t *map = nullptr;
    const int32_t *d_n_map = nullptr;
    if (use_filter && ind_bits && mode == 0) {  // indicators of every level precomputed
        if ((rc = launch_compact_bits(ind_bits, li.level, F, bins->d_map, bins->d_n_map, w.scan_ws, st)))
            return rc;
        map = bins->d_map;
        d_n_map = bins->d_n_map;
    } else if (use_filter) {
        if ((rc = launch_indicators(li, mode, faces, F, w.ind, st))) return rc;
        if ((rc = launch_compact(w.ind, F, bins->d_map, bins->d_n_map, w.scan_ws, st))) return rc;
        map = bins->d_map;
        d_n_map = bins->d_n_map;
    } else {
        // identity map (filter off): still publish a FilterMap for the API
        if ((rc = launch_iota(bins->d_map, F, bins->d_n_map, st))) return rc;
    }
    cudaMemsetAsync(bins->d_counts, 0, sizeof(int32_t) * (size_t)n_bins, st);
    kt_point("memset:bin_counts");
    k_pairs<<<grid_for(F, kPairThreads, max_ctas(VF_GRID_PAIRS * 2)), kPairThreads, 0, st>>>(li, nlim, faces, map, d_n_map, F, w.slots,
                                                         w.slot_cnt, bins->d_counts, d_status);
    if ((rc = check_launch("k_pairs"))) return rc;
    if ((rc = launch_exclusive_scan(bins->d_counts, n_bins, nullptr, bins->d_offsets,
                                    bins->d_n_face_ids, w.scan_ws, st)))
        return rc;
    k_scatter_slots<<<grid_for(F, 256, max_ctas(8)), 256, 0, st>>>(
        nlim, map, d_n_map, F, w.slots, w.slot_cnt, bins->d_offsets, bins->d_counts,
        bins->d_face_ids, bins->face_ids_cap, d_status);
    if ((rc = check_launch("k_scatter_slots"))) return rc;
    // unsorted (embed): the voxelizer tie-breaks on face ids and derives the
    // slice lengths from the offsets, so neither the per-bin order nor the
    // counts (used as scatter cursors) need restoring
    if (!sorted) return VF_OK;
    return sort_bins(n_bins, bins->d_offsets, bins->d_n_face_ids, bins->d_counts, bins->d_face_ids,
                     w.large, w.scalars, w.slots, st);
}

int sort_bins(int64_t n_bins, const int32_t *offsets, const int32_t *d_total, int32_t *counts,
              int32_t *face_ids, int32_t *large, int32_t *scalars, int32_t *scratch,
              cudaStream_t st) {
    cudaMemsetAsync(scalars, 0, sizeof(int32_t), st);
    k_bin_sort_small<<<grid_for(n_bins, 256, max_ctas(16)), 256, 0, st>>>(
        n_bins, offsets, d_total, counts, face_ids, large, scalars);
    int rc = check_launch("k_bin_sort_small");
    if (rc) return rc;
    static bool attr = false;
    if (!attr) {
        cudaFuncSetAttribute(k_bin_sort_large, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)(kLargeSmem * sizeof(int32_t)));
        attr = true;
    }
    k_bin_sort_large<<<max_ctas(2), 256, kLargeSmem * sizeof(int32_t), st>>>(
        large, scalars, offsets, counts, face_ids, scratch);
    return check_launch("k_bin_sort_large");
}

// API: pair list in face-major emission order
int bin_pairs_impl(const LevelInfo &li, int nlim, const double *faces, int64_t F,
                   const int32_t *map, const int32_t *d_n_map, int32_t *pair_bin,
                   int32_t *pair_face, int64_t pair_cap, int32_t *d_n_pairs, int32_t *d_status,
                   void *ws, size_t ws_bytes, cudaStream_t st) {
    BinsWs w;
    if (bins_ws_layout(F, nlim, 1, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "pairs workspace too small");
    k_pairs<<<grid_for(F, kPairThreads, max_ctas(16)), kPairThreads, 0, st>>>(li, nlim, faces, map, d_n_map, F,
                                                         w.slots, w.slot_cnt, nullptr, d_status);
    int rc = check_launch("k_pairs");
    if (rc) return rc;
    if ((rc = launch_exclusive_scan(w.slot_cnt, F, d_n_map, w.pos, d_n_pairs, w.scan_ws, st)))
        return rc;
    k_pairs_emit<<<grid_for(F, 256, max_ctas(8)), 256, 0, st>>>(nlim, map, d_n_map, F, w.slots,
                                                              w.slot_cnt, w.pos, pair_bin,
                                                              pair_face, pair_cap, d_status);
    return check_launch("k_pairs_emit");
}

// API: assemble from a pair list
int assemble_impl(const int32_t *pair_bin, const int32_t *pair_face, const int32_t *d_n_pairs,
                  int64_t pair_cap, int64_t n_bins, int32_t *counts, int32_t *offsets,
                  int32_t *face_ids, void *ws, size_t ws_bytes, cudaStream_t st) {
    BinsWs w;
    if (bins_ws_layout(pair_cap, 1, n_bins, (char *)ws, &w) > ws_bytes)
        return set_error(VF_EARG, "assemble workspace too small");
    // total pairs -> w.scalars[1]
    cudaMemsetAsync(counts, 0, sizeof(int32_t) * (size_t)n_bins, st);
    k_hist_pairs<<<grid_for(pair_cap, 256, max_ctas(8)), 256, 0, st>>>(pair_bin, d_n_pairs, counts);
    int rc = check_launch("k_hist_pairs");
    if (rc) return rc;
    if ((rc = launch_exclusive_scan(counts, n_bins, nullptr, offsets, w.scalars + 1, w.scan_ws, st)))
        return rc;
    k_scatter_pairs<<<grid_for(pair_cap, 256, max_ctas(8)), 256, 0, st>>>(
        pair_bin, pair_face, d_n_pairs, offsets, counts, face_ids);
    if ((rc = check_launch("k_scatter_pairs"))) return rc;
    return sort_bins(n_bins, offsets, w.scalars + 1, counts, face_ids, w.large, w.scalars,
                     w.slots, st);
}

size_t assemble_workspace_size(int64_t pair_cap, int64_t n_bins) {
    return bins_ws_layout(pair_cap, 1, n_bins, nullptr, nullptr);
}

}  // namespace vf
