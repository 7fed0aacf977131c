// vf_common.cuh -- shared device code for the B200 geometry-embedding engine.
//
// Exact FP64 predicates: every floating-point operation that feeds a decision
// (SAT, plane distance, cell/box coordinates) is written with explicit
// round-to-nearest intrinsics (__dadd_rn/__dsub_rn/__dmul_rn/__ddiv_rn) so
// nvcc can never contract into FMA and the association matches the
// reference's numba code (geometry.py:441-500, compiled without contraction)
// operation for operation.  The library is additionally built -fmad=false.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/voxforest_b200.h"

#define VF_DADD(a, b) __dadd_rn((a), (b))
#define VF_DSUB(a, b) __dsub_rn((a), (b))
#define VF_DMUL(a, b) __dmul_rn((a), (b))
#define VF_DDIV(a, b) __ddiv_rn((a), (b))

namespace vf {

constexpr int kFaceStride = 12;  // doubles per face record: v1 v2 v3 n (96 B)
constexpr int kWarp = 32;

// D3Q27 order of lattice.py:19-39 (rest first, antiparallel pairs (2k-1,2k))
// Component d of c_q, packed as 2-bit fields (c + 1) of one 64-bit immediate
// per axis: a shift and a mask, no table -- a runtime-indexed table becomes a
// constant-bank load that serialises over the distinct q of a warp.
__host__ __device__ constexpr __forceinline__ int c27(int q, int d) {
    const uint64_t k = d == 0 ? 0x8889548889549ull : (d == 1 ? 0x220888a1549495ull : 0x20a0a096094955ull);
    return (int)((k >> (2 * q)) & 3u) - 1;
}

// slot of direction (dx,dy,dz) in {-1,0,1}^3: 5-bit fields, one word per dz
__host__ __device__ __forceinline__ int slot_of(int dx, int dy, int dz) {
    const uint64_t w = dz < 0 ? 0x158e16656614ull : (dz == 0 ? 0x71b82013488ull : 0x137e92565e56ull);
    return (int)((w >> (5 * ((dx + 1) + 3 * (dy + 1)))) & 31u);
}

// Bit-parallel 26-neighbour dilation of the SOLID cells.  A block's cells
// are one 64-bit word (bit t = I + 4J + 16K, the finalize solid64 layout);
// the 3x3x3 dilation is separable: D = Dz(Dy(Dx(S))) over the 27 blocks
// around b -- Dx on the 9 block columns (oy, oz), Dy on the 3 planes oz, Dz
// once -- with in-block shifts plus the facing layer of the neighbour block
// (k_boundary; the LBM's simple-cell test).
constexpr uint64_t kI0 = 0x1111111111111111ull, kI3 = 0x8888888888888888ull;
constexpr uint64_t kJ0 = 0x000F000F000F000Full, kJ3 = 0xF000F000F000F000ull;
constexpr uint64_t kK0 = 0x000000000000FFFFull, kK3 = 0xFFFF000000000000ull;

__host__ __device__ __forceinline__ uint64_t dil_x(uint64_t lo, uint64_t c, uint64_t hi) {
    return c | ((c << 1) & ~kI0) | ((c >> 1) & ~kI3) | ((lo & kI3) >> 3) | ((hi & kI0) << 3);
}
__host__ __device__ __forceinline__ uint64_t dil_y(uint64_t lo, uint64_t c, uint64_t hi) {
    return c | ((c << 4) & ~kJ0) | ((c >> 4) & ~kJ3) | ((lo & kJ3) >> 12) | ((hi & kJ0) << 12);
}
__host__ __device__ __forceinline__ uint64_t dil_z(uint64_t lo, uint64_t c, uint64_t hi) {
    return c | (c << 16) | (c >> 16) | ((lo & kK3) >> 48) | ((hi & kK0) << 48);
}

// per-level constants, computed on the host (ldexp => exact dx_L)
struct LevelInfo {
    double dx;       // cell spacing dx_L
    double h;        // block / bin edge 4*dx_L
    double eps;      // eps_slab
    double eps_par;  // EPS_PARALLEL
    double len[3];   // domain lengths
    int cells[3];    // cells per axis at L
    int bins[3];     // bins (= blocks) per axis at L
    int level;
    int shard_rank;  // block-row ownership (multi-GPU), see owns_row
    int shard_count;
    const uint8_t *owner;  // balanced row -> rank map of this level (or null)
};

// owner rank of the level-L block row (j,k) without an owner map:
// interleaved, so neighbouring rows land on different ranks while x-runs stay
// rank-local.  The sharded embed uses the balanced contiguous map instead
// (vf_shard_owner_map): a face then touches the rows of one or two ranks.
__host__ __device__ __forceinline__ int row_owner(int j, int k, int by, int nranks) {
    return nranks <= 1 ? 0 : (int)(((int64_t)j + (int64_t)by * k) % nranks);
}
__host__ __device__ __forceinline__ bool owns_row(const LevelInfo &li, int j, int k) {
    if (li.shard_count <= 1) return true;
#ifdef __CUDA_ARCH__
    if (li.owner) return li.owner[j + (int64_t)li.bins[1] * k] == li.shard_rank;
#endif
    return row_owner(j, k, li.bins[1], li.shard_count) == li.shard_rank;
}

// A2: lattice node / cell centre, one rounding
__device__ __forceinline__ double node_c(int gi, double dx) {
    return VF_DMUL(VF_DADD((double)gi, 0.5), dx);
}

// A7/A17: plane-distance numerator (v0-x).n with fixed association
__device__ __forceinline__ double plane_num(const double *v, const double *n, double x,
                                           double y, double z) {
    return VF_DADD(VF_DMUL(VF_DSUB(v[0], x), n[0]),
                   VF_DADD(VF_DMUL(VF_DSUB(v[1], y), n[1]), VF_DMUL(VF_DSUB(v[2], z), n[2])));
}

// ---------------------------------------------------------------------------
// SAT triangle/AABB overlap, bit-exact port of geometry.py:441-500.
// The predicate is a conjunction of independent tests (plane cut, 15 axis
// gaps); each test is evaluated exactly as the reference evaluates it, and
// because AND is order-free the cheap box-axis comparisons run first.

struct SatFace {
    double v[9];     // v1 v2 v3
    double lo[3];    // per-axis vertex min (== tmin of the box-axis tests)
    double hi[3];    // per-axis vertex max
    double pn[3];    // un-normalised plane normal of _plane_cuts_box
};

__device__ __forceinline__ void sat_face_init(SatFace &f, const double *v) {
#pragma unroll
    for (int k = 0; k < 9; ++k) f.v[k] = v[k];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        f.lo[d] = fmin(fmin(v[d], v[3 + d]), v[6 + d]);
        f.hi[d] = fmax(fmax(v[d], v[3 + d]), v[6 + d]);
    }
    const double v1x = v[0], v1y = v[1], v1z = v[2], v2x = v[3], v2y = v[4], v2z = v[5],
                 v3x = v[6], v3y = v[7], v3z = v[8];
    // geometry.py:444-446
    f.pn[0] = VF_DSUB(VF_DMUL(VF_DSUB(v2y, v1y), VF_DSUB(v3z, v1z)),
                      VF_DMUL(VF_DSUB(v2z, v1z), VF_DSUB(v3y, v1y)));
    f.pn[1] = VF_DSUB(VF_DMUL(VF_DSUB(v2z, v1z), VF_DSUB(v3x, v1x)),
                      VF_DMUL(VF_DSUB(v2x, v1x), VF_DSUB(v3z, v1z)));
    f.pn[2] = VF_DSUB(VF_DMUL(VF_DSUB(v2x, v1x), VF_DSUB(v3y, v1y)),
                      VF_DMUL(VF_DSUB(v2y, v1y), VF_DSUB(v3x, v1x)));
}

// geometry.py:447-454
__device__ __forceinline__ bool sat_plane_cut(const SatFace &f, double mx, double my, double mz,
                                              double Mx, double My, double Mz) {
    const double nx = f.pn[0], ny = f.pn[1], nz = f.pn[2];
    const double v1x = f.v[0], v1y = f.v[1], v1z = f.v[2];
    const double cx = (nx > 0.0) ? VF_DSUB(Mx, mx) : 0.0;
    const double cy = (ny > 0.0) ? VF_DSUB(My, my) : 0.0;
    const double cz = (nz > 0.0) ? VF_DSUB(Mz, mz) : 0.0;
    const double d = VF_DADD(VF_DADD(VF_DMUL(nx, mx), VF_DMUL(ny, my)), VF_DMUL(nz, mz));
    const double d1 = VF_DADD(VF_DADD(VF_DMUL(nx, VF_DSUB(cx, v1x)), VF_DMUL(ny, VF_DSUB(cy, v1y))),
                              VF_DMUL(nz, VF_DSUB(cz, v1z)));
    const double d2 = VF_DADD(
        VF_DADD(VF_DMUL(nx, VF_DSUB(VF_DSUB(VF_DSUB(Mx, mx), cx), v1x)),
                VF_DMUL(ny, VF_DSUB(VF_DSUB(VF_DSUB(My, my), cy), v1y))),
        VF_DMUL(nz, VF_DSUB(VF_DSUB(VF_DSUB(Mz, mz), cz), v1z)));
    return VF_DMUL(VF_DADD(d, d1), VF_DADD(d, d2)) <= 0.0;
}

// geometry.py:457-481 for the edge axes (k = 2,3,4); true = separated
__device__ __forceinline__ bool sat_edge_gap(double ex, double ey, double a1, double b1,
                                             double a2, double b2, double a3, double b3,
                                             double ra, double rb, double Ra, double Rb) {
    const double t1 = VF_DADD(VF_DMUL(a1, ex), VF_DMUL(b1, ey));
    const double t2 = VF_DADD(VF_DMUL(a2, ex), VF_DMUL(b2, ey));
    const double t3 = VF_DADD(VF_DMUL(a3, ex), VF_DMUL(b3, ey));
    const double tmin = fmin(fmin(t1, t2), t3);
    const double tmax = fmax(fmax(t1, t2), t3);
    const double r1 = VF_DADD(VF_DMUL(ra, ex), VF_DMUL(rb, ey));
    const double r2 = VF_DADD(VF_DMUL(Ra, ex), VF_DMUL(rb, ey));
    const double r3 = VF_DADD(VF_DMUL(ra, ex), VF_DMUL(Rb, ey));
    const double r4 = VF_DADD(VF_DMUL(Ra, ex), VF_DMUL(Rb, ey));
    const double rmin = fmin(fmin(r1, r2), fmin(r3, r4));
    const double rmax = fmax(fmax(r1, r2), fmax(r3, r4));
    return (tmax < rmin) || (rmax < tmin);
}

// the three edge axes of one projection plane (a, b) = coordinate pair
__device__ __forceinline__ bool sat_plane_edges_gap(double a1, double b1, double a2, double b2,
                                                    double a3, double b3, double ra, double rb,
                                                    double Ra, double Rb) {
    if (sat_edge_gap(VF_DSUB(b2, b1), VF_DSUB(a1, a2), a1, b1, a2, b2, a3, b3, ra, rb, Ra, Rb))
        return true;
    if (sat_edge_gap(VF_DSUB(b3, b2), VF_DSUB(a2, a3), a1, b1, a2, b2, a3, b3, ra, rb, Ra, Rb))
        return true;
    if (sat_edge_gap(VF_DSUB(b1, b3), VF_DSUB(a3, a1), a1, b1, a2, b2, a3, b3, ra, rb, Ra, Rb))
        return true;
    return false;
}

// box-axis tests: axis 0/1 of each plane reduce to exact comparisons
// (t = v*1.0 + w*0.0 == v up to the sign of zero; r likewise)
__device__ __forceinline__ bool sat_box_axes_overlap(const SatFace &f, double mx, double my,
                                                     double mz, double Mx, double My, double Mz) {
    const double m[3] = {mx, my, mz}, M[3] = {Mx, My, Mz};
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        const double rmin = fmin(m[d], M[d]), rmax = fmax(m[d], M[d]);
        if (f.hi[d] < rmin || rmax < f.lo[d]) return false;
    }
    return true;
}

__device__ __forceinline__ bool sat_exact(const SatFace &f, double mx, double my, double mz,
                                          double Mx, double My, double Mz) {
    if (!sat_box_axes_overlap(f, mx, my, mz, Mx, My, Mz)) return false;
    const double *v = f.v;
    // yz plane (geometry.py:494-496)
    if (sat_plane_edges_gap(v[1], v[2], v[4], v[5], v[7], v[8], my, mz, My, Mz)) return false;
    // xy plane (geometry.py:491-493)
    if (sat_plane_edges_gap(v[0], v[1], v[3], v[4], v[6], v[7], mx, my, Mx, My)) return false;
    // zx plane (geometry.py:497-499)
    if (sat_plane_edges_gap(v[2], v[0], v[5], v[3], v[8], v[6], mz, mx, Mz, Mx)) return false;
    return sat_plane_cut(f, mx, my, mz, Mx, My, Mz);
}

// ---------------------------------------------------------------------------
// FP32 x-row classifier (voxelizer rows, 1D ray indicators).
//
// Decides the SAT of the row box [0, lx] x [y +- eps] x [z +- eps] against a
// face without FP64 where the outcome is certain: 0 = the x-row misses the
// face, 1 = it pierces the face interior, 2 = undecided (run sat_exact).
// The box overlaps the face iff the point (y, z) is within the eps-square of
// the face's yz projection (the other SAT axes follow from the x-extent).
// Edge functions are evaluated relative to v1 with margins
// t_k = tol |e_k| + 4e-6 (ext + dx)^2, tol = 1e-5 (ext + dx) + 6 eps: >= 10x
// the FP32 error of E_k (incl. sliver edges) plus the eps-square reach:
//   E_k < -t_k for some k: the row box misses the triangle by > tol - 2 eps;
//     the exact predicate is false with a gap >> the FP64 rounding of the
//     reference SAT, which therefore rejects;
//   E_k >= t_k for all k, |n_x| >= 1e-3 and the face's x-range inside
//     (1e-6 lx, lx - 1e-6 lx): the row pierces the face interior at a point
//     of the box, every one of the 13 SAT axes has slack >> FP64 rounding, and
//     the reference SAT (geometry.py:441-500) accepts.
struct RowClass {
    float4 yz;   // yz projection of v2 - v1, v3 - v1
    float4 tol;  // per-edge margins t0, t1, t2; w = orientation sign, |w| = 2: no fast accept
};

__device__ __forceinline__ void row_class_init(RowClass &R, const double *v, const double *n,
                                               double xlo, double xhi, double dx, double eps,
                                               double lx) {
    const float a1 = (float)(v[4] - v[1]), b1 = (float)(v[5] - v[2]);
    const float a2 = (float)(v[7] - v[1]), b2 = (float)(v[8] - v[2]);
    const float cr = a1 * b2 - b1 * a2;
    const float ext = fmaxf(fmaxf(fabsf(a1), fabsf(b1)), fmaxf(fabsf(a2), fabsf(b2)));
    const float tol = 1e-5f * (ext + (float)dx) + 6.0f * (float)eps;
    const float ab = 4e-6f * (ext + (float)dx) * (ext + (float)dx);
    const float e1a = a2 - a1, e1b = b2 - b1;
    const float sg = cr >= 0.0f ? 1.0f : -1.0f;
    const double tx = 1e-6 * lx;
    // no fast accept: ill-conditioned x crossing or face near the domain x ends
    const bool acc = fabs(n[0]) >= 1e-3 && xlo > tx && xhi < lx - tx && cr != 0.0f;
    R.yz = make_float4(a1, b1, a2, b2);
    R.tol = make_float4(tol * sqrtf(a1 * a1 + b1 * b1) + ab, tol * sqrtf(e1a * e1a + e1b * e1b) + ab,
                        tol * sqrtf(a2 * a2 + b2 * b2) + ab, acc ? sg : 2.0f * sg);
}

__device__ __forceinline__ void row_class_init(RowClass &R, const SatFace &f, const double *n,
                                               double dx, double eps, double lx) {
    row_class_init(R, f.v, n, f.lo[0], f.hi[0], dx, eps, lx);
}

// (Ry, Rz) = (y - v1_y, z - v1_z) rounded to FP32
__device__ __forceinline__ int row_class(const RowClass &R, float Ry, float Rz) {
    const float4 p = R.yz, t = R.tol;
    const float sg = t.w > 0.0f ? 1.0f : -1.0f;
    const float E0 = sg * (p.x * Rz - p.y * Ry);
    const float E1 = sg * ((p.z - p.x) * (Rz - p.y) - (p.w - p.y) * (Ry - p.x));
    const float E2 = sg * (p.w * Ry - p.z * Rz);
    if (E0 < -t.x || E1 < -t.y || E2 < -t.z) return 0;
    const bool acc = fabsf(t.w) == 1.0f;
    return (acc && E0 >= t.x && E1 >= t.y && E2 >= t.z) ? 1 : 2;
}

// exact SAT of the x-row box (y, z) of the face record f (the classifiers'
// undecided band; rare, so the face is re-read and the SAT set up here)
static __device__ __noinline__ bool row_sat_exact_f(const double *__restrict__ faces, int64_t f,
                                                    double y, double z, double eps, double lx);

// ---------------------------------------------------------------------------
// small helpers

__device__ __forceinline__ void load_face(const double *__restrict__ faces, int64_t f,
                                          double *v, double *n) {
    const double2 *p = reinterpret_cast<const double2 *>(faces + f * kFaceStride);
    double2 a = __ldg(p + 0), b = __ldg(p + 1), c = __ldg(p + 2), d = __ldg(p + 3),
            e = __ldg(p + 4), g = __ldg(p + 5);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = c.x; v[5] = c.y;
    v[6] = d.x; v[7] = d.y; v[8] = e.x;
    n[0] = e.y; n[1] = g.x; n[2] = g.y;
}

__device__ __forceinline__ int warp_sum(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// level-L block with block coordinates (bi, bj, bk), found by descending the
// forest from its root block through the child links (child ids are
// parent-first + octant, ox + 2 oy + 4 oz, vf_forest.cu); -1: no such block.
// (a level dropped on capacity exhaustion leaves child ids >= n_used: no block)
__device__ __forceinline__ int32_t block_of_key(int L, int bi, int bj, int bk, const int3 nb0,
                                                const int32_t *__restrict__ child, int32_t n_used) {
    int32_t b = (bi >> L) + nb0.x * ((bj >> L) + nb0.y * (bk >> L));
    for (int l = L - 1; l >= 0; --l) {
        const int32_t c = child[b];
        if (c < 0 || c >= n_used) return -1;
        b = c + ((bi >> l) & 1) + 2 * ((bj >> l) & 1) + 4 * ((bk >> l) & 1);
    }
    return b;
}

__device__ __forceinline__ void latch_status(int32_t *d_status, int code) {
    if (d_status) atomicMax(d_status, code);
}

static __device__ __noinline__ bool row_sat_exact_f(const double *__restrict__ faces, int64_t f,
                                                    double y, double z, double eps, double lx) {
    double v[9], n[3];
    load_face(faces, f, v, n);
    SatFace sf;
    sat_face_init(sf, v);
    return sat_exact(sf, 0.0, VF_DSUB(y, eps), VF_DSUB(z, eps), lx, VF_DADD(y, eps), VF_DADD(z, eps));
}

}  // namespace vf
