// vf_io.cu -- host <-> device formats of the end-to-end (serving) path.
//
//   K-pack-idx  face records from an INDEXED mesh (vertices + faces_indexed,
//               the reference TriangleMesh's own fields, geometry.py:65-90):
//               v1 v2 v3 gathered from the vertex table and the unit normal
//               computed as TriangleMesh._face_normals does
//               (geometry.py:114-124: np.cross of the edges from vertex 0,
//               divided by np.linalg.norm along the row) -- 24 B per vertex
//               + 12 B per face cross PCIe instead of the 96-B records.
//   K-lut-sparse  the cut links of a LUT as (flat index, q) pairs in index
//               order: the -1 entries (about 90% of [N_b][27][64]) stay
//               implicit, so the device -> host copy carries only the links.
#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

// numpy's float64 ops, one rounding each: np.cross (a1 b2 - a2 b1, ...),
// norm = sqrt((x*x + y*y) + z*z) (add.reduce over the row, in order), n / norm
__global__ void k_pack_indexed(const double *__restrict__ verts, int64_t V, const int32_t *__restrict__ fidx,
                               int64_t F, double *__restrict__ out, int32_t *__restrict__ status) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < F;
         f += (int64_t)gridDim.x * blockDim.x) {
        double v[9];
        bool bad = false;
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            const int32_t id = __ldg(fidx + 3 * f + c);
            bad |= id < 0 || id >= V;
            const int64_t k = bad ? 0 : id;
#pragma unroll
            for (int d = 0; d < 3; ++d) v[3 * c + d] = __ldg(verts + 3 * k + d);
        }
        const double a0 = VF_DSUB(v[3], v[0]), a1 = VF_DSUB(v[4], v[1]), a2 = VF_DSUB(v[5], v[2]);
        const double b0 = VF_DSUB(v[6], v[0]), b1 = VF_DSUB(v[7], v[1]), b2 = VF_DSUB(v[8], v[2]);
        const double n0 = VF_DSUB(VF_DMUL(a1, b2), VF_DMUL(a2, b1));
        const double n1 = VF_DSUB(VF_DMUL(a2, b0), VF_DMUL(a0, b2));
        const double n2 = VF_DSUB(VF_DMUL(a0, b1), VF_DMUL(a1, b0));
        const double len = __dsqrt_rn(VF_DADD(VF_DADD(VF_DMUL(n0, n0), VF_DMUL(n1, n1)), VF_DMUL(n2, n2)));
        if (bad) latch_status(status, VF_EMESH);       // face index out of range (MeshError)
        else if (len == 0.0) latch_status(status, VF_EMESH);  // zero normal (MeshError)
        double2 *p = reinterpret_cast<double2 *>(out + kFaceStride * f);
        p[0] = make_double2(v[0], v[1]);
        p[1] = make_double2(v[2], v[3]);
        p[2] = make_double2(v[4], v[5]);
        p[3] = make_double2(v[6], v[7]);
        p[4] = make_double2(v[8], VF_DDIV(n0, len));
        p[5] = make_double2(VF_DDIV(n1, len), VF_DDIV(n2, len));
    }
}

// LUT -> sparse: scan over float4 groups of the N_b x 27 x 64 entries
struct LoadPos4 {
    const float4 *p;
    __device__ int operator()(int64_t i) const {
        const float4 v = p[i];
        return (v.x >= 0.0f) + (v.y >= 0.0f) + (v.z >= 0.0f) + (v.w >= 0.0f);
    }
};
struct EmitSparse {
    const float4 *p;
    int32_t *idx;
    float *val;
    int64_t cap;
    __device__ void operator()(int64_t i, int n, int ex) const {
        if (!n) return;
        const float4 v = p[i];
        const float a[4] = {v.x, v.y, v.z, v.w};
        int k = ex;
#pragma unroll
        for (int j = 0; j < 4; ++j)
            if (a[j] >= 0.0f) {
                if (k < cap) {
                    idx[k] = (int32_t)(uint32_t)(4 * i + j);  // unsigned 32-bit flat index
                    val[k] = a[j];
                }
                ++k;
            }
    }
};
// group count from the device-resident N_b (27 x 64 / 4 = 432 float4 per slot)
struct ScanLutN {
    const int32_t *d_n_b;
    int64_t bound;
    __device__ int64_t operator()() const {
        const int64_t n = (int64_t)(*d_n_b) * 432;
        return n < bound ? n : bound;
    }
};

}  // namespace vf

using namespace vf;

extern "C" {

int vf_pack_indexed(const double *verts, int64_t V, const int32_t *faces_idx, int64_t F, double *out,
                    int32_t *d_status, void *stream) {
    if (!verts || !faces_idx || !out || V <= 0 || F <= 0 || V > INT32_MAX)
        return set_error(VF_EARG, "vf_pack_indexed: bad argument");
    int64_t g = (F + 255) / 256;
    if (g > max_ctas(8)) g = max_ctas(8);
    k_pack_indexed<<<(int)g, 256, 0, (cudaStream_t)stream>>>(verts, V, faces_idx, F, out, d_status);
    return check_launch("k_pack_indexed");
}

size_t vf_lut_sparse_workspace_size(int64_t lengths_cap) {
    return scan_workspace_bytes((lengths_cap > 0 ? lengths_cap : 1) * 432);
}

int vf_lut_sparse(const float *lengths, int64_t lengths_cap, const int32_t *d_n_b, int32_t *idx, float *val,
                  int64_t cap, int32_t *d_count, void *ws, size_t ws_bytes, void *stream) {
    if (!lengths || !d_n_b || !idx || !val || !d_count || lengths_cap < 1 || cap < 0 ||
        ws_bytes < vf_lut_sparse_workspace_size(lengths_cap))
        return set_error(VF_EARG, "vf_lut_sparse: bad argument");
    cudaError_t e = scan_launch_fn(LoadPos4{reinterpret_cast<const float4 *>(lengths)},
                                   EmitSparse{reinterpret_cast<const float4 *>(lengths), idx, val, cap},
                                   lengths_cap * 432, ScanLutN{d_n_b, lengths_cap * 432}, d_count, ws,
                                   (cudaStream_t)stream);
    return e == cudaSuccess ? check_launch("k_lut_sparse") : set_cuda_error(e, "vf_lut_sparse");
}

}  // extern "C"
