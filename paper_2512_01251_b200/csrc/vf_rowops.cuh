// vf_rowops.cuh -- Alg. 5 row-word operations shared by the propagation
// kernels (vf_voxelize.cu pointer jumping, vf_rows.cu sorted rows).
#pragma once

#include "vf_common.cuh"

namespace vf {

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


}  // namespace vf
