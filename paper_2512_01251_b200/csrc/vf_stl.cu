// vf_stl.cu -- GPU ingestion of ASCII STL: the
// reference's parse_stl + _weld + TriangleMesh normals (geometry.py:114-229)
// as data-parallel passes over the text in HBM.
//
//   K-tok     token starts (a non-blank byte after a blank or at 0; blanks are
//             str.split()'s ASCII whitespace) -> compaction scan -> starts
//   K-head    first 'facet' / 'endsolid' token after 'solid' (atomicMin)
//   K-nfacet  facet count = first 21-token block not opened by 'facet'
//   K-facet   per facet: the 20 keywords / numbers checked in token order
//             (the first failing token index wins, as the sequential parser
//             raises at the first error), vertex numbers parsed to the
//             correctly rounded double (Python float()): Clinger's exact
//             fast path, else a few-ulp estimate corrected exactly with
//             big-integer midpoint comparisons
//   K-weld    vertices keyed by rint(v / tol) (np.round), open-addressing hash
//             table, first occurrence = min raw index per key (atomicMin),
//             ids by a scan over first occurrences (ascending raw index =
//             the reference's dict insertion order)
//   K-norm    faces_coord, normals as np.cross / np.linalg.norm (same
//             operation order, no contraction) -> bit-identical arrays
#include <math.h>

#include "vf_common.cuh"
#include "vf_internal.h"
#include "vf_scan.cuh"

namespace vf {

__device__ __forceinline__ bool stl_blank(uint8_t ch) {
    // ASCII whitespace of str.split(): \t \n \v \f \r, \x1c-\x1f, space
    return ch == ' ' || (ch >= 9 && ch <= 13) || (ch >= 0x1c && ch <= 0x1f);
}

__global__ void k_stl_flags(const uint8_t *__restrict__ text, int64_t n, uint8_t *__restrict__ start,
                            int32_t *__restrict__ err) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const uint8_t ch = text[i];
        if (ch >= 0x80) atomicMin(&err[3], 1);  // not an ASCII stream
        start[i] = !stl_blank(ch) && (i == 0 || stl_blank(text[i - 1]));
    }
}

struct LoadU8Flag {
    const uint8_t *p;
    __device__ int operator()(int64_t i) const { return p[i]; }
};
struct EmitStart {
    int64_t *pos;
    __device__ void operator()(int64_t i, int v, int ex) const {
        if (v) pos[ex] = i;
    }
};

// case-insensitive token == word (word lower case)
__device__ __forceinline__ bool tok_is(const uint8_t *text, int64_t n, int64_t p, const char *word) {
    int k = 0;
    for (; word[k]; ++k) {
        if (p + k >= n) return false;
        uint8_t ch = text[p + k];
        if (ch >= 'A' && ch <= 'Z') ch = ch - 'A' + 'a';
        if (ch != (uint8_t)word[k]) return false;
    }
    return p + k >= n || stl_blank(text[p + k]);
}

// first token (index >= 1) that is 'facet' or 'endsolid'
__global__ void k_stl_head(const uint8_t *__restrict__ text, int64_t n, const int64_t *__restrict__ tok,
                           const int32_t *__restrict__ d_ntok, int32_t *__restrict__ head) {
    const int64_t nt = *d_ntok;
    for (int64_t t = 1 + blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
         t += (int64_t)gridDim.x * blockDim.x)
        if (tok_is(text, n, tok[t], "facet") || tok_is(text, n, tok[t], "endsolid"))
            atomicMin(head, (int32_t)t);
}

// facet count: the first block k whose opening token is not 'facet'
__global__ void k_stl_nfacet(const uint8_t *__restrict__ text, int64_t n, const int64_t *__restrict__ tok,
                             const int32_t *__restrict__ d_ntok, const int32_t *__restrict__ head,
                             int32_t *__restrict__ nfacet) {
    const int64_t nt = *d_ntok, h = *head;
    // blocks 0 .. ceil((nt - h) / 21): the last one always opens past the end
    const int64_t nb = nt > h ? (nt - h) / 21 + 2 : 1;
    for (int64_t k = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; k < nb;
         k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t t = h + 21 * k;
        if (t >= nt || !tok_is(text, n, tok[t], "facet")) atomicMin(nfacet, (int32_t)k);
    }
}

// ---------------------------------------------------------------------------
// decimal -> double, correctly rounded (Python float() of a decimal string)
//
// Fast path (Clinger): <= 19 significant digits forming an integer m <= 2^53
// and |E| <= 22: m and 10^|E| are exact doubles, so one IEEE multiply or
// divide is the correctly rounded result.  Otherwise an estimate within a few
// ulps (two scaled multiplies) is corrected exactly: V = D x 10^E is compared
// with the midpoints to its neighbours as big integers (D x 5^E x 2^E vs
// (2M + 1) x 2^(e-1)), ties to even.

// every double midpoint has <= 767 significant digits, so 800 stored digits
// plus a sticky flag decide every rounding exactly (ties included)
constexpr int kMaxDigits = 800;
constexpr int kBigLimbs = 144;  // 4608 bits: D (<= 2658 bits) x 5^|E| x 2^shift

struct Big {
    uint32_t w[kBigLimbs];
    int n;
};

__device__ void big_set(Big &a, uint64_t v) {
    a.n = 0;
    while (v) { a.w[a.n++] = (uint32_t)v; v >>= 32; }
}
__device__ void big_mul_add(Big &a, uint32_t m, uint32_t add) {
    uint64_t carry = add;
    for (int i = 0; i < a.n; ++i) {
        const uint64_t t = (uint64_t)a.w[i] * m + carry;
        a.w[i] = (uint32_t)t;
        carry = t >> 32;
    }
    if (carry && a.n < kBigLimbs) a.w[a.n++] = (uint32_t)carry;
}
__device__ void big_mul_pow5(Big &a, int k) {
    while (k >= 13) { big_mul_add(a, 1220703125u, 0); k -= 13; }  // 5^13
    uint32_t m = 1;
    while (k-- > 0) m *= 5;
    if (m > 1) big_mul_add(a, m, 0);
}
__device__ void big_shl(Big &a, int k) {
    if (a.n == 0 || k <= 0) return;
    const int ws = k >> 5, bs = k & 31;
    int n = a.n + ws + 1;
    if (n > kBigLimbs) n = kBigLimbs;
    for (int i = n - 1; i >= 0; --i) {
        const int j = i - ws;
        uint32_t v = 0;
        if (j >= 0 && j < a.n) v = a.w[j] << bs;
        if (bs && j - 1 >= 0 && j - 1 < a.n) v |= a.w[j - 1] >> (32 - bs);
        a.w[i] = v;
    }
    a.n = n;
    while (a.n > 0 && a.w[a.n - 1] == 0) --a.n;
}
__device__ int big_cmp(const Big &a, const Big &b) {
    if (a.n != b.n) return a.n < b.n ? -1 : 1;
    for (int i = a.n - 1; i >= 0; --i)
        if (a.w[i] != b.w[i]) return a.w[i] < b.w[i] ? -1 : 1;
    return 0;
}

struct DecNum {
    uint8_t d[kMaxDigits];
    int nd;       // significant digits stored
    int E;        // value = D x 10^E (D = the stored digits as an integer)
    bool sticky;  // nonzero digits beyond kMaxDigits
};

// sign of V - (2M + 1) 2^(e2 - 1): V vs the midpoint above M 2^e2
__device__ int cmp_mid(const DecNum &x, uint64_t M, int e2, Big &L, Big &R) {
    big_set(L, 0);
    for (int i = 0; i < x.nd; ++i) {
        if (L.n == 0) big_set(L, x.d[i]);
        else big_mul_add(L, 10, x.d[i]);
    }
    big_set(R, 2 * M + 1);
    int le = x.E, re = e2 - 1;
    if (x.E >= 0) big_mul_pow5(L, x.E);
    else big_mul_pow5(R, -x.E);
    if (le >= re) big_shl(L, le - re);
    else big_shl(R, re - le);
    const int c = big_cmp(L, R);
    return (c == 0 && x.sticky) ? 1 : c;
}

__device__ __forceinline__ void dbl_parts(double c, uint64_t &M, int &e2) {
    const uint64_t b = (uint64_t)__double_as_longlong(c);
    const int be = (int)((b >> 52) & 0x7ff);
    const uint64_t f = b & ((1ull << 52) - 1);
    if (be == 0) { M = f; e2 = -1074; }
    else { M = f | (1ull << 52); e2 = be - 1075; }
}

// correctly rounded |value| of x (x.nd > 0) from an estimate within a few ulps
__device__ double dec_exact(const DecNum &x, double est) {
    Big L, R;
    double c = est;
    if (!(c < INFINITY)) c = 1.7976931348623157e308;
    if (!(c >= 0.0)) c = 0.0;
    for (int it = 0; it < 64; ++it) {
        uint64_t M;
        int e2;
        dbl_parts(c, M, e2);
        const bool odd = M & 1;
        const int up = cmp_mid(x, M, e2, L, R);
        if (up > 0 || (up == 0 && odd)) {
            if (c == 1.7976931348623157e308) return INFINITY;  // past the overflow midpoint
            c = __longlong_as_double(__double_as_longlong(c) + 1);
            continue;
        }
        if (c > 0.0) {
            const double cm = __longlong_as_double(__double_as_longlong(c) - 1);
            uint64_t Mm;
            int em;
            dbl_parts(cm, Mm, em);
            const int dn = cmp_mid(x, Mm, em, L, R);  // V vs midpoint between cm and c
            if (dn < 0 || (dn == 0 && odd)) {
                c = cm;
                continue;
            }
        }
        return c;
    }
    return c;
}

// Python float() of one token: false on a syntax error
__device__ bool stl_float(const uint8_t *text, int64_t n, int64_t p, double &out, DecNum &x) {
    int64_t q = p;
    bool neg = false;
    if (q < n && (text[q] == '+' || text[q] == '-')) {
        neg = text[q] == '-';
        ++q;
    }
    if (tok_is(text, n, q, "infinity") || tok_is(text, n, q, "inf")) {
        out = neg ? -INFINITY : INFINITY;
        return true;
    }
    if (tok_is(text, n, q, "nan")) {
        out = __longlong_as_double(neg ? (long long)0xfff8000000000000ull : 0x7ff8000000000000ll);
        return true;
    }
    // mantissa: digitpart ["." [digitpart]] | "." digitpart; "_" only between digits
    x.nd = 0;
    x.sticky = false;
    int dp = 0;  // value = 0.D x 10^dp before the exponent
    bool any = false, dot = false, prev_digit = false, started = false;
    uint64_t m19 = 0;
    int n19 = 0;
    for (; q < n && !stl_blank(text[q]); ++q) {
        const uint8_t ch = text[q];
        if (ch >= '0' && ch <= '9') {
            any = true;
            prev_digit = true;
            const int dg = ch - '0';
            if (!started && dg == 0) {
                if (dot) --dp;  // leading zero after the point
                continue;
            }
            started = true;
            if (!dot) ++dp;
            if (x.nd < kMaxDigits) x.d[x.nd++] = (uint8_t)dg;
            else if (dg) x.sticky = true;
            if (n19 < 19) { m19 = m19 * 10 + dg; ++n19; }
            continue;
        }
        if (ch == '_') {
            if (!prev_digit || q + 1 >= n || text[q + 1] < '0' || text[q + 1] > '9') return false;
            prev_digit = false;
            continue;
        }
        if (ch == '.' && !dot) {
            if (q > p && text[q - 1] == '_') return false;
            dot = true;
            prev_digit = false;
            continue;
        }
        break;
    }
    if (!any) return false;
    long long e10 = 0;
    if (q < n && (text[q] == 'e' || text[q] == 'E')) {
        ++q;
        bool eneg = false;
        if (q < n && (text[q] == '+' || text[q] == '-')) {
            eneg = text[q] == '-';
            ++q;
        }
        bool edig = false, eprev = false;
        for (; q < n && !stl_blank(text[q]); ++q) {
            const uint8_t ch = text[q];
            if (ch >= '0' && ch <= '9') {
                edig = true;
                eprev = true;
                if (e10 < 100000000) e10 = e10 * 10 + (ch - '0');
            } else if (ch == '_' && eprev && q + 1 < n && text[q + 1] >= '0' && text[q + 1] <= '9') {
                eprev = false;
            } else {
                return false;
            }
        }
        if (!edig) return false;
        if (eneg) e10 = -e10;
    }
    if (q < n && !stl_blank(text[q])) return false;
    while (x.nd > 0 && x.d[x.nd - 1] == 0) --x.nd;  // trailing zeros
    if (x.nd == 0) {
        out = __longlong_as_double(neg ? (long long)0x8000000000000000ull : 0ll);  // signed zero
        return true;
    }
    const long long E = (long long)dp + e10 - x.nd;  // value = D x 10^E
    if (E + x.nd > 310) {
        out = neg ? -INFINITY : INFINITY;
        return true;
    }
    if (E + x.nd < -330) {
        out = __longlong_as_double(neg ? (long long)0x8000000000000000ull : 0ll);  // signed zero
        return true;
    }
    x.E = (int)E;
    // Clinger's fast path (D = the stored digits after trailing zeros)
    uint64_t D = 0;
    if (x.nd <= 19)
        for (int i = 0; i < x.nd; ++i) D = D * 10 + x.d[i];
    if (x.nd <= 19 && !x.sticky && D <= (1ull << 53) && x.E >= -22 && x.E <= 22) {
        const double pw[23] = {1e0,  1e1,  1e2,  1e3,  1e4,  1e5,  1e6,  1e7,  1e8,  1e9,  1e10, 1e11,
                               1e12, 1e13, 1e14, 1e15, 1e16, 1e17, 1e18, 1e19, 1e20, 1e21, 1e22};
        const double m = (double)D;  // exact
        const double v = x.E >= 0 ? __dmul_rn(m, pw[x.E]) : __ddiv_rn(m, pw[-x.E]);
        out = neg ? -v : v;
        return true;
    }
    // estimate from the leading <= 19 digits (a few ulps), then exact correction
    const int Ee = (int)(E + x.nd - n19);  // value ~ m19 x 10^Ee
    double est = (double)m19;
    int k = Ee;
    while (k > 0) { const int s = k > 100 ? 100 : k; est *= pow(10.0, (double)s); k -= s; }
    while (k < 0) { const int s = k < -100 ? -100 : k; est *= pow(10.0, (double)s); k -= s; }
    const double v = dec_exact(x, est);
    out = neg ? __longlong_as_double(__double_as_longlong(v) | (long long)0x8000000000000000ull) : v;
    return true;
}

// ---------------------------------------------------------------------------
// grammar + vertices

// error codes (err[0] = first failing token, err[1] = kind, err[2] = expected word)
enum { STL_E_WORD = 1, STL_E_NUMBER = 2, STL_E_EOF = 3 };

__device__ __forceinline__ void stl_fail(int32_t *err, int64_t t, int kind, int word) {
    // first error in token order; ties impossible (one kind per token)
    const unsigned long long key = ((unsigned long long)t << 16) | ((unsigned)kind << 8) | (unsigned)word;
    atomicMin(reinterpret_cast<unsigned long long *>(err + 4), key);
}

__constant__ char c_words[8][9] = {"solid", "facet", "normal", "outer", "loop", "vertex", "endloop", "endfacet"};

// one thread per (facet, token slot 0..20)
__global__ void k_stl_facets(const uint8_t *__restrict__ text, int64_t n, const int64_t *__restrict__ tok,
                             const int32_t *__restrict__ d_ntok, const int32_t *__restrict__ head,
                             const int32_t *__restrict__ nfacet, double *__restrict__ raw,
                             int32_t *__restrict__ err) {
    // slot layout: 0 facet 1 normal 2-4 f 5 outer 6 loop 7 vertex 8-10 f
    // 11 vertex 12-14 f 15 vertex 16-18 f 19 endloop 20 endfacet
    constexpr int8_t kw[21] = {1, 2, -1, -1, -1, 3, 4, 5, -1, -1, -1, 5, -1, -1, -1, 5, -1, -1, -1, 6, 7};
    const int64_t nt = *d_ntok, h = *head, nf = *nfacet;
    for (int64_t it = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; it < nf * 21;
         it += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = it / 21;
        const int slot = (int)(it - 21 * k);
        const int64_t t = h + it;
        if (t >= nt) {
            stl_fail(err, t, STL_E_EOF, 0);
            continue;
        }
        const int w = kw[slot];
        if (w >= 0) {
            if (!tok_is(text, n, tok[t], c_words[w])) stl_fail(err, t, STL_E_WORD, w);
            continue;
        }
        DecNum dec;
        double v;
        if (!stl_float(text, n, tok[t], v, dec)) {
            stl_fail(err, t, STL_E_NUMBER, 0);
            continue;
        }
        if (slot >= 8) {  // vertex coordinate: slots 8-10, 12-14, 16-18
            const int vi = (slot - 8) / 4, ci = (slot - 8) % 4;
            raw[(k * 3 + vi) * 3 + ci] = v;
        }
    }
}

// trailer: 'endsolid' after the last facet; empty mesh
__global__ void k_stl_trailer(const uint8_t *__restrict__ text, int64_t n, const int64_t *__restrict__ tok,
                              const int32_t *__restrict__ d_ntok, const int32_t *__restrict__ head,
                              const int32_t *__restrict__ nfacet, int32_t *__restrict__ err) {
    const int64_t nt = *d_ntok, h = *head, nf = *nfacet;
    if (nt == 0 || !tok_is(text, n, tok[0], "solid")) {
        stl_fail(err, 0, nt == 0 ? STL_E_EOF : STL_E_WORD, 0);
        return;
    }
    const int64_t t = h + 21 * nf;
    if (t >= nt) stl_fail(err, t, STL_E_EOF, 8);
    else if (!tok_is(text, n, tok[t], "endsolid")) stl_fail(err, t, STL_E_WORD, 8);
}

// ---------------------------------------------------------------------------
// weld (geometry.py:212-225) and the mesh arrays

// key of a raw vertex: rint(v / tol) as int64 (np.round + astype), or the
// value itself (tol <= 0; -0.0 == 0.0 as in the tuple-key dict)
__device__ __forceinline__ void weld_key(const double *v, double tol, long long *k) {
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        if (tol > 0.0) {
            k[d] = (long long)rint(__ddiv_rn(v[d], tol));
        } else {
            const double x = v[d] == 0.0 ? 0.0 : v[d];
            k[d] = __double_as_longlong(x);
        }
    }
}

__device__ __forceinline__ uint64_t hash_key(const long long *k) {
    uint64_t h = 0x9e3779b97f4a7c15ull;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
        h ^= (uint64_t)k[d] + 0x9e3779b97f4a7c15ull + (h << 6) + (h >> 2);
        h *= 0xbf58476d1ce4e5b9ull;
    }
    return h ^ (h >> 31);
}

// insert every raw vertex; slot[s] = a representative raw index (CAS winner),
// first[s] = the minimum raw index with this key (atomicMin), rep[i] = slot
__global__ void k_weld_insert(const double *__restrict__ raw, int64_t nv, double tol,
                              int32_t *__restrict__ slot, int32_t *__restrict__ first,
                              int32_t *__restrict__ rep, int64_t cap) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x) {
        long long k[3];
        weld_key(raw + 3 * i, tol, k);
        uint64_t h = hash_key(k) & (uint64_t)(cap - 1);
        while (true) {
            int32_t cur = slot[h];
            if (cur < 0) {
                const int32_t prev = atomicCAS(&slot[h], -1, (int32_t)i);
                if (prev < 0) cur = (int32_t)i;
                else cur = prev;
            }
            long long kc[3];
            weld_key(raw + 3 * (int64_t)cur, tol, kc);
            if (kc[0] == k[0] && kc[1] == k[1] && kc[2] == k[2]) {
                atomicMin(&first[h], (int32_t)i);
                rep[i] = (int32_t)h;
                break;
            }
            h = (h + 1) & (uint64_t)(cap - 1);
        }
    }
}

struct LoadFirst {
    const int32_t *first, *rep;
    __device__ int operator()(int64_t i) const { return first[rep[i]] == (int32_t)i ? 1 : 0; }
};
struct EmitVertex {
    const int32_t *first, *rep;
    const double *raw;
    int32_t *newid;  // new id of first occurrences (indexed by raw index)
    double *verts;
    __device__ void operator()(int64_t i, int v, int ex) const {
        if (!v) return;
        newid[i] = ex;
        verts[3 * (int64_t)ex + 0] = raw[3 * i + 0];
        verts[3 * (int64_t)ex + 1] = raw[3 * i + 1];
        verts[3 * (int64_t)ex + 2] = raw[3 * i + 2];
    }
};

// faces_indexed, faces_coord and unit normals of TriangleMesh
// (geometry.py:86-90, 114-124): np.cross(v1 - v0, v2 - v0) / norm, where
// norm = sqrt((x*x + y*y) + z*z); a zero norm is a degenerate face (MeshError)
__global__ void k_stl_mesh(const int32_t *__restrict__ first, const int32_t *__restrict__ rep,
                           const int32_t *__restrict__ newid, const double *__restrict__ verts, int64_t nf,
                           int64_t *__restrict__ faces_idx, double *__restrict__ fc,
                           double *__restrict__ nrm, double *__restrict__ packed, int32_t *__restrict__ err) {
    for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf;
         f += (int64_t)gridDim.x * blockDim.x) {
        double v[9];
        for (int c = 0; c < 3; ++c) {
            const int64_t i = 3 * f + c;
            const int32_t id = newid[first[rep[i]]];
            faces_idx[i] = id;
            for (int d = 0; d < 3; ++d) v[3 * c + d] = verts[3 * (int64_t)id + d];
        }
        const double a0 = VF_DSUB(v[3], v[0]), a1 = VF_DSUB(v[4], v[1]), a2 = VF_DSUB(v[5], v[2]);
        const double b0 = VF_DSUB(v[6], v[0]), b1 = VF_DSUB(v[7], v[1]), b2 = VF_DSUB(v[8], v[2]);
        const double n0 = VF_DSUB(VF_DMUL(a1, b2), VF_DMUL(a2, b1));
        const double n1 = VF_DSUB(VF_DMUL(a2, b0), VF_DMUL(a0, b2));
        const double n2 = VF_DSUB(VF_DMUL(a0, b1), VF_DMUL(a1, b0));
        const double len = __dsqrt_rn(VF_DADD(VF_DADD(VF_DMUL(n0, n0), VF_DMUL(n1, n1)), VF_DMUL(n2, n2)));
        if (len == 0.0) atomicMin(&err[3], 2);  // degenerate face
        const double u0 = VF_DDIV(n0, len), u1 = VF_DDIV(n1, len), u2 = VF_DDIV(n2, len);
        for (int k = 0; k < 9; ++k) fc[9 * f + k] = v[k];
        nrm[3 * f + 0] = u0;
        nrm[3 * f + 1] = u1;
        nrm[3 * f + 2] = u2;
        double *p = packed + kFaceStride * f;  // the engine's face record
        for (int k = 0; k < 9; ++k) p[k] = v[k];
        p[9] = u0;
        p[10] = u1;
        p[11] = u2;
    }
}

__global__ void k_extent(const double *__restrict__ raw, int64_t nv, unsigned long long *__restrict__ mm) {
    // per axis min / max of raw vertices (order-preserving integer maps)
    double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
         i += (int64_t)gridDim.x * blockDim.x)
        for (int d = 0; d < 3; ++d) {
            lo[d] = fmin(lo[d], raw[3 * i + d]);
            hi[d] = fmax(hi[d], raw[3 * i + d]);
        }
    auto ord = [](double x) {
        const unsigned long long b = (unsigned long long)__double_as_longlong(x);
        return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
    };
    for (int d = 0; d < 3; ++d) {
        atomicMin(&mm[d], ord(lo[d]));
        atomicMax(&mm[3 + d], ord(hi[d]));
    }
}

}  // namespace vf

using namespace vf;

// ---- host side -------------------------------------------------------------

struct StlWs {
    uint8_t *flags;     // [n]
    int64_t *tok;       // [n/2 + 2] token start offsets
    int32_t *scal;      // 0 n_tok, 1 head, 2 n_facet, 3 ascii/degenerate, 4-5 first error key
    unsigned long long *mm;  // [6] extent (ordered ints)
    double *raw;        // [max facets * 9]
    void *scan_ws;
    int64_t max_tok, max_facets;
};

static size_t al2(size_t x) { return (x + 255) & ~(size_t)255; }

static size_t stl_layout(int64_t n, char *base, StlWs *w) {
    size_t off = 0;
    auto take = [&](size_t b) { char *p = base ? base + off : nullptr; off += al2(b); return (void *)p; };
    StlWs t;
    t.max_tok = n / 2 + 2;
    t.max_facets = t.max_tok / 21 + 1;
    t.flags = (uint8_t *)take((size_t)n + 1);
    t.tok = (int64_t *)take(sizeof(int64_t) * (size_t)t.max_tok);
    t.scal = (int32_t *)take(256);
    t.mm = (unsigned long long *)take(6 * sizeof(unsigned long long));
    t.raw = (double *)take(sizeof(double) * 9 * (size_t)t.max_facets);
    t.scan_ws = take(scan_workspace_bytes(n + 1));
    if (w) *w = t;
    return off;
}

extern "C" {

size_t vf_stl_workspace_size(int64_t n_bytes) { return n_bytes < 0 ? 0 : stl_layout(n_bytes, nullptr, nullptr); }

// tokenize + grammar + numbers (synchronizes): info[0] n_facets, info[1]
// error kind (0 ok, 1 expected word, 2 bad number, 3 end of file, 4 not
// ASCII), info[2] failing token index, info[3] expected-word code, info[4]
// head token, info[5] n_tokens; extent[6] = per-axis min, max of the raw
// vertices; *tok_off = byte offset of the failing token (or -1)
int vf_stl_scan(const uint8_t *d_text, int64_t n, void *ws, size_t ws_bytes, int64_t *info,
                double *extent, int64_t *tok_off, void *stream) {
    if (!d_text || n < 0 || !info || !extent || !tok_off) return set_error(VF_EARG, "vf_stl_scan: bad argument");
    StlWs w;
    if (stl_layout(n, (char *)ws, &w) > ws_bytes) return set_error(VF_EARG, "vf_stl_scan: workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    const int32_t init[6] = {0, 0x7fffffff, 0x7fffffff, 0x7fffffff, -1, -1};
    cudaMemcpyAsync(w.scal, init, sizeof(init), cudaMemcpyHostToDevice, st);
    const unsigned long long mm0[6] = {~0ull, ~0ull, ~0ull, 0ull, 0ull, 0ull};
    cudaMemcpyAsync(w.mm, mm0, sizeof(mm0), cudaMemcpyHostToDevice, st);
    int64_t g = (n + 255) / 256;
    if (g > max_ctas(8)) g = max_ctas(8);
    if (g < 1) g = 1;
    if (n > 0) {
        k_stl_flags<<<(int)g, 256, 0, st>>>(d_text, n, w.flags, w.scal);
        cudaError_t e = scan_launch(LoadU8Flag{w.flags}, EmitStart{w.tok}, n, nullptr, w.scal, w.scan_ws, st);
        if (e != cudaSuccess) return set_cuda_error(e, "stl token scan");
    }
    k_stl_head<<<max_ctas(4), 256, 0, st>>>(d_text, n, w.tok, w.scal, w.scal + 1);
    // head = n_tok when no facet / endsolid token: fixed up in k_stl_nfacet's view
    int32_t h_scal[6];
    cudaMemcpyAsync(h_scal, w.scal, sizeof(h_scal), cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return set_cuda_error(e, "vf_stl_scan");
    const int64_t nt = h_scal[0];
    const int64_t head = h_scal[1] == 0x7fffffff ? nt : h_scal[1];
    cudaMemcpyAsync(w.scal + 1, &head, sizeof(int32_t), cudaMemcpyHostToDevice, st);
    k_stl_nfacet<<<max_ctas(4), 256, 0, st>>>(d_text, n, w.tok, w.scal, w.scal + 1, w.scal + 2);
    k_stl_trailer<<<1, 1, 0, st>>>(d_text, n, w.tok, w.scal, w.scal + 1, w.scal + 2, w.scal);
    int32_t nf32 = 0;
    cudaMemcpyAsync(&nf32, w.scal + 2, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return set_cuda_error(e, "vf_stl_scan");
    const int64_t nf = nf32 == 0x7fffffff ? 0 : nf32;
    if (nf > 0) {
        int64_t g2 = (nf * 21 + 127) / 128;
        if (g2 > max_ctas(8)) g2 = max_ctas(8);
        k_stl_facets<<<(int)g2, 128, 0, st>>>(d_text, n, w.tok, w.scal, w.scal + 1, w.scal + 2, w.raw, w.scal);
        int64_t g3 = (nf * 3 + 255) / 256;
        if (g3 > max_ctas(8)) g3 = max_ctas(8);
        k_extent<<<(int)g3, 256, 0, st>>>(w.raw, nf * 3, w.mm);
    }
    int32_t h2[6];
    unsigned long long hm[6];
    cudaMemcpyAsync(h2, w.scal, sizeof(h2), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(hm, w.mm, sizeof(hm), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return set_cuda_error(e, "vf_stl_scan");
    info[0] = nf;
    info[1] = 0;
    info[2] = -1;
    info[3] = -1;
    info[4] = head;
    info[5] = nt;
    *tok_off = -1;
    const unsigned long long key = ((unsigned long long)(uint32_t)h2[5] << 32) | (uint32_t)h2[4];
    if (h2[3] == 1) {
        info[1] = 4;  // not ASCII (decode fails before any parsing)
    } else if (key != ~0ull) {
        info[2] = (int64_t)(key >> 16);
        info[1] = (int64_t)((key >> 8) & 0xff);
        info[3] = (int64_t)(key & 0xff);
        if (info[2] < nt) cudaMemcpy(tok_off, w.tok + info[2], sizeof(int64_t), cudaMemcpyDeviceToHost);
    }
    auto unord = [](unsigned long long u) {
        const unsigned long long b = (u >> 63) ? (u & 0x7fffffffffffffffull) : ~u;
        double d;
        memcpy(&d, &b, sizeof(d));
        return d;
    };
    for (int d = 0; d < 6; ++d) extent[d] = unord(hm[d]);
    return VF_OK;
}

// weld + mesh arrays from the scanned raw vertices (synchronizes once for
// the vertex count).  Outputs (device, caller-allocated for nf facets):
// d_verts [3 nf][3] (first n_verts rows used), d_faces [nf][3] int64,
// d_fc [nf][9], d_nrm [nf][3], d_packed [nf][12] (engine face records).
// scratch: vf_stl_weld_workspace_size(nf) bytes.
size_t vf_stl_weld_workspace_size(int64_t nf) {
    int64_t cap = 1;
    while (cap < 6 * nf + 2) cap <<= 1;
    return al2(sizeof(int32_t) * (size_t)cap) * 2 + al2(sizeof(int32_t) * (size_t)(3 * nf + 1)) * 2 +
           al2(scan_workspace_bytes(3 * nf + 1)) + 256;
}

int vf_stl_build(const uint8_t *d_text, int64_t n, void *ws, size_t ws_bytes, int64_t nf, double tol,
                 void *weld_ws, size_t weld_bytes, double *d_verts, int64_t *d_faces, double *d_fc,
                 double *d_nrm, double *d_packed, int64_t *n_verts, int32_t *degenerate, void *stream) {
    if (!d_text || nf <= 0 || !d_verts || !d_faces || !d_fc || !d_nrm || !d_packed || !n_verts || !degenerate)
        return set_error(VF_EARG, "vf_stl_build: bad argument");
    StlWs w;
    if (stl_layout(n, (char *)ws, &w) > ws_bytes || weld_bytes < vf_stl_weld_workspace_size(nf))
        return set_error(VF_EARG, "vf_stl_build: workspace too small");
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t nv = 3 * nf;
    int64_t cap = 1;
    while (cap < 2 * nv + 2) cap <<= 1;
    char *b = (char *)weld_ws;
    int32_t *slot = (int32_t *)b;
    b += al2(sizeof(int32_t) * (size_t)cap);
    int32_t *first = (int32_t *)b;
    b += al2(sizeof(int32_t) * (size_t)cap);
    int32_t *rep = (int32_t *)b;
    b += al2(sizeof(int32_t) * (size_t)(nv + 1));
    int32_t *newid = (int32_t *)b;
    b += al2(sizeof(int32_t) * (size_t)(nv + 1));
    void *scan_ws = b;
    b += al2(scan_workspace_bytes(nv + 1));
    int32_t *cnt = (int32_t *)b;
    cudaMemsetAsync(slot, 0xff, sizeof(int32_t) * (size_t)cap, st);
    cudaMemsetAsync(first, 0x7f, sizeof(int32_t) * (size_t)cap, st);
    cudaMemsetAsync(w.scal + 3, 0x7f, sizeof(int32_t), st);
    int64_t g = (nv + 255) / 256;
    if (g > max_ctas(8)) g = max_ctas(8);
    k_weld_insert<<<(int)g, 256, 0, st>>>(w.raw, nv, tol, slot, first, rep, cap);
    cudaError_t e = scan_launch(LoadFirst{first, rep}, EmitVertex{first, rep, w.raw, newid, d_verts}, nv,
                                nullptr, cnt, scan_ws, st);
    if (e != cudaSuccess) return set_cuda_error(e, "stl weld scan");
    int64_t g2 = (nf + 255) / 256;
    if (g2 > max_ctas(8)) g2 = max_ctas(8);
    k_stl_mesh<<<(int)g2, 256, 0, st>>>(first, rep, newid, d_verts, nf, d_faces, d_fc, d_nrm, d_packed,
                                        w.scal);
    int32_t h[2];
    cudaMemcpyAsync(&h[0], cnt, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(&h[1], w.scal + 3, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
    if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return set_cuda_error(e, "vf_stl_build");
    *n_verts = h[0];
    *degenerate = h[1] == 2;
    return check_launch("vf_stl_build");
}

}  // extern "C"
