// common.cuh -- shared device helpers of libroix (sm_100a).  Product code: shares nothing with oracle/.
#pragma once
#include <atomic>
#include <cstdint>
#include <cuda_runtime.h>

#include "roix.h"

namespace roix {

constexpr uint32_t FULL = 0xffffffffu;

// ------------------------------------------------------------------------------------ error word
__device__ __forceinline__ void set_err(roix_scalars *sc, uint32_t bits) {
    if (bits) atomicOr(&sc->err, bits);
}
__device__ __forceinline__ uint32_t get_err(const roix_scalars *sc) {
    return *((volatile const uint32_t *)&sc->err);
}

// --------------------------------------------------------- ordered-int encoding of fp32 (a0 range)
__host__ __device__ __forceinline__ uint32_t f2ord(float f) {
    uint32_t b;
#ifdef __CUDA_ARCH__
    b = __float_as_uint(f);
#else
    __builtin_memcpy(&b, &f, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
__host__ __device__ __forceinline__ float ord2f(uint32_t o) {
    uint32_t b = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
#ifdef __CUDA_ARCH__
    return __uint_as_float(b);
#else
    float f;
    __builtin_memcpy(&f, &b, 4);
    return f;
#endif
}

// ------------------------------------------------------------------------- a1 quantiser (G-2..G-4)
// code = RNE(x / s): the integer nearest the exact real quotient, ties to the even integer.
//
// Exact path (reading G-4): q = div.rn(x, s) is correctly rounded, and for |x/s| < 2^23 every
// half-integer is representable, so fl(x/s) lands on k+1/2 only when x/s is within half an ulp of
// it; then the sign of the residual x - q*s (one fma rounding, sign-exact) decides.
static __device__ __noinline__ float rne_exact(float x, float s) {
    float q = __fdiv_rn(x, s);
    float c = rintf(q);
    float fl = floorf(q);
    if (q - fl == 0.5f) {
        float r = __fmaf_rn(-q, s, x);
        c = r > 0.0f ? fl + 1.0f : (r < 0.0f ? fl : c);
    }
    return c;
}

// Fast path: q' = x * fl(1/s) is within |q'| * 2^-22.9 of x/s; when q' is farther than |q'| * 2^-22
// from a half-integer, rint(q') already equals RNE(x/s).  Otherwise fall back to rne_exact.
__device__ __forceinline__ float rne_fast(float x, float s, float s_inv) {
    float q = x * s_inv;
    float fr = q - floorf(q);
    if (fabsf(fr - 0.5f) > fabsf(q) * 2.384185791015625e-07f) return rintf(q);
    return rne_exact(x, s);
}

struct QP {
    float s, s_inv;
    uint32_t s_int, magic;
    uint32_t k;                  // log2(s_int) when s_int >= 2 is a power of two, else 0
    uint32_t m_hi, m_lo, m_half; // k >= 1: (0xffff >> k), 2^k - 1, 2^(k-1) - 1 in both halfwords
};
__device__ __forceinline__ QP load_qp(const roix_scalars *sc) {
    QP q;
    q.s = sc->s;
    q.s_inv = sc->s_inv;
    q.s_int = sc->s_int;
    q.magic = sc->s_magic;
    q.k = (q.s_int >= 2 && (q.s_int & (q.s_int - 1)) == 0) ? (uint32_t)(__ffs(q.s_int) - 1) : 0u;
    const uint32_t lanes = 0x00010001u, k = q.k ? q.k : 1u;
    q.m_hi = (0xffffu >> k) * lanes;
    q.m_lo = ((1u << k) - 1u) * lanes;
    q.m_half = ((1u << (k - 1)) - 1u) * lanes;
    return q;
}

// u16 input.  Integer step: d = floor(v / s_int) exactly via umulhi with ceil(2^32 / s_int) (the
// error term v * e / 2^32 < 2^-16 <= 1/s_int), r = v - d s_int, round half to even on (d, r).
__device__ __forceinline__ uint32_t code_u16(uint32_t v, const QP &q, uint32_t &err) {
    if (q.s_int) {
        if (q.s_int == 1) return v;
        uint32_t d = __umulhi(v, q.magic);
        uint32_t r = v - d * q.s_int;
        return d + ((2 * r > q.s_int) | ((2 * r == q.s_int) & (d & 1u)));
    }
    float x = (float)v;
    if (!(x < q.s * 8388608.0f)) err |= ROIX_ERR_RANGE;
    float c = rne_fast(x, q.s, q.s_inv);
    if (c > 65535.0f) err |= ROIX_ERR_RANGE;
    return (uint32_t)c;
}

// Quantiser modes for u16 input, fixed per launch so each kernel body holds one code path:
//   QM_FLOAT: non-integer step (rne_fast); QM_ONE: s = 1 (identity); QM_POW2: s = 2^k; QM_INT: other
//   integer steps (exact division by multiply-high).  fp32 input always uses QM_FLOAT.
enum { QM_FLOAT = 0, QM_ONE = 1, QM_POW2 = 2, QM_INT = 3 };
__device__ __forceinline__ int qmode(const QP &q) {
    return q.s_int == 0 ? QM_FLOAT : q.s_int == 1 ? QM_ONE : q.k ? QM_POW2 : QM_INT;
}

template <int M>
__device__ __forceinline__ uint32_t code_u16_m(uint32_t v, const QP &q, uint32_t &err) {
    if constexpr (M == QM_ONE) return v;
    if constexpr (M == QM_FLOAT) {
        float x = (float)v;
        if (!(x < q.s * 8388608.0f)) err |= ROIX_ERR_RANGE;
        float c = rne_fast(x, q.s, q.s_inv);
        if (c > 65535.0f) err |= ROIX_ERR_RANGE;
        return (uint32_t)c;
    }
    if constexpr (M == QM_POW2) {
        const uint32_t qq = v >> q.k, r = v & ((1u << q.k) - 1u);
        return qq + ((r + (qq & 1u) + (1u << (q.k - 1)) - 1u) >> q.k);
    }
    uint32_t d = __umulhi(v, q.magic);
    uint32_t r = v - d * q.s_int;
    return d + ((2 * r > q.s_int) | ((2 * r == q.s_int) & (d & 1u)));
}

template <int M>
__device__ __forceinline__ uint32_t code_pair_u16_m(uint32_t w, const QP &q, uint32_t &err) {
    if constexpr (M == QM_ONE) return w;
    if constexpr (M == QM_POW2) {
        const uint32_t lanes = 0x00010001u, k = q.k;
        const uint32_t qq = (w >> k) & q.m_hi;
        const uint32_t t = (w & q.m_lo) + (qq & lanes) + q.m_half;
        return qq + ((t >> k) & lanes);
    }
    return code_u16_m<M>(w & 0xffffu, q, err) | (code_u16_m<M>(w >> 16, q, err) << 16);
}

// Two u16 voxels packed in one word (lo, hi) -> two packed codes.  For a power-of-two step s = 2^k
// both halves are rounded at once: v = q 2^k + r rounds up iff r + (q & 1) > 2^(k-1), i.e. iff
// t = r + (q & 1) + 2^(k-1) - 1 >= 2^k; every 16-bit field of t stays below 2^(k+1) <= 2^16, so no
// carry crosses the halves.  Other steps go voxel by voxel through code_u16.
__device__ __forceinline__ uint32_t code_pair_u16(uint32_t w, const QP &q, uint32_t &err) {
    if (q.k) {
        const uint32_t lanes = 0x00010001u, k = q.k;
        const uint32_t qq = (w >> k) & q.m_hi;
        const uint32_t t = (w & q.m_lo) + (qq & lanes) + q.m_half;
        return qq + ((t >> k) & lanes);
    }
    if (q.s_int == 1) return w;
    return code_u16(w & 0xffffu, q, err) | (code_u16(w >> 16, q, err) << 16);
}

// fp32 input (validity range |x| < 2^23 s, G-4; non-finite x fails the same test)
__device__ __forceinline__ int32_t code_f32(float x, const QP &q, uint32_t &err) {
    if (!(fabsf(x) < q.s * 8388608.0f)) {
        err |= (x - x == 0.0f) ? ROIX_ERR_RANGE : ROIX_ERR_NONFINITE;
        return 0;
    }
    return (int32_t)rne_fast(x, q.s, q.s_inv);
}

// --------------------------------------------------------------------------------- small helpers
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
        T o = __shfl_up_sync(FULL, v, d);
        if ((int)lane_id() >= d) v += o;
    }
    return v;
}

// bits: 0..31 -> mask of the low `n` bits (n in 0..32)
__device__ __forceinline__ uint32_t low_mask(uint32_t n) { return n >= 32 ? FULL : ((1u << n) - 1u); }

// Host: cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per device and call site -- the attribute
// is per device, `done` is the call site's bitmask of the devices already set (races are harmless:
// the call is idempotent).
template <typename K>
inline cudaError_t dyn_smem_once(K kern, int bytes, std::atomic<unsigned long long> &done) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    const unsigned long long bit = dev < 64 ? 1ull << dev : 0ull;
    if (bit && (done.load(std::memory_order_relaxed) & bit)) return cudaSuccess;
    if ((e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes)) != cudaSuccess) return e;
    done.fetch_or(bit);
    return cudaSuccess;
}

}  // namespace roix
