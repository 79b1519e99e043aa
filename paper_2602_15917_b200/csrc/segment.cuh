// segment.cuh -- quantise-and-copy of contiguous segments of x into the code stream (used by the
// run gather and the NEXT-1 row spans): 16-byte loads of x, V codes quantised in registers, 16-byte
// streaming stores, whatever the relative alignment of source and destination.
#pragma once
#include "common.cuh"

namespace roix {

template <typename T>
__host__ __device__ constexpr int gr_v() { return 16 / (int)sizeof(T); }   // elements per 16-byte group

// V consecutive elements starting at element k (0 <= k < V) of the 32 bytes {b0, b1}
template <typename T>
__device__ __forceinline__ uint4 window16(uint4 b0, uint4 b1, uint32_t k) {
    const uint32_t w[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    const uint32_t q = sizeof(T) == 2 ? k >> 1 : k;   // whole-word shift
    uint32_t t[6], u[5];
#pragma unroll
    for (int i = 0; i < 6; i++) t[i] = (q & 2) ? w[i + 2] : w[i];
#pragma unroll
    for (int i = 0; i < 5; i++) u[i] = (q & 1) ? t[i + 1] : t[i];
    if constexpr (sizeof(T) == 2) {
        const uint32_t sh = (k & 1) * 16;
        return make_uint4(__funnelshift_r(u[0], u[1], sh), __funnelshift_r(u[1], u[2], sh),
                          __funnelshift_r(u[2], u[3], sh), __funnelshift_r(u[3], u[4], sh));
    } else {
        return make_uint4(u[0], u[1], u[2], u[3]);
    }
}

template <typename T, int QM>
__device__ __forceinline__ uint32_t code1(T v, const QP &q, uint32_t &err) {
    if constexpr (sizeof(T) == 2) return code_u16_m<QM>(v, q, err);
    else return (uint32_t)code_f32(v, q, err);
}

template <typename T, int QM>
__device__ __forceinline__ uint4 code_group(uint4 v, const QP &q, uint32_t &err) {
    if constexpr (sizeof(T) == 2) {
        return make_uint4(code_pair_u16_m<QM>(v.x, q, err), code_pair_u16_m<QM>(v.y, q, err),
                          code_pair_u16_m<QM>(v.z, q, err), code_pair_u16_m<QM>(v.w, q, err));
    } else {
        return make_uint4((uint32_t)code_f32(__uint_as_float(v.x), q, err), (uint32_t)code_f32(__uint_as_float(v.y), q, err),
                          (uint32_t)code_f32(__uint_as_float(v.z), q, err), (uint32_t)code_f32(__uint_as_float(v.w), q, err));
    }
}






// One warp: codes of x[src0, src0 + len) into out[dst0, dst0 + len); positions >= cap are not
// written.  Scalar head up to a 16-byte boundary of out, then whole groups of V codes -- each from one
// or two aligned 16-byte loads of x (the source misalignment is the same for every group) -- U per
// lane in flight, then a scalar tail.
template <typename T, typename C, int QM, int U>
__device__ __forceinline__ void warp_segment(const T *__restrict__ x, uint64_t src0, C *__restrict__ out,
                                             uint64_t dst0, uint64_t len, uint64_t cap, const QP &q, uint32_t &err) {
    constexpr int V = gr_v<T>();
    static_assert(V == 16 / (int)sizeof(C), "codes and input have the same width");
    const uint32_t lane = lane_id();
    const uint64_t head = min((uint64_t)((V - dst0 % V) % V), len);
    if (lane < head) {
        const uint32_t cd = code1<T, QM>(x[src0 + lane], q, err);
        if (dst0 + lane < cap) out[dst0 + lane] = (C)cd;
    }
    const uint64_t body = (len - head) / V;
    const uint64_t s1 = src0 + head, d1 = dst0 + head;
    const uint32_t k = (uint32_t)(s1 % V);
    const uint4 *xs = reinterpret_cast<const uint4 *>(x) + s1 / V;
    uint4 *od = reinterpret_cast<uint4 *>(out + d1);
    for (uint64_t g0 = 0; g0 < body; g0 += 32 * U) {
        uint4 b0[U], b1[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t g = g0 + lane + 32 * u;
            b0[u] = b1[u] = make_uint4(0, 0, 0, 0);
            if (g < body) {
                b0[u] = __ldcs(xs + g);
                if (k) b1[u] = __ldcs(xs + g + 1);
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t g = g0 + lane + 32 * u;
            if (g >= body) continue;
            const uint4 cv = code_group<T, QM>(window16<T>(b0[u], b1[u], k), q, err);
            const uint64_t p = d1 + g * V;
            if (p + V <= cap) {
                __stcs(od + g, cv);
            } else {
                const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                for (int e = 0; e < V; e++)
                    if (p + e < cap) out[p + e] = (C)(sizeof(C) == 2 ? (cw[e >> 1] >> ((e & 1) * 16)) & 0xffffu : cw[e]);
            }
        }
    }
    const uint64_t t0 = head + body * V;
    if (t0 + lane < len) {
        const uint32_t cd = code1<T, QM>(x[src0 + t0 + lane], q, err);
        if (dst0 + t0 + lane < cap) out[dst0 + t0 + lane] = (C)cd;
    }
}

}  // namespace roix
