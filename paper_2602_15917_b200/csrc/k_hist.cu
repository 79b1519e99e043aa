// k_hist.cu -- a2 HISTOGRAM ("based on intensity distribution") and the standalone
// a1 QUANTISE pass (BJ north_star).
//
// u16: shared-memory privatised counters.  A CTA keeps uint32 counters for the value window
// [0, 16384) (64 KiB, two CTAs per SM, 32 warps each -- measured on B200: 4.6 TB/s of input for
// CT-like value distributions); values >= 16384 go straight to the global uint64 bins, which keeps
// the result exact for every input while the common 10..14-bit CT range stays on chip.
// fp32: 256 normalised-intensity bins (needs the edges of roix_resolve).
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace roix {

constexpr int HWIN = 16384;

__device__ __forceinline__ void hist_add(uint32_t *sh, uint64_t *gh, uint32_t v) {
    if (v < (uint32_t)HWIN) atomicAdd(&sh[v], 1u);
    else atomicAdd((unsigned long long *)&gh[v], 1ull);
}

// the 8 values of a 16-byte group: unconditional shared adds when all of them are inside the window
// (one test per group instead of a branch per value -- the kernel is bound by instruction issue)
__device__ __forceinline__ void hist_add8(uint32_t *sh, uint64_t *gh, uint4 a) {
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
    if (((a.x | a.y | a.z | a.w) & 0xC000C000u) == 0) {   // HWIN = 16384: no value has bit 14 or 15
#pragma unroll
        for (int k = 0; k < 4; k++) {
            atomicAdd(&sh[w[k] & 0xffffu], 1u);
            atomicAdd(&sh[w[k] >> 16], 1u);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            hist_add(sh, gh, w[k] & 0xffffu);
            hist_add(sh, gh, w[k] >> 16);
        }
    }
}

__global__ void __launch_bounds__(1024, 2) k_hist_u16(const uint16_t *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                       uint64_t *gh) {
    extern __shared__ uint32_t sh[];
    if (get_err(sc)) return;
    for (int i = threadIdx.x; i < HWIN; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint4 *x8 = reinterpret_cast<const uint4 *>(x);
    const uint64_t n8 = n / 8, stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + stride < n8; i += 2 * stride) {
        const uint4 a = __ldcs(x8 + i), b = __ldcs(x8 + i + stride);
        hist_add8(sh, gh, a);
        hist_add8(sh, gh, b);
    }
    for (; i < n8; i += stride) hist_add8(sh, gh, __ldcs(x8 + i));
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) hist_add(sh, gh, x[n8 * 8 + threadIdx.x]);
    __syncthreads();
    for (int b = threadIdx.x; b < HWIN; b += blockDim.x) {
        uint32_t c = sh[b];
        if (c) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)c);
    }
}

// Lane-banked replicated window.  The u16 kernel is bound by the shared-memory pipe, not by HBM, when
// the values spread over a few hundred bins (C4 / C5 backgrounds): the 32 lanes of one atomic
// instruction hit random banks, and the instruction takes as many wavefronts as its busiest bank
// (3.2 on average at C5).  Each CTA therefore also keeps RW bins [lo, lo + RW) -- around the mode of
// its first 16-byte groups -- with one counter per lane: value v in the window is counted at
// RBASE + 32 (v - lo) + lane, i.e. in the lane's own bank, so in-window lanes never conflict.  The
// window is only a second privatised copy: every value is counted exactly once, in one of the
// windows or in the global bins, and the flush adds all of them.
constexpr int RW = 384;
constexpr int RBASE = HWIN;   // word offset of the replicated window (a multiple of 32)

__device__ __forceinline__ void hist_add_rw(uint32_t *sh, uint64_t *gh, uint32_t v, uint32_t lo, uint32_t lb) {
    if (v - lo < (uint32_t)RW) atomicAdd(&sh[lb + 32u * v], 1u);
    else hist_add(sh, gh, v);
}

// lb = RBASE + lane - 32 lo (mod 2^32): the slot of value v in the lane's column is lb + 32 v
__device__ __forceinline__ void hist_add8_rw(uint32_t *sh, uint64_t *gh, uint4 a, uint32_t lo, uint32_t lb) {
    const uint32_t w[4] = {a.x, a.y, a.z, a.w};
    if (((a.x | a.y | a.z | a.w) & 0xC000C000u) == 0) {   // every value inside the 16 K window
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const uint32_t v0 = w[k] & 0xffffu, v1 = w[k] >> 16;
            atomicAdd(&sh[v0 - lo < (uint32_t)RW ? lb + 32u * v0 : v0], 1u);
            atomicAdd(&sh[v1 - lo < (uint32_t)RW ? lb + 32u * v1 : v1], 1u);
        }
    } else {
#pragma unroll
        for (int k = 0; k < 4; k++) {
            hist_add_rw(sh, gh, w[k] & 0xffffu, lo, lb);
            hist_add_rw(sh, gh, w[k] >> 16, lo, lb);
        }
    }
}

__global__ void __launch_bounds__(1024, 2) k_hist_u16_rw(const uint16_t *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                          uint64_t *gh) {
    extern __shared__ uint32_t sh[];
    __shared__ uint32_t best[32];
    if (get_err(sc)) return;
    for (int i = threadIdx.x; i < HWIN + 32 * RW; i += blockDim.x) sh[i] = 0;
    __syncthreads();
    const uint4 *x8 = reinterpret_cast<const uint4 *>(x);
    const uint64_t n8 = n / 8, stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // the CTA's first groups go to the plain window; their densest 16-bin bucket centres the window
    if (i < n8) hist_add8(sh, gh, __ldcs(x8 + i));
    i += stride;
    __syncthreads();
    uint32_t s = 0;
    for (int b = 0; b < 16; b++) s += sh[16 * threadIdx.x + b];   // blockDim = 1024: buckets cover HWIN
    uint32_t key = __reduce_max_sync(FULL, (s << 10) | threadIdx.x);   // s <= 8192 (1024 groups x 8)
    if (lane_id() == 0) best[threadIdx.x >> 5] = key;
    __syncthreads();
    key = best[lane_id()];
    key = __reduce_max_sync(FULL, key);
    const uint32_t centre = 16u * (key & 1023u) + 8u;
    const uint32_t lo = centre > (uint32_t)RW / 2 ? centre - RW / 2 : 0u;
    const uint32_t lb = (uint32_t)RBASE + lane_id() - 32u * lo;
    for (; i + stride < n8; i += 2 * stride) {
        const uint4 a = __ldcs(x8 + i), b = __ldcs(x8 + i + stride);
        hist_add8_rw(sh, gh, a, lo, lb);
        hist_add8_rw(sh, gh, b, lo, lb);
    }
    for (; i < n8; i += stride) hist_add8_rw(sh, gh, __ldcs(x8 + i), lo, lb);
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) hist_add(sh, gh, x[n8 * 8 + threadIdx.x]);
    __syncthreads();
    for (int b = threadIdx.x; b < HWIN; b += blockDim.x) {
        const uint32_t c = sh[b];
        if (c) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)c);
    }
    for (int r = threadIdx.x; r < RW; r += blockDim.x) {
        uint32_t c = 0;
        for (int l = 0; l < 32; l++) c += sh[RBASE + 32 * r + ((l + r) & 31)];   // rotated: no bank conflict
        if (c) atomicAdd((unsigned long long *)&gh[lo + r], (unsigned long long)c);
    }
}

// NEXT-3 per-frame histograms (uint16 frame stacks): frame z = voxels [z A, (z + 1) A) into
// gh + z * 65536, with the same privatised window as k_hist_u16.  Persistent: CTA c owns the contiguous
// range [c n / G, (c + 1) n / G) of the stack (balanced whatever the frame count) and walks it frame
// segment by frame segment, flushing its window into the segment's frame histogram; segments need not
// start on a 16-byte boundary (head and tail voxel by voxel).
__global__ void __launch_bounds__(1024, 2) k_hist_u16_frames(const uint16_t *__restrict__ x, uint64_t n, uint64_t A,
                                                              roix_scalars *sc, uint64_t *gh_all) {
    extern __shared__ uint32_t sh[];
    if (get_err(sc)) return;
    const uint64_t r0 = n * blockIdx.x / gridDim.x, r1 = n * (blockIdx.x + 1) / gridDim.x;
    const uint4 *x8 = reinterpret_cast<const uint4 *>(x);
    for (uint64_t s = r0; s < r1;) {
        const uint64_t z = s / A, e = min(r1, (z + 1) * A);
        uint64_t *gh = gh_all + z * 65536;
        for (int i = threadIdx.x; i < HWIN; i += blockDim.x) sh[i] = 0;
        __syncthreads();
        const uint64_t a = min(e, (uint64_t)((s + 7) & ~7ull)), e8 = max(a, (uint64_t)(e & ~7ull));
        if (threadIdx.x < a - s) hist_add(sh, gh, x[s + threadIdx.x]);
        if (threadIdx.x < e - e8) hist_add(sh, gh, x[e8 + threadIdx.x]);
        uint64_t i = a / 8 + threadIdx.x;
        const uint64_t i1 = e8 / 8;
        for (; i + blockDim.x < i1; i += 2 * blockDim.x) {
            const uint4 u = __ldcs(x8 + i), v = __ldcs(x8 + i + blockDim.x);
            hist_add8(sh, gh, u);
            hist_add8(sh, gh, v);
        }
        if (i < i1) hist_add8(sh, gh, __ldcs(x8 + i));
        __syncthreads();
        for (int b = threadIdx.x; b < HWIN; b += blockDim.x) {
            const uint32_t c = sh[b];
            if (c) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)c);
        }
        __syncthreads();
        s = e;
    }
}

// norm8 of a finite fp32 value from the edges table e[0..256] (e[0] = -inf, e[256] = +inf):
// norm8(x) = #{k >= 1 : x >= e[k]} -- an estimate from x * 255 / I_max corrected against the edges.
// x * fl(255 / I_max) is within ~3e-5 of the exact 255 x / I_max for x <= I_max, so the estimate is
// within one bin of norm8(x) and one correction in each direction is exact.  `exact_est` is false
// only for a subnormal I_max (255 / I_max overflows); the edges are then walked.
__device__ __forceinline__ int norm8_edges(float x, float scale, const float *e, bool exact_est) {
    const float t = fminf(fmaxf(x * scale + 0.5f, 0.0f), 255.0f);   // NaN -> 0 (flagged by the caller)
    int k = __float2int_rz(t);
    if (exact_est) {
        // t is within ~1e-4 of the exact 255 x / I_max + 1/2 (x <= I_max); away from an integer the
        // estimate is the bin, next to one the edges decide
        const float fr = t - (float)k;
        if (fr < 1e-3f || fr > 0.999f) {
            k = min(k + (x >= e[k + 1]), 255);   // (x = +inf would step past 255)
            k -= (x < e[k]);
        }
    } else {
        while (k < 255 && x >= e[k + 1]) k++;
        while (k > 0 && x < e[k]) k--;
    }
    return k;
}

// 256 bins x 32 lane slots: lane l increments slot l of its bin, so the lanes of a warp never hit
// the same shared-memory word or bank (CT volumes put most voxels into a few normalised bins -- air,
// one material -- which would otherwise serialise 32-way on one counter).
__global__ void __launch_bounds__(512, 3) k_hist_f32(const float *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                  uint64_t *gh) {
    __shared__ uint32_t sh[256 * 32];
    __shared__ float e[257];
    if (get_err(sc)) return;
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) sh[i] = 0;
    for (int i = threadIdx.x; i < 256; i += blockDim.x) e[i] = i == 0 ? -INFINITY : sc->edges[i];
    if (threadIdx.x == 0) e[256] = INFINITY;
    const float scale = 255.0f / sc->i_max;
    const bool ex = scale <= 1e30f;
    __syncthreads();
    uint32_t *my = sh + lane_id();
    bool bad = false;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    const uint64_t n4 = n / 4, stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (ex && i + stride < n4) {
        // branch-free body: a non-finite voxel only sets the (sticky, fatal) error bit; its count
        // lands in a clamped bin of a histogram that is then discarded.  The next pair of loads is
        // issued before the current pair is binned.
        float4 a = __ldcs(x4 + i), b = __ldcs(x4 + i + stride);
        while (true) {
            const uint64_t in = i + 2 * stride;
            const bool more = in + stride < n4;
            float4 na = a, nb = b;
            if (more) {
                na = __ldcs(x4 + in);
                nb = __ldcs(x4 + in + stride);
            }
            float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
            for (int k = 0; k < 8; k++) {
                bad |= !(fabsf(v[k]) <= FLT_MAX);
                atomicAdd(my + 32 * norm8_edges(v[k], scale, e, true), 1u);
            }
            i = in;
            if (!more) break;
            a = na;
            b = nb;
        }
    }
    for (; i + stride < n4; i += 2 * stride) {
        float4 a = __ldcs(x4 + i), b = __ldcs(x4 + i + stride);
        float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
#pragma unroll
        for (int k = 0; k < 8; k++) {
            if (fabsf(v[k]) <= FLT_MAX) atomicAdd(my + 32 * norm8_edges(v[k], scale, e, ex), 1u);
            else bad = true;
        }
    }
    for (; i < n4; i += stride) {
        float4 a = __ldcs(x4 + i);
        float v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            if (fabsf(v[k]) <= FLT_MAX) atomicAdd(my + 32 * norm8_edges(v[k], scale, e, ex), 1u);
            else bad = true;
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        float v = x[n4 * 4 + threadIdx.x];
        if (fabsf(v) <= FLT_MAX) atomicAdd(my + 32 * norm8_edges(v, scale, e, ex), 1u);
        else bad = true;
    }
    if (bad) set_err(sc, ROIX_ERR_NONFINITE);
    __syncthreads();
    // bin b = warp-sum of its 32 slots
    for (int b = threadIdx.x >> 5; b < 256; b += blockDim.x >> 5) {
        const uint32_t c = __reduce_add_sync(FULL, sh[b * 32 + lane_id()]);
        if (lane_id() == 0 && c) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)c);
    }
}

// ---------------------------------------------------------------------------- a1 standalone pass
__global__ void __launch_bounds__(512) k_quantize_u16(const uint16_t *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                      uint16_t *__restrict__ codes) {
    if (get_err(sc)) return;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t n8 = n / 8, stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += stride) {
        uint4 a = __ldcs(reinterpret_cast<const uint4 *>(x) + i);
        uint32_t w[4] = {a.x, a.y, a.z, a.w}, o[4];
#pragma unroll
        for (int k = 0; k < 4; k++) o[k] = code_pair_u16(w[k], q, err);
        __stcs(reinterpret_cast<uint4 *>(codes) + i, make_uint4(o[0], o[1], o[2], o[3]));
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 7)) {
        uint64_t j = n8 * 8 + threadIdx.x;
        codes[j] = (uint16_t)code_u16(x[j], q, err);
    }
    if (err) set_err(sc, err);
}

__global__ void __launch_bounds__(512) k_quantize_f32(const float *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                      int32_t *__restrict__ codes) {
    if (get_err(sc)) return;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t n4 = n / 4, stride = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
        float4 a = __ldcs(reinterpret_cast<const float4 *>(x) + i);
        int4 o = make_int4(code_f32(a.x, q, err), code_f32(a.y, q, err), code_f32(a.z, q, err), code_f32(a.w, q, err));
        __stcs(reinterpret_cast<int4 *>(codes) + i, o);
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        uint64_t j = n4 * 4 + threadIdx.x;
        codes[j] = code_f32(x[j], q, err);
    }
    if (err) set_err(sc, err);
}

}  // namespace roix

using namespace roix;

static int grid_for(uint64_t work_items, int threads, int per_sm) {
    uint64_t need = (work_items + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms() * per_sm;
    if (need < 1) need = 1;
    return (int)(need < cap ? need : cap);
}

cudaError_t launch_hist_u16(const uint16_t *x, uint64_t n, roix_scalars *sc, uint64_t *hist, cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    constexpr int smem = (HWIN + 32 * RW) * 4;   // 112 KiB: two CTAs per SM
    const cudaError_t e = dyn_smem_once(k_hist_u16_rw, smem, attr);
    if (e != cudaSuccess) return e;
    k_hist_u16_rw<<<grid_for(n / 8, 1024, 2), 1024, smem, st>>>(x, n, sc, hist);
    return cudaGetLastError();
}

cudaError_t launch_hist_u16_frames(const uint16_t *x, uint64_t nframes, uint64_t A, roix_scalars *sc, uint64_t *hist,
                                   cudaStream_t st) {
    static std::atomic<unsigned long long> attr{0};
    const cudaError_t e = dyn_smem_once(k_hist_u16_frames, HWIN * 4, attr);
    if (e != cudaSuccess) return e;
    const uint64_t n = nframes * A;
    if (n == 0) return cudaSuccess;
    k_hist_u16_frames<<<grid_for(n / 8, 1024, 2), 1024, HWIN * 4, st>>>(x, n, A, sc, hist);
    return cudaGetLastError();
}

cudaError_t launch_hist_f32(const float *x, uint64_t n, roix_scalars *sc, uint64_t *hist, cudaStream_t st) {
    k_hist_f32<<<grid_for(n / 4, 512, 3), 512, 0, st>>>(x, n, sc, hist);
    return cudaGetLastError();
}

cudaError_t launch_quantize(const void *x, int dtype, uint64_t n, roix_scalars *sc, void *codes, cudaStream_t st) {
    if (dtype == ROIX_U16)
        k_quantize_u16<<<grid_for(n / 8, 512, 4), 512, 0, st>>>((const uint16_t *)x, n, sc, (uint16_t *)codes);
    else
        k_quantize_f32<<<grid_for(n / 4, 512, 4), 512, 0, st>>>((const float *)x, n, sc, (int32_t *)codes);
    return cudaGetLastError();
}
