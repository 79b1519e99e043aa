// k_setup.cu -- scalars initialisation, a0 RANGE (fp32 min/max) and eb / I_max / norm8-edge
// resolution (readings G-6, G-8, G-30).
#include <cfloat>

#include "common.cuh"
#include "kernels.cuh"

namespace roix {

__global__ void k_scalars_init(roix_scalars *sc, float eb) {
    int t = threadIdx.x;
    if (t == 0) {
        sc->err = 0;
        sc->min_ord = f2ord(INFINITY);
        sc->max_ord = f2ord(-INFINITY);
        sc->polarity = 0;
        sc->eb = eb;
        sc->s = 0.0f;
        sc->s_inv = 0.0f;
        sc->s_int = 0;
        sc->s_magic = 0;
        sc->t8_all = 0;
        sc->i_max = 1.0f;
        sc->t8 = 0;
        sc->thr_u16 = 0;
        sc->thr_f32 = 0.0f;
        sc->count = 0;
        sc->n_components = 0;
        sc->n_kept = 0;
        sc->n_runs = 0;
        sc->spec_lo = sc->spec_hi = 0;
        sc->spec_state = 0;
        sc->run_slots = 0;
        sc->n_uncertain = 0;
    }
    for (int k = t; k < 256; k += blockDim.x) sc->edges[k] = 0.0f;
}

// a0: min / max over all voxels; non-finite voxels set ROIX_ERR_NONFINITE (G-32).
__global__ void __launch_bounds__(512) k_range(const float *__restrict__ x, uint64_t n, roix_scalars *sc) {
    if (get_err(sc)) return;
    float lo = INFINITY, hi = -INFINITY;
    bool bad = false;
    const uint64_t n4 = n / 4;
    const float4 *x4 = reinterpret_cast<const float4 *>(x);
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
    uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (; i + 7 * stride < n4; i += 8 * stride) {   // 8 x 16 bytes in flight per thread
        float4 a[8];
#pragma unroll
        for (int u = 0; u < 8; u++) a[u] = __ldcs(x4 + i + u * stride);
#pragma unroll
        for (int u = 0; u < 8; u++) {
            const float v[4] = {a[u].x, a[u].y, a[u].z, a[u].w};
#pragma unroll
            for (int k = 0; k < 4; k++) {
                bad |= !(fabsf(v[k]) <= FLT_MAX);
                lo = fminf(lo, v[k]);
                hi = fmaxf(hi, v[k]);
            }
        }
    }
    for (; i < n4; i += stride) {
        float4 a = __ldcs(x4 + i);
        float v[4] = {a.x, a.y, a.z, a.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            bad |= !(fabsf(v[k]) <= FLT_MAX);
            lo = fminf(lo, v[k]);
            hi = fmaxf(hi, v[k]);
        }
    }
    if (blockIdx.x == 0 && threadIdx.x < (n & 3)) {
        float v = x[n4 * 4 + threadIdx.x];
        bad |= !(fabsf(v) <= FLT_MAX);
        lo = fminf(lo, v);
        hi = fmaxf(hi, v);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        lo = fminf(lo, __shfl_xor_sync(FULL, lo, d));
        hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, d));
    }
    bad = __any_sync(FULL, bad);
    if (lane_id() == 0) {
        if (bad) set_err(sc, ROIX_ERR_NONFINITE);
        if (lo <= hi) {
            atomicMin(&sc->min_ord, f2ord(lo));
            atomicMax(&sc->max_ord, f2ord(hi));
        }
    }
}

// G-30: norm8(x) = clamp(floor(fl64(fl64(x) * 255 / fl64(I_max)) + 0.5), 0, 255), IEEE binary64.
__device__ __forceinline__ int norm8_f64(float x, double imax) {
    double q = __ddiv_rn(__dmul_rn((double)x, 255.0), imax);
    double r = floor(__dadd_rn(q, 0.5));
    if (!(r > 0.0)) return 0;
    if (r > 255.0) return 255;
    return (int)r;
}

// One CTA of 256 threads.  Thread k >= 1 bisects over the ordered encoding of the non-negative
// floats [+0, I_max] for the smallest x with norm8(x) >= k (norm8 is monotone and norm8(I_max) = 255).
__global__ void k_resolve(roix_scalars *sc, int dtype, double rel_eb) {
    __shared__ float s_eb;
    const int t = threadIdx.x;
    if (t == 0) {
        float eb = sc->eb;
        if (rel_eb > 0.0) {
            float mn = ord2f(sc->min_ord), mx = ord2f(sc->max_ord);
            eb = (float)(rel_eb * ((double)mx - (double)mn));   // G-6
            sc->eb = eb;
        }
        float s = 2.0f * eb;
        if (!(eb > 0.0f) || !(s <= FLT_MAX)) set_err(sc, ROIX_ERR_RANGE);
        sc->s = s;
        sc->s_inv = __fdiv_rn(1.0f, s);
        uint32_t si = 0, mg = 0;
        if (s >= 1.0f && s <= 65535.0f && rintf(s) == s) {
            si = (uint32_t)s;
            if (si >= 2) mg = (uint32_t)((0x100000000ull + si - 1) / si);
        }
        sc->s_int = si;
        sc->s_magic = mg;
        if (dtype == ROIX_F32) {
            float mx = ord2f(sc->max_ord);
            sc->i_max = mx > 0.0f ? mx : 1.0f;                 // G-8
        }
        s_eb = eb;
    }
    __syncthreads();
    if (dtype != ROIX_F32) return;
    const float imax_f = sc->i_max;
    const double imax = (double)imax_f;
    if (t == 0) sc->edges[0] = -INFINITY;
    if (t >= 1 && t < 256) {
        uint32_t lo = f2ord(0.0f), hi = f2ord(imax_f);   // norm8(lo) = 0 < t <= 255 = norm8(hi)
        while (lo + 1 < hi) {                            // invariant: norm8(lo) < t <= norm8(hi)
            uint32_t mid = lo + (hi - lo) / 2;
            if (norm8_f64(ord2f(mid), imax) >= t) hi = mid;
            else lo = mid;
        }
        sc->edges[t] = ord2f(hi);
    }
}

}  // namespace roix

using namespace roix;

cudaError_t launch_scalars_init(roix_scalars *sc, float eb, cudaStream_t st) {
    k_scalars_init<<<1, 256, 0, st>>>(sc, eb);
    return cudaGetLastError();
}

// zero an accumulating histogram (16-byte stores, grid-stride)
__global__ void k_hist_clear(uint64_t *hist, uint64_t nbins) {
    const uint64_t n2 = nbins / 2;
    ulonglong2 *h2 = reinterpret_cast<ulonglong2 *>(hist);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (uint64_t)gridDim.x * blockDim.x)
        h2[i] = make_ulonglong2(0ull, 0ull);
    if ((nbins & 1) && blockIdx.x == 0 && threadIdx.x == 0) hist[nbins - 1] = 0ull;
}

cudaError_t launch_hist_clear(uint64_t *hist, uint64_t nbins, cudaStream_t st) {
    uint64_t need = (nbins / 2 + 255) / 256;
    const uint64_t cap = (uint64_t)num_sms() * 4;
    if (need < 1) need = 1;
    k_hist_clear<<<(unsigned)(need < cap ? need : cap), 256, 0, st>>>(hist, nbins);
    return cudaGetLastError();
}

cudaError_t launch_range(const float *x, uint64_t n, roix_scalars *sc, cudaStream_t st) {
    int blocks = num_sms() * 3;
    uint64_t need = (n / 4 + 511) / 512;
    if ((uint64_t)blocks > need) blocks = (int)(need > 0 ? need : 1);
    k_range<<<blocks, 512, 0, st>>>(x, n, sc);
    return cudaGetLastError();
}

cudaError_t launch_resolve(roix_scalars *sc, int dtype, double rel_eb, cudaStream_t st) {
    k_resolve<<<1, 256, 0, st>>>(sc, dtype, rel_eb);
    return cudaGetLastError();
}
