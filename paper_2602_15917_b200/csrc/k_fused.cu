// k_fused.cu -- a2 HISTOGRAM fused with a4 BINARISE by speculation (one read of x instead of two).
//
// The threshold of Eq. 2 depends on the histogram of all voxels, so a plain pipeline reads
// x twice.  Here a sample of the volume (1/64 of it, in 64 equal segments) gives Otsu a speculative
// window [lo, hi] for the raw threshold (k_spec).  One pass then accumulates the full histogram and
// writes, for every voxel, the mask bit that is already certain for any threshold inside the window
// (HIGH: x >= hi -> 1, x < lo -> 0; LOW mirrored); voxels with lo <= x < hi are "uncertain" and their
// indices are queued.  After the exact threshold is known, k_spec_fix resolves the queued voxels; if
// the exact threshold fell outside the window or the queue overflowed, the plain binarisation pass
// runs instead (k_binarize checks spec_state), so the mask is exactly that of Eq. 2 either way.
#include <cfloat>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace roix {

constexpr int FHWIN = 16384;   // u16 shared-histogram window (as k_hist_u16)

struct FusedWS {
    uint32_t *m;          // [nwords + 64] mask words (shared with roix_morph's workspace layout)
    uint64_t *shist;      // [65536] sample histogram
    uint64_t *unc;        // [ucap] uncertain voxel indices
    uint64_t ucap;
};

static size_t fused_carve(void *base, uint64_t n, FusedWS *w) {
    const uint64_t nwords = (n + 31) / 32;
    const size_t a = ((nwords + 64) * 4 + 255) & ~(size_t)255;
    const size_t b = 65536 * 8;
    const uint64_t ucap = n / 512 > (1u << 16) ? n / 512 : (1u << 16);
    if (w) {
        w->m = (uint32_t *)base;
        w->shist = (uint64_t *)((char *)base + a);
        w->unc = (uint64_t *)((char *)base + a + b);
        w->ucap = ucap;
    }
    return a + b + ucap * 8;
}

// ---------------------------------------------------------------------------------- sample pass
// every rs-th row of X voxels (rows spread over y and z): a representative 1/rs of the volume
__device__ __forceinline__ int norm8_edges_f(float x, float scale, const float *e) {
    int k = __float2int_rz(fminf(fmaxf(x * scale + 0.5f, 0.0f), 255.0f));
    while (x >= e[k + 1]) k++;
    while (x < e[k]) k--;
    return k;
}

// one warp per sampled row (coalesced loads along the row), counters in a shared window of FHWIN
// bins (u16; values above it go to the global bins) or the 256 norm8 bins (fp32)
template <typename T>
__global__ void __launch_bounds__(512) k_sample_hist(const T *__restrict__ x, uint64_t X, uint64_t nrows, uint64_t rs,
                                                     roix_scalars *sc, uint64_t *gh) {
    extern __shared__ uint32_t sh[];   // u16: FHWIN bins; f32: 256 bins + 257 edges
    if (get_err(sc)) return;
    constexpr bool f32 = sizeof(T) == 4;
    const int nb = f32 ? 256 : FHWIN;
    float *e = reinterpret_cast<float *>(sh + 256);
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    if (f32) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) e[i] = i == 0 ? -INFINITY : sc->edges[i];
        if (threadIdx.x == 0) e[256] = INFINITY;
    }
    const float scale = f32 ? 255.0f / sc->i_max : 0.0f;
    __syncthreads();
    const uint64_t ns = (nrows + rs - 1) / rs;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t k = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < ns; k += nw) {
        const T *row = x + k * rs * X;
        for (uint64_t c = lane_id(); c < X; c += 32) {
            const T v = row[c];
            if constexpr (sizeof(T) == 2) {
                if ((uint32_t)v < (uint32_t)FHWIN) atomicAdd(&sh[v], 1u);
                else atomicAdd((unsigned long long *)&gh[v], 1ull);
            } else {
                if (fabsf(v) <= FLT_MAX) atomicAdd(&sh[norm8_edges_f(v, scale, e)], 1u);
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        if (sh[b]) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)sh[b]);
}

// ------------------------------------------------------------------------------ the fused pass
// Warp iteration = 1024 voxels = 32 mask words (as k_binarize): lane l loads the 16-byte groups
// c * 32 + l, counts them into the shared histogram and packs their certain / uncertain bits.
template <typename T>
struct Spec;
template <>
struct Spec<uint16_t> {
    static constexpr int VPL = 8;
    uint32_t lo, hi;
    bool low;
    __device__ Spec(const roix_scalars *sc) : lo(sc->spec_lo), hi(sc->spec_hi), low(sc->polarity != 0) {}
    __device__ __forceinline__ void bits(uint32_t v, uint32_t &cert, uint32_t &unc) const {
        const bool ge_hi = v >= hi, ge_lo = v >= lo;
        cert = low ? !ge_lo : ge_hi;
        unc = ge_lo && !ge_hi;
    }
};
template <>
struct Spec<float> {
    static constexpr int VPL = 4;
    float lo, hi;
    bool low;
    __device__ Spec(const roix_scalars *sc) : low(sc->polarity != 0) {
        memcpy(&lo, &sc->spec_lo, 4);
        memcpy(&hi, &sc->spec_hi, 4);
    }
    __device__ __forceinline__ void bits(float v, uint32_t &cert, uint32_t &unc) const {
        const bool ge_hi = v >= hi, ge_lo = v >= lo;
        cert = low ? !ge_lo : ge_hi;
        unc = ge_lo && !ge_hi;
    }
};

template <typename T>
__global__ void __launch_bounds__(512, 3) k_hist_bin(const T *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                       uint64_t *gh, FusedWS W) {
    extern __shared__ uint32_t sh[];   // u16: FHWIN bins; f32: 256 bins + 257 edges
    constexpr int VPL = Spec<T>::VPL, CH = 32 / VPL, GPW = 32 / VPL;
    if (get_err(sc)) return;
    const bool f32 = sizeof(T) == 4;
    float *e = reinterpret_cast<float *>(sh + 256);
    const int nb = f32 ? 256 : FHWIN;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0;
    if (f32) {
        for (int i = threadIdx.x; i < 256; i += blockDim.x) e[i] = i == 0 ? -INFINITY : sc->edges[i];
        if (threadIdx.x == 0) e[256] = INFINITY;
    }
    const float scale = f32 ? 255.0f / sc->i_max : 0.0f;
    const bool spec = sc->spec_state == 1;
    const Spec<T> sp(sc);
    __syncthreads();
    const uint32_t lane = lane_id();
    const uint64_t iters = (n + 1023) / 1024, nwords = (n + 31) / 32;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    bool bad = false;
    for (uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < iters; it += wstride) {
        const uint64_t g0 = it * 32 * CH;
        uint32_t Pc = 0, Pu = 0;
        constexpr int B = CH < 4 ? CH : 4;   // loads in flight per batch
        uint4 v[B];
        const bool whole = (it + 1) * 1024 <= n;
#pragma unroll
        for (int c = 0; c < CH; c++) {
            if (c % B == 0) {
#pragma unroll
                for (int u = 0; u < B; u++) v[u] = whole ? __ldcs(x4 + g0 + (c + u) * 32 + lane) : make_uint4(0, 0, 0, 0);
            }
            const uint64_t vb = (g0 + c * 32 + lane) * VPL;
            T vals[VPL];
            uint32_t valid = (1u << VPL) - 1u;
            if (whole) {
                const uint4 vv = v[c % B];
                if constexpr (sizeof(T) == 2) {
                    const uint32_t w[4] = {vv.x, vv.y, vv.z, vv.w};
#pragma unroll
                    for (int k = 0; k < 8; k++) vals[k] = (T)((w[k >> 1] >> ((k & 1) * 16)) & 0xffffu);
                } else {
                    vals[0] = __uint_as_float(vv.x);
                    vals[1] = __uint_as_float(vv.y);
                    vals[2] = __uint_as_float(vv.z);
                    vals[3] = __uint_as_float(vv.w);
                }
            } else {
                valid = 0;
#pragma unroll
                for (int k = 0; k < VPL; k++) {
                    vals[k] = (T)0;
                    if (vb + k < n) {
                        vals[k] = x[vb + k];
                        valid |= 1u << k;
                    }
                }
            }
#pragma unroll
            for (int k = 0; k < VPL; k++) {
                if (!((valid >> k) & 1)) continue;
                if constexpr (sizeof(T) == 2) {
                    const uint32_t val = vals[k];
                    if (val < (uint32_t)FHWIN) atomicAdd(&sh[val], 1u);
                    else atomicAdd((unsigned long long *)&gh[val], 1ull);
                } else {
                    const float val = vals[k];
                    if (fabsf(val) <= FLT_MAX) atomicAdd(&sh[norm8_edges_f(val, scale, e)], 1u);
                    else bad = true;
                }
                uint32_t cb, ub;
                sp.bits(vals[k], cb, ub);
                Pc |= cb << (c * VPL + k);
                Pu |= ub << (c * VPL + k);
            }
        }
        if (!spec) continue;
        // word j = groups j * GPW .. of chunk c = j / VPL (see k_binarize)
        const uint32_t cc = lane / VPL, src0 = (lane % VPL) * GPW;
        uint32_t wc = 0, wu = 0;
#pragma unroll
        for (int i = 0; i < GPW; i++) {
            const uint32_t qc = __shfl_sync(FULL, Pc, src0 + i), qu = __shfl_sync(FULL, Pu, src0 + i);
            wc |= ((qc >> (cc * VPL)) & ((1u << VPL) - 1u)) << (i * VPL);
            wu |= ((qu >> (cc * VPL)) & ((1u << VPL) - 1u)) << (i * VPL);
        }
        const uint64_t wi = it * 32 + lane;
        if (wi < nwords) W.m[wi] = wc;
        // queue the uncertain voxels (rare: they lie inside the threshold window)
        if (__any_sync(FULL, wu != 0)) {
            const uint32_t cnt = __popc(wu);
            const uint32_t incl = warp_incl_scan(cnt);
            unsigned long long at = 0;
            if (lane == 31 && incl) at = atomicAdd((unsigned long long *)&sc->n_uncertain, (unsigned long long)incl);
            at = __shfl_sync(FULL, at, 31) + incl - cnt;
            uint32_t bits = wu;
            while (bits) {
                const uint32_t b = __ffs(bits) - 1;
                bits &= bits - 1;
                if (at < W.ucap) W.unc[at] = wi * 32 + b;
                at++;
            }
        }
    }
    if (bad) set_err(sc, ROIX_ERR_NONFINITE);
    __syncthreads();
    for (int b = threadIdx.x; b < nb; b += blockDim.x)
        if (sh[b]) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)sh[b]);
}

// uint16 volumes of whole 16-byte groups (n % 8 == 0, every BASELINE config): the lean form of
// k_hist_bin, shaped like k_hist_u16.  A warp iteration covers 64 groups (512 voxels, 16 mask words):
// lane l takes groups l and 32 + l (two loads in flight), adds their 16 voxels to the shared window and
// forms their certain / uncertain bits (one byte each per group); lane j < 16 then gathers mask word j
// from the 4 lanes that hold its groups.
__global__ void __launch_bounds__(1024, 2) k_hist_bin_u16(const uint16_t *__restrict__ x, uint64_t n,
                                                         roix_scalars *sc, uint64_t *gh, FusedWS W) {
    extern __shared__ uint32_t sh[];   // FHWIN bins
    if (get_err(sc)) return;
    for (int i = threadIdx.x; i < FHWIN; i += blockDim.x) sh[i] = 0;
    const bool spec = sc->spec_state == 1;
    const uint32_t lo = sc->spec_lo, hi = sc->spec_hi;
    const uint32_t low = sc->polarity != 0;
    __syncthreads();
    const uint32_t lane = lane_id();
    const uint64_t ng = n / 8, nwords = (n + 31) / 32;
    const uint64_t iters = (ng + 63) / 64;
    const uint64_t nwarps = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint4 *x8 = reinterpret_cast<const uint4 *>(x);
    auto add = [&](uint32_t v) {
        if (v < (uint32_t)FHWIN) atomicAdd(&sh[v], 1u);
        else atomicAdd((unsigned long long *)&gh[v], 1ull);
    };
    const uint32_t hi2 = hi | (hi << 16), lo2 = lo | (lo << 16);
    // the 8 voxels of a group into the histogram (branch-free unless a value leaves the shared window),
    // and their certain (bit k) / uncertain (bit 8 + k) bits from halfword SIMD compares
    auto group = [&](uint4 d) -> uint32_t {
        const uint32_t w[4] = {d.x, d.y, d.z, d.w};
        if (((d.x | d.y | d.z | d.w) & 0xC000C000u) == 0) {   // every value < 16384 = FHWIN
#pragma unroll
            for (int k = 0; k < 8; k++) atomicAdd(&sh[(w[k >> 1] >> ((k & 1) * 16)) & 0xffffu], 1u);
        } else {
#pragma unroll
            for (int k = 0; k < 8; k++) add((w[k >> 1] >> ((k & 1) * 16)) & 0xffffu);
        }
        uint32_t gh = 0, gl = 0;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const uint32_t rh = __vcmpgeu2(w[j], hi2), rl = __vcmpgeu2(w[j], lo2);   // 0xffff where >=
            gh |= (((rh >> 15) & 1u) | ((rh >> 30) & 2u)) << (2 * j);
            gl |= (((rl >> 15) & 1u) | ((rl >> 30) & 2u)) << (2 * j);
        }
        const uint32_t cert = low ? (~gl & 0xffu) : gh;
        return cert | ((gl & ~gh & 0xffu) << 8);
    };
    for (uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < iters; it += nwarps) {
        const uint64_t g0 = it * 64;
        const bool va = g0 + lane < ng, vb = g0 + 32 + lane < ng;
        const uint4 a = va ? __ldcs(x8 + g0 + lane) : make_uint4(0, 0, 0, 0);
        const uint4 b = vb ? __ldcs(x8 + g0 + 32 + lane) : make_uint4(0, 0, 0, 0);
        const uint32_t pa = va ? group(a) : 0u, pb = vb ? group(b) : 0u;
        if (!spec) continue;
        uint32_t wc = 0, wu = 0;
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const uint32_t src = 4 * (lane & 7) + i;
            const uint32_t qa = __shfl_sync(FULL, pa, src), qb = __shfl_sync(FULL, pb, src);
            const uint32_t q = lane < 8 ? qa : qb;
            wc |= (q & 0xffu) << (8 * i);
            wu |= ((q >> 8) & 0xffu) << (8 * i);
        }
        const uint64_t wi = it * 16 + lane;
        if (lane < 16 && wi < nwords) W.m[wi] = wc;
        else wu = 0;
        if (__any_sync(FULL, wu != 0)) {   // queue the uncertain voxels (rare: inside the window)
            const uint32_t cnt = __popc(wu);
            const uint32_t incl = warp_incl_scan(cnt);
            unsigned long long at = 0;
            if (lane == 31 && incl) at = atomicAdd((unsigned long long *)&sc->n_uncertain, (unsigned long long)incl);
            at = __shfl_sync(FULL, at, 31) + incl - cnt;
            uint32_t bits = wu;
            while (bits) {
                const uint32_t bb = __ffs(bits) - 1;
                bits &= bits - 1;
                if (at < W.ucap) W.unc[at] = wi * 32 + bb;
                at++;
            }
        }
    }
    __syncthreads();
    for (int b = threadIdx.x; b < FHWIN; b += blockDim.x)
        if (sh[b]) atomicAdd((unsigned long long *)&gh[b], (unsigned long long)sh[b]);
}

// After the exact threshold: resolve the queued voxels, or flag the plain binarisation.
__global__ void k_spec_check(roix_scalars *sc, int dtype, uint64_t ucap) {
    if (get_err(sc)) return;
    if (sc->spec_state != 1) {
        sc->spec_state = 3;
        return;
    }
    bool ok = sc->n_uncertain <= ucap;
    if (dtype == ROIX_U16) ok = ok && sc->spec_lo <= sc->thr_u16 && sc->thr_u16 <= sc->spec_hi;
    else ok = ok && __uint_as_float(sc->spec_lo) <= sc->thr_f32 && sc->thr_f32 <= __uint_as_float(sc->spec_hi);
    sc->spec_state = ok ? 2 : 3;
}

template <typename T>
__global__ void k_spec_fix(const T *__restrict__ x, roix_scalars *sc, FusedWS W) {
    if (get_err(sc) || sc->spec_state != 2) return;
    const uint64_t nu = sc->n_uncertain;
    const bool low = sc->polarity != 0;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nu; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t i = W.unc[k];
        bool ge;
        if constexpr (sizeof(T) == 2) ge = (uint32_t)x[i] >= sc->thr_u16;
        else ge = x[i] >= sc->thr_f32;
        if (ge != low) atomicOr(&W.m[i >> 5], 1u << (i & 31));
    }
}

}  // namespace roix

using namespace roix;

size_t fused_workspace_bytes(const roix_geom &g) { return fused_carve(nullptr, g.nz * g.ny * g.nx, nullptr); }

cudaError_t launch_histogram_binarize(const void *x, int dtype, const roix_geom &g, int polarity, roix_scalars *sc,
                                      uint64_t *hist, void *ws, cudaStream_t st) {
    FusedWS W;
    const uint64_t n = g.nz * g.ny * g.nx;
    fused_carve(ws, n, &W);
    cudaError_t e;
    // 1. sample histogram: every rs-th row (about 1/64 of the voxels, at least 4096 rows when possible)
    if ((e = cudaMemsetAsync(W.shist, 0, 65536 * 8, st)) != cudaSuccess) return e;
    const uint64_t nrows = g.nz * g.ny;
    uint64_t rs = nrows / 4096 < 64 ? (nrows / 4096 ? nrows / 4096 : 1) : 64;
    static std::atomic<unsigned long long> attr{0}, attr_s{0};
    if ((e = dyn_smem_once(k_hist_bin<uint16_t>, FHWIN * 4, attr)) != cudaSuccess) return e;
    if ((e = dyn_smem_once(k_sample_hist<uint16_t>, FHWIN * 4, attr_s)) != cudaSuccess) return e;
    const int sms = num_sms();
    if (dtype == ROIX_U16)
        k_sample_hist<uint16_t><<<sms * 2, 512, FHWIN * 4, st>>>((const uint16_t *)x, g.nx, nrows, rs, sc, W.shist);
    else
        k_sample_hist<float><<<sms * 2, 512, (256 + 257) * 4, st>>>((const float *)x, g.nx, nrows, rs, sc, W.shist);
    // 2. speculative window
    if ((e = launch_spec(W.shist, dtype, polarity, sc, st)) != cudaSuccess) return e;
    // 3. full histogram + certain mask bits + uncertain queue
    const uint64_t iters = (n + 1023) / 1024;
    uint64_t blocks = (iters + 15) / 16;
    if (blocks > (uint64_t)sms * 3) blocks = (uint64_t)sms * 3;
    if (blocks < 1) blocks = 1;
    static std::atomic<unsigned long long> attr_b{0};
    if (dtype == ROIX_U16 && n % 8 == 0) {
        if ((e = dyn_smem_once(k_hist_bin_u16, FHWIN * 4, attr_b)) != cudaSuccess) return e;
        const uint64_t wit = (n / 8 + 63) / 64;
        uint64_t b16 = (wit + 31) / 32;
        if (b16 > (uint64_t)sms * 2) b16 = (uint64_t)sms * 2;
        k_hist_bin_u16<<<(unsigned)(b16 ? b16 : 1), 1024, FHWIN * 4, st>>>((const uint16_t *)x, n, sc, hist, W);
    } else if (dtype == ROIX_U16)
        k_hist_bin<uint16_t><<<(unsigned)blocks, 512, FHWIN * 4, st>>>((const uint16_t *)x, n, sc, hist, W);
    else
        k_hist_bin<float><<<(unsigned)blocks, 512, (256 + 257) * 4, st>>>((const float *)x, n, sc, hist, W);
    return cudaGetLastError();
}

// the mask of the fused pass, completed with the exact threshold (called by roix_morph_prebinarized)
cudaError_t launch_spec_resolve(const void *x, int dtype, const roix_geom &g, roix_scalars *sc, void *ws,
                                cudaStream_t st) {
    FusedWS W;
    fused_carve(ws, g.nz * g.ny * g.nx, &W);
    k_spec_check<<<1, 1, 0, st>>>(sc, dtype, W.ucap);
    const int blocks = num_sms() * 2;
    if (dtype == ROIX_U16) k_spec_fix<uint16_t><<<blocks, 256, 0, st>>>((const uint16_t *)x, sc, W);
    else k_spec_fix<float><<<blocks, 256, 0, st>>>((const float *)x, sc, W);
    return cudaGetLastError();
}
