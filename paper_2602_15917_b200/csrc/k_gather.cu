// k_gather.cu -- a1+a8 EXTRACT from the kept x-runs of a6/a7 (roix_extract_runs).
//
// The code stream is the concatenation, in run order (= increasing linear index, G-17), of the
// quantised voxels of every run whose component was kept.  So instead of scanning the kept mask K
// (N/8 bytes) and gathering x under its set bits, this path reads exactly the kept voxels of x,
// contiguously run by run, and never reads K:
//   1. k_kept_len     klen[r] = x1 - x0 if run r's component is kept, else 0
//   2. scan           koff = exclusive prefix of klen (uint64): run r's codes are [koff[r], koff[r+1])
//   3. k_chunk_first  cfirst[c] = the run holding the first code of output chunk c
//   4. k_gather       persistent warps over output chunks of 32 x 4 groups of V = 16 / sizeof(x)
//                     consecutive codes.  A chunk's runs (<= 31; more: element-wise path) sit in
//                     the warp's registers, one per lane; each lane finds its groups' runs by a
//                     5-step shfl search, loads a group inside one run as one or two 16-byte loads
//                     of x (all 4 groups in flight, the next chunk's run table behind them),
//                     quantises V codes in registers and writes one 16-byte streaming store.
//                     Groups across a run boundary (and the stream's ragged ends) go element by
//                     element.  (A TMA-staged variant -- producer warps bulk-copying each run into
//                     a shared-memory ring -- was measured slower on B200.)
// Output positions are handled in the global stream space p = offset + j so that every group is
// 16-byte aligned in codes_out whatever the rank's offset.
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace roix {

template <typename T>
__host__ __device__ constexpr int gr_v() { return 16 / (int)sizeof(T); }   // elements per 16-byte group

__global__ void k_kept_len(const RunsView R, uint32_t *klen, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        klen[i] = R.kept[R.parent[i]] ? R.x1[i] - R.x0[i] : 0u;
}

// chunk c starts at j = max(0, c * CH - a), a = offset mod V; it belongs to the run r with
// koff[r] <= j < koff[r + 1]
__global__ void k_chunk_first(const RunsView R, const uint64_t *koff, const uint64_t *offset, uint64_t ch,
                              uint32_t V, uint32_t *cfirst, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    const uint64_t a = (offset ? *offset : 0) % V;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = koff[r], e = koff[r + 1];
        if (b == e) continue;
        if (b == 0) cfirst[0] = (uint32_t)r;
        for (uint64_t c = (b + a + ch - 1) / ch; c * ch < e + a; c++)
            if (c > 0) cfirst[c] = (uint32_t)r;
    }
}

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

constexpr int GW_G = 4;   // groups per lane per warp chunk

template <typename T>
__host__ __device__ constexpr uint64_t gw_ch() { return (uint64_t)32 * GW_G * gr_v<T>(); }   // codes per warp chunk

// Run table of one warp chunk (chunk-relative positions r = j - jc0, jc0 = c * CH - a): lane l < nb
// holds run rb + l -- kof = its first code's position, clamped to [0, CH + 1], and xb = the x element
// of position 0 if that run extended there (x element of position r = xb + r); lane nb holds the end
// of run re; lanes above nb hold UINT32_MAX.  slow: the chunk touches more than 31 runs.
struct WTable {
    uint32_t kof;
    int64_t xb;
    uint64_t rb, re;
    uint32_t slow;
};

__device__ __forceinline__ void wt_range(const uint32_t *cfirst, uint64_t c, uint64_t nchunks, uint64_t nruns,
                                         uint64_t &rb, uint64_t &re) {
    rb = cfirst[c];
    re = c + 1 < nchunks ? cfirst[c + 1] : nruns - 1;
}

__device__ __forceinline__ WTable wt_load(const RunsView &R, const uint64_t *koff, uint64_t nx, uint64_t rb,
                                          uint64_t re, int64_t jc0, uint32_t ch) {
    WTable t;
    const uint32_t lane = lane_id();
    const uint64_t nb = re - rb + 1;
    t.rb = rb;
    t.re = re;
    t.slow = nb > 31;
    t.kof = 0xffffffffu;
    t.xb = 0;
    if (!t.slow && lane <= nb) {
        const uint64_t r = rb + lane;
        const int64_t ko = (int64_t)koff[r];
        const int64_t rel = ko - jc0;
        t.kof = rel < 0 ? 0u : (rel > (int64_t)ch ? ch + 1 : (uint32_t)rel);
        if (lane < nb) t.xb = (int64_t)((uint64_t)R.rrow[r] * nx + R.x0[r]) - ko + jc0;
    }
    return t;
}

// code of output j from the runs [rb, re] in global memory (chunks touching more than 31 runs)
template <typename T, int QM>
__device__ __forceinline__ uint32_t code_at(const T *x, const RunsView &R, uint64_t nx, const uint64_t *koff,
                                            uint64_t rb, uint64_t re, uint64_t j, const QP &q, uint32_t &err) {
    uint64_t lo = rb, hi = re + 1;
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (koff[mid] <= j) lo = mid;
        else hi = mid;
    }
    const uint64_t v = (uint64_t)R.rrow[lo] * nx + R.x0[lo] + (j - koff[lo]);
    return code1<T, QM>(x[v], q, err);
}

// codes of the group at chunk position r, element by element through the shared-memory copy of the
// run table (positions in [r_lo, r_hi); stores below r_cap)
template <typename T, typename C, int QM>
__device__ __noinline__ void gather_elems(const T *__restrict__ x, C *__restrict__ out, uint64_t pbase, uint32_t r,
                                          uint32_t r_lo, uint32_t r_hi, uint32_t r_cap, const uint32_t *s_kof,
                                          const int64_t *s_xb, const QP &q, uint32_t &err) {
    constexpr int V = gr_v<T>();
    uint32_t h = 0;
    for (uint32_t e = 0; e < (uint32_t)V; e++) {
        const uint32_t rj = r + e;
        if (rj < r_lo || rj >= r_hi) continue;
        while (s_kof[h + 1] <= rj) h++;
        const uint32_t cd = code1<T, QM>(x[(uint64_t)(s_xb[h] + rj)], q, err);
        if (rj < r_cap) out[pbase + rj] = (C)cd;
    }
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void gather_w(const T *__restrict__ x, const RunsView &R, uint64_t nx,
                                         const uint64_t *__restrict__ koff, const uint32_t *__restrict__ cfirst,
                                         roix_scalars *sc, C *__restrict__ out, uint64_t capacity, uint64_t base_off,
                                         const QP &q, uint32_t *s_kof, int64_t *s_xb) {
    constexpr int V = gr_v<T>();
    constexpr uint32_t LV = V == 8 ? 3 : 2;
    constexpr uint32_t CH = (uint32_t)gw_ch<T>();
    const uint32_t lane = lane_id();
    const uint64_t nruns = *R.n_runs;
    const uint64_t total = nruns ? koff[nruns] : 0;
    const uint64_t a = base_off % V;
    const uint64_t nchunks = total ? (total + a + CH - 1) / CH : 0;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    uint32_t err = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && base_off + total > capacity) err |= ROIX_ERR_CAPACITY;
    uint64_t c = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (c < nchunks) {
        uint64_t rb, re;
        wt_range(cfirst, c, nchunks, nruns, rb, re);
        WTable tb = wt_load(R, koff, nx, rb, re, (int64_t)(c * CH) - (int64_t)a, CH);
        for (; c < nchunks; c += nw) {
            const uint64_t cn = c + nw;
            uint64_t rb2 = 0, re2 = 0;
            if (cn < nchunks) wt_range(cfirst, cn, nchunks, nruns, rb2, re2);   // next chunk's runs
            const int64_t jc0 = (int64_t)(c * CH) - (int64_t)a;
            const uint64_t pbase = base_off + (uint64_t)jc0;                       // output of position 0
            const uint32_t r_lo = jc0 < 0 ? (uint32_t)(-jc0) : 0u;
            const uint32_t r_hi = (uint32_t)min((int64_t)CH, (int64_t)total - jc0);
            const uint32_t r_cap = capacity > pbase ? (uint32_t)min((uint64_t)CH, capacity - pbase) : 0u;
            if (!tb.slow) {
                __syncwarp();
                s_kof[lane] = tb.kof;
                if (lane == 0) s_kof[32] = 0xffffffffu;
                s_xb[lane] = tb.xb;
                __syncwarp();
                bool whole[GW_G];
                uint32_t kk[GW_G];
                uint4 b0[GW_G], b1[GW_G];
#pragma unroll
                for (int u = 0; u < GW_G; u++) {
                    const uint32_t r = (lane + 32u * u) * V;
                    const uint32_t rs = max(r, r_lo);
                    // run of position rs: the largest lane k with kof_k <= rs (lanes hold increasing kof)
                    uint32_t k = 0;
#pragma unroll
                    for (int step = 16; step > 0; step >>= 1) {
                        const uint32_t kv = __shfl_sync(FULL, tb.kof, k + step);
                        if (kv <= rs) k += step;
                    }
                    const uint32_t kend = __shfl_sync(FULL, tb.kof, (k + 1) & 31);
                    const int64_t xb = __shfl_sync(FULL, tb.xb, k);
                    whole[u] = r >= r_lo && r + V <= r_hi && kend >= r + V;
                    const uint64_t v = (uint64_t)(xb + r);
                    kk[u] = (uint32_t)v & (V - 1);
                    b0[u] = b1[u] = make_uint4(0, 0, 0, 0);
                    if (whole[u]) {
                        b0[u] = __ldcs(x4 + (v >> LV));
                        if (kk[u]) b1[u] = __ldcs(x4 + (v >> LV) + 1);
                    }
                }
                WTable tn = tb;
                if (cn < nchunks) tn = wt_load(R, koff, nx, rb2, re2, (int64_t)(cn * CH) - (int64_t)a, CH);
#pragma unroll
                for (int u = 0; u < GW_G; u++) {
                    const uint32_t r = (lane + 32u * u) * V;
                    if (whole[u]) {
                        const uint4 cv = code_group<T, QM>(window16<T>(b0[u], b1[u], kk[u]), q, err);
                        if (r + V <= r_cap) {
                            __stcs(reinterpret_cast<uint4 *>(out + pbase + r), cv);
                        } else {
                            const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                            for (int e = 0; e < V; e++)
                                if (r + e < r_cap)
                                    out[pbase + r + e] = (C)(sizeof(C) == 2 ? (cw[e >> 1] >> ((e & 1) * 16)) & 0xffffu
                                                                            : cw[e]);
                        }
                    }
                }
                // groups across a run boundary / at the stream's ends (a warp-uniform branch)
#pragma unroll
                for (int u = 0; u < GW_G; u++) {
                    const uint32_t r = (lane + 32u * u) * V;
                    const bool need = !whole[u] && r + V > r_lo && r < r_hi;
                    if (__any_sync(FULL, need) && need)
                        gather_elems<T, C, QM>(x, out, pbase, r, r_lo, r_hi, r_cap, s_kof, s_xb, q, err);
                }
                tb = tn;
            } else {
                for (uint32_t r = max(r_lo, 0u) + lane; r < r_hi; r += 32) {
                    const uint32_t cd = code_at<T, QM>(x, R, nx, koff, tb.rb, tb.re, (uint64_t)(jc0 + r), q, err);
                    if (r < r_cap) out[pbase + r] = (C)cd;
                }
                if (cn < nchunks) tb = wt_load(R, koff, nx, rb2, re2, (int64_t)(cn * CH) - (int64_t)a, CH);
            }
        }
    }
    if (err) set_err(sc, err);
}

template <typename T, typename C>
__global__ void __launch_bounds__(256, 2) k_gather(const T *__restrict__ x, const RunsView R, uint64_t nx,
                                                   const uint64_t *__restrict__ koff, const uint32_t *__restrict__ cfirst,
                                                   roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                                                   const uint64_t *offset) {
    // each warp's run table, mirrored in shared memory for the element-wise (divergent) cases
    __shared__ uint32_t s_kof[8][33];
    __shared__ int64_t s_xb[8][32];
    if (get_err(sc)) return;
    const QP q = load_qp(sc);
    const uint64_t base_off = offset ? *offset : 0;
    const int w = threadIdx.x >> 5;
    if constexpr (sizeof(T) == 4) {
        gather_w<T, C, QM_FLOAT>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, s_kof[w], s_xb[w]);
    } else {
        switch (qmode(q)) {
        case QM_POW2: gather_w<T, C, QM_POW2>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, s_kof[w], s_xb[w]); break;
        case QM_INT: gather_w<T, C, QM_INT>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, s_kof[w], s_xb[w]); break;
        case QM_ONE: gather_w<T, C, QM_ONE>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, s_kof[w], s_xb[w]); break;
        default: gather_w<T, C, QM_FLOAT>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, s_kof[w], s_xb[w]); break;
        }
    }
}

__global__ void k_gather_total(const RunsView R, const uint64_t *koff, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    sc->count += n ? koff[n] : 0;
}

}  // namespace roix

using namespace roix;

uint64_t gather_chunks_max(uint64_t n) { return (n + 16) / gw_ch<float>() + 2; }

template <typename T, typename C>
static cudaError_t gather_grid(int *grid) {
    int occ = 0;
    cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<T, C>, 256, 0);
    if (e != cudaSuccess) return e;
    *grid = num_sms() * (occ > 0 ? occ : 1);
    return cudaSuccess;
}

cudaError_t launch_gather(const void *x, int dtype, uint64_t nx, const RunsView &R, uint64_t cap, uint32_t *klen,
                          uint64_t *koff, uint32_t *cfirst, uint64_t *scan_tmp, roix_scalars *sc, void *codes,
                          uint64_t capacity, const uint64_t *offset, cudaStream_t st) {
    const int grid = num_sms() * 8;
    k_kept_len<<<grid, 256, 0, st>>>(R, klen, sc);
    cudaError_t e = scan_u64_dev(klen, koff, R.n_runs, cap, scan_tmp, st);
    if (e != cudaSuccess) return e;
    static int g16 = 0, g32 = 0;
    if (dtype == ROIX_U16) {
        if (!g16 && (e = gather_grid<uint16_t, uint16_t>(&g16)) != cudaSuccess) return e;
        k_chunk_first<<<grid, 256, 0, st>>>(R, koff, offset, gw_ch<uint16_t>(), gr_v<uint16_t>(), cfirst, sc);
        k_gather<uint16_t, uint16_t><<<g16, 256, 0, st>>>((const uint16_t *)x, R, nx, koff, cfirst, sc,
                                                         (uint16_t *)codes, capacity, offset);
    } else {
        if (!g32 && (e = gather_grid<float, int32_t>(&g32)) != cudaSuccess) return e;
        k_chunk_first<<<grid, 256, 0, st>>>(R, koff, offset, gw_ch<float>(), gr_v<float>(), cfirst, sc);
        k_gather<float, int32_t><<<g32, 256, 0, st>>>((const float *)x, R, nx, koff, cfirst, sc, (int32_t *)codes,
                                                      capacity, offset);
    }
    k_gather_total<<<1, 1, 0, st>>>(R, koff, sc);
    return cudaGetLastError();
}
