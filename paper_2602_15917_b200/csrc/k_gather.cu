// k_gather.cu -- a1+a8 EXTRACT from the kept x-runs of a6/a7 (roix_extract_runs).
//
// The code stream is the concatenation, in run order (= increasing linear index, G-17), of the
// quantised voxels of every run whose component was kept.  So instead of scanning the kept mask K
// (N/8 bytes) and gathering x under its set bits, this path reads exactly the kept voxels of x,
// contiguously run by run, and never reads K:
//   1. k_kept_len     klen[r] = x1 - x0 if run r's component is kept, else 0
//   2. scan           koff = exclusive prefix of klen (uint64): run r's codes are [koff[r], koff[r+1])
//   3. k_gather_runs  a warp per kept run (grid-stride), warp_segment: 16-byte loads of x, codes
//                     quantised in registers, 16-byte stores; the next run's metadata is loaded while
//                     this run's x is in flight.
// (Measured variants: chunked register gathers and a TMA-staged producer/consumer ring were slower,
// DESIGN.md section 9.)
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"
#include "segment.cuh"

namespace roix {


__global__ void k_kept_len(const RunsView R, uint32_t *klen, roix_scalars *sc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *R.err_snap = get_err(sc);
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        klen[i] = R.kept[R.parent[i]] ? R.x1[i] - R.x0[i] : 0u;
}

// Warp per kept run (grid-stride over runs): warp_segment copies-and-quantises the run's voxels to
// its stream position koff[r]; the next run's metadata is loaded while this run's x is in flight.
// One run's segment, loaded into registers ahead of its quantise-and-store (software pipeline across
// the runs of a warp): groups g = lane + 32 u of the stream-aligned body (first 16-byte block each;
// the second block of a misaligned group is the next group's first, taken from the neighbouring lane,
// except for the last group), and this lane's head / tail element.
template <typename T, int U>
struct SegRegs {
    uint64_t src0, dst0;
    uint32_t len, head, body, k, tail;
    uint4 b0[U];
    uint4 bx;   // second block of the last body group (its owner lane)
    T hv, tv;
};

template <typename T, int U>
__device__ __forceinline__ void seg_issue(const T *__restrict__ x, uint64_t src0, uint64_t dst0, uint32_t len,
                                          SegRegs<T, U> &S) {
    constexpr int V = gr_v<T>();
    const uint32_t lane = lane_id();
    S.src0 = src0;
    S.dst0 = dst0;
    S.len = len;
    S.head = (uint32_t)min((uint64_t)((V - dst0 % V) % V), (uint64_t)len);
    S.body = (len - S.head) / V;
    S.tail = len - S.head - S.body * V;
    const uint64_t s1 = src0 + S.head;
    S.k = (uint32_t)(s1 % V);
    const uint4 *xs = reinterpret_cast<const uint4 *>(x) + s1 / V;
#pragma unroll
    for (int u = 0; u < U; u++) {
        const uint32_t g = lane + 32 * u;
        S.b0[u] = g < S.body ? __ldcs(xs + g) : make_uint4(0, 0, 0, 0);
    }
    S.bx = (S.k && S.body && (S.body - 1) % 32 == lane) ? __ldcs(xs + S.body) : make_uint4(0, 0, 0, 0);
    S.hv = lane < S.head ? x[src0 + lane] : (T)0;
    S.tv = lane < S.tail ? x[s1 + (uint64_t)S.body * V + lane] : (T)0;
}

template <typename T, typename C, int QM, int U>
__device__ __forceinline__ void seg_finish(C *__restrict__ out, uint64_t cap, const SegRegs<T, U> &S, const QP &q,
                                           uint32_t &err) {
    constexpr int V = gr_v<T>();
    const uint32_t lane = lane_id();
    if (lane < S.head && S.dst0 + lane < cap) out[S.dst0 + lane] = (C)code1<T, QM>(S.hv, q, err);
    const uint64_t d1 = S.dst0 + S.head;
    uint4 *od = reinterpret_cast<uint4 *>(out + d1);
#pragma unroll
    for (int u = 0; u < U; u++) {
        // second block of group g = first block of group g + 1 (lane + 1, or lane 0 of the next u)
        uint4 nx_;
        nx_.x = __shfl_down_sync(FULL, S.b0[u].x, 1);
        nx_.y = __shfl_down_sync(FULL, S.b0[u].y, 1);
        nx_.z = __shfl_down_sync(FULL, S.b0[u].z, 1);
        nx_.w = __shfl_down_sync(FULL, S.b0[u].w, 1);
        if (u + 1 < U) {
            const uint4 w = S.b0[u + 1 < U ? u + 1 : u];
            const uint4 wr = make_uint4(__shfl_sync(FULL, w.x, 0), __shfl_sync(FULL, w.y, 0), __shfl_sync(FULL, w.z, 0),
                                        __shfl_sync(FULL, w.w, 0));
            if (lane == 31) nx_ = wr;
        }
        const uint32_t g = lane + 32 * u;
        if (g >= S.body) continue;
        const uint4 b1 = g + 1 == S.body ? S.bx : nx_;
        const uint4 cv = code_group<T, QM>(window16<T>(S.b0[u], b1, S.k), q, err);
        const uint64_t p = d1 + (uint64_t)g * V;
        if (p + V <= cap) {
            __stcs(od + g, cv);
        } else {
            const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
            for (int e = 0; e < V; e++)
                if (p + e < cap) out[p + e] = (C)(sizeof(C) == 2 ? (cw[e >> 1] >> ((e & 1) * 16)) & 0xffffu : cw[e]);
        }
    }
    const uint64_t t0 = d1 + (uint64_t)S.body * V;
    if (lane < S.tail && t0 + lane < cap) out[t0 + lane] = (C)code1<T, QM>(S.tv, q, err);
}

// Warp per kept run (grid-stride over runs), software-pipelined: while run r's codes are quantised
// and stored, run r + nw's x is already loading (SegRegs) and run r + 2 nw's metadata too.  Runs
// longer than 32 U groups go through warp_segment.
template <typename T, typename C, int QM>
__device__ __forceinline__ void gather_runs_w(const T *__restrict__ x, const RunsView &R, uint64_t nx,
                                              const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                              roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                                              uint64_t base_off, const QP &q) {
    constexpr int U = 2, V = gr_v<T>();
    const uint64_t nruns = *R.n_runs;
    const uint64_t total = nruns ? koff[nruns] : 0;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t err = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && base_off + total > capacity) err |= ROIX_ERR_CAPACITY;
    struct Meta {
        uint32_t len, row, x0;
        uint64_t ko;
    };
    auto meta = [&](uint64_t r) {
        Meta m = {0, 0, 0, 0};
        if (r < nruns) {
            m.len = klen[r];
            m.ko = koff[r];
            m.row = R.rrow[r];
            m.x0 = R.x0[r];
        }
        return m;
    };
    auto fits = [&](const Meta &m) { return m.len < (uint32_t)(32 * U * V); };   // body <= 32 U groups
    uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    Meta mc = meta(r), mn = meta(r + nw);
    SegRegs<T, U> cur, nxt;
    if (fits(mc)) seg_issue<T, U>(x, (uint64_t)mc.row * nx + mc.x0, base_off + mc.ko, mc.len, cur);
    while (r < nruns) {
        const Meta mn2 = meta(r + 2 * nw);   // prefetch
        if (r + nw < nruns && fits(mn)) seg_issue<T, U>(x, (uint64_t)mn.row * nx + mn.x0, base_off + mn.ko, mn.len, nxt);
        if (mc.len) {
            if (fits(mc)) seg_finish<T, C, QM, U>(out, capacity, cur, q, err);
            else warp_segment<T, C, QM, 2>(x, (uint64_t)mc.row * nx + mc.x0, out, base_off + mc.ko, mc.len, capacity, q, err);
        }
        r += nw;
        mc = mn;
        mn = mn2;
        cur = nxt;
    }
    if (err) set_err(sc, err);
}

template <typename T, typename C>
__global__ void __launch_bounds__(256, 3) k_gather_runs(const T *__restrict__ x, const RunsView R, uint64_t nx,
                                                     const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                                     roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                                                     const uint64_t *offset) {
    if (*R.err_snap) return;   // (not get_err: this kernel's own capacity bit must not stop its other CTAs)
    const QP q = load_qp(sc);
    const uint64_t base_off = offset ? *offset : 0;
    if constexpr (sizeof(T) == 4) {
        gather_runs_w<T, C, QM_FLOAT>(x, R, nx, koff, klen, sc, out, capacity, base_off, q);
    } else {
        switch (qmode(q)) {
        case QM_POW2: gather_runs_w<T, C, QM_POW2>(x, R, nx, koff, klen, sc, out, capacity, base_off, q); break;
        case QM_INT: gather_runs_w<T, C, QM_INT>(x, R, nx, koff, klen, sc, out, capacity, base_off, q); break;
        case QM_ONE: gather_runs_w<T, C, QM_ONE>(x, R, nx, koff, klen, sc, out, capacity, base_off, q); break;
        default: gather_runs_w<T, C, QM_FLOAT>(x, R, nx, koff, klen, sc, out, capacity, base_off, q); break;
        }
    }
}

__global__ void k_gather_total(const RunsView R, const uint64_t *koff, roix_scalars *sc) {
    if (*R.err_snap) return;
    const uint64_t n = *R.n_runs;
    sc->count += n ? koff[n] : 0;
}

}  // namespace roix

using namespace roix;

cudaError_t launch_gather(const void *x, int dtype, uint64_t nx, const RunsView &R, uint64_t cap, uint32_t *klen,
                          uint64_t *koff, uint64_t *scan_tmp, roix_scalars *sc, void *codes,
                          uint64_t capacity, const uint64_t *offset, cudaStream_t st) {
    const int grid = num_sms() * 8;
    k_kept_len<<<grid, 256, 0, st>>>(R, klen, sc);
    cudaError_t e = scan_u64_dev(klen, koff, R.n_runs, cap, scan_tmp, st);
    if (e != cudaSuccess) return e;
    const unsigned wgrid = (unsigned)num_sms() * 8;
    if (dtype == ROIX_U16)
        k_gather_runs<uint16_t, uint16_t><<<wgrid, 256, 0, st>>>((const uint16_t *)x, R, nx, koff, klen, sc,
                                                                 (uint16_t *)codes, capacity, offset);
    else
        k_gather_runs<float, int32_t><<<wgrid, 256, 0, st>>>((const float *)x, R, nx, koff, klen, sc, (int32_t *)codes,
                                                             capacity, offset);
    k_gather_total<<<1, 1, 0, st>>>(R, koff, sc);
    return cudaGetLastError();
}
