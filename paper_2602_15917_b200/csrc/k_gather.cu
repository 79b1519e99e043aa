// k_gather.cu -- a1+a8 EXTRACT from the kept x-runs of a6/a7 (roix_extract_runs): never reads K,
// reads x only under kept runs (the output-driven kernels below).  The mask-driven roix_extract
// (k_compact.cu) is the pipeline default; DESIGN.md section 9 compares them.
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

__global__ void k_gather_total(const RunsView R, const uint64_t *koff, roix_scalars *sc) {
    if (*R.err_snap) return;
    const uint64_t n = *R.n_runs;
    sc->count += n ? koff[n] : 0;
}


// ---------------------------------------------------------------- output-driven run extraction
// a1+a8 EXTRACT from the kept x-runs of a6/a7 (roix_extract_runs), output-driven.
//
// The code stream is the concatenation, in run order (= increasing linear index, G-17), of the
// quantised voxels of every run whose component was kept (P:316-334's pixel sections, without the
// gaps).  After a6/a7 every run r has its stream range [koff[r], koff[r] + klen[r]) (klen = 0 for a
// dropped run; koff = exclusive scan), so every aligned 16-byte output vector of the stream can find
// its source directly -- no kept mask is read and x is read only under kept runs:
//   1. k_kept_len (k_gather.cu) + scan: klen, koff;
//   2. k_rx_map: task t (RX_TV consecutive output vectors) -> the run holding its first code;
//   3. k_rx_extract: persistent warps over tasks; per step the warp covers 32 vectors (one per lane)
//      with a batch of 32 consecutive runs in its lanes (lane k = run r_cur + k).  A vector inside one
//      run is one 16-byte window of x (two aligned loads + a funnel shift), quantised in registers
//      and stored with one 16-byte store; a vector across one run end takes the rest of that run and
//      the head of the next non-empty run (two windows, one select); anything else (three or more
//      runs in 8 codes, the stream's ragged ends, the capacity edge) goes element by element.


constexpr int RX_STEPS = 8;                // 32-vector steps per task
constexpr int RX_TV = 32 * RX_STEPS;       // vectors per task

// k_rx_map: task_run[t] = the run holding task t's first code (t >= 1: code t*TC - d0; t = 0: code 0)
__global__ void k_rx_map(const RunsView R, const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                         uint32_t vpg, const uint64_t *offset, uint32_t *task_run) {
    if (*R.err_snap) return;
    const uint64_t n = *R.n_runs;
    const uint64_t tc = (uint64_t)RX_TV * vpg;
    const uint64_t d0 = (offset ? *offset : 0) % vpg;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t l = klen[r];
        if (!l) continue;
        const uint64_t a = koff[r] + d0, b = a + l;
        if (koff[r] == 0) task_run[0] = (uint32_t)r;
        for (uint64_t t = (a + tc - 1) / tc; t * tc < b; t++)
            if (t) task_run[t] = (uint32_t)r;
    }
}

// last run (global index) with koff <= j, by binary search over koff[lo .. hi)
__device__ __forceinline__ uint64_t rx_find(const uint64_t *__restrict__ koff, uint64_t lo, uint64_t hi, uint64_t j) {
    while (hi - lo > 1) {
        const uint64_t mid = (lo + hi) >> 1;
        if (koff[mid] <= j) lo = mid;
        else hi = mid;
    }
    return lo;
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void rx_task(const T *__restrict__ x, const RunsView &R, uint64_t nx,
                                        const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                        uint64_t nruns, uint64_t total, uint64_t t, uint32_t r_first, uint64_t off0,
                                        C *__restrict__ out, uint64_t capacity, const QP &q, uint32_t &err) {
    constexpr int V = gr_v<T>();   // codes per 16-byte vector = voxels per 16-byte block of x
    const uint32_t lane = lane_id();
    const uint64_t d0 = off0 % V, ab = off0 - d0;   // output vector 0 starts at code index -d0
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    uint64_t rc = r_first;
    for (int s = 0; s < RX_STEPS; s++) {
        // this step's vectors: (t RX_TV + 32 s + lane) relative to ab; first code of the lane's vector
        const int64_t jw = (int64_t)(t * RX_TV + 32 * (uint64_t)s) * V - (int64_t)d0;
        if (jw >= (int64_t)total) return;
        const int64_t jv = jw + (int64_t)lane * V;
        // the batch: lane k holds run rc + k (koff, klen, source index of its first voxel)
        const uint64_t rk = rc + lane;
        const bool ok = rk < nruns;
        const uint64_t ko = ok ? koff[rk] : ~0ull;
        const uint32_t kl = ok ? klen[rk] : 0u;
        const uint64_t src = ok ? (uint64_t)R.rrow[rk] * nx + R.x0[rk] : 0ull;
        const int64_t jend = jw + 32 * V;   // first code after this step
        // does the batch reach past this step?  (run rc + 31 starts at or after jend)
        const uint64_t ko31 = __shfl_sync(FULL, ko, 31);
        const bool covered = ko31 >= (uint64_t)max(jend, (int64_t)0);
        // lane's run within the batch: last k with koff_k <= max(jv, 0)
        const uint64_t jq = (uint64_t)max(jv, (int64_t)0);
        int k = 0;
#pragma unroll
        for (int b = 16; b >= 1; b >>= 1) {
            const uint64_t kk = __shfl_sync(FULL, ko, k + b);
            if (k + b < 32 && kk <= jq) k += b;
        }
        const uint64_t kor = __shfl_sync(FULL, ko, k);
        const uint32_t klr = __shfl_sync(FULL, kl, k);
        const uint64_t srcr = __shfl_sync(FULL, src, k);
        // the next non-empty run after k within the batch (for a vector across a run end)
        const uint32_t ne_mask = __ballot_sync(FULL, kl != 0) & ~(k >= 31 ? FULL : ((2u << k) - 1u));
        const int k2 = ne_mask ? __ffs(ne_mask) - 1 : -1;
        const uint64_t ko2 = __shfl_sync(FULL, ko, k2 < 0 ? 0 : k2);
        const uint32_t kl2 = __shfl_sync(FULL, kl, k2 < 0 ? 0 : k2);
        const uint64_t src2 = __shfl_sync(FULL, src, k2 < 0 ? 0 : k2);
        const bool in_range = jv >= 0 && jv + V <= (int64_t)total && ab + (uint64_t)(jv + (int64_t)d0) + V <= capacity;
        const uint64_t a_left = covered && jv >= 0 && (uint64_t)jv < kor + klr ? kor + klr - (uint64_t)jv : 0;   // codes left in run k
        // the source of this lane's vector two steps ahead into L2 when the run continues that far
        if (covered && jv >= 0 && (uint64_t)jv + 65 * V <= kor + klr)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(x + srcr + ((uint64_t)jv - kor) + 64 * V));
        bool done = false;
        if (covered && in_range && a_left > 0) {
            C *dst = out + ab + (uint64_t)(jv + (int64_t)d0);
            if (a_left >= V) {   // one window
                const uint64_t sp = srcr + ((uint64_t)jv - kor);
                const uint32_t kk = (uint32_t)(sp % V);
                const uint4 b0 = __ldcs(x4 + sp / V);
                const uint4 b1 = kk ? __ldcs(x4 + sp / V + 1) : b0;
                __stcs(reinterpret_cast<uint4 *>(dst), code_group<T, QM>(window16<T>(b0, b1, kk), q, err));
                done = true;
            } else if (k2 >= 0 && ko2 == (uint64_t)jv + a_left && kl2 >= V - a_left) {   // two windows
                const uint64_t sp = srcr + ((uint64_t)jv - kor);
                const uint32_t kk = (uint32_t)(sp % V), k2s = (uint32_t)(src2 % V);
                const uint4 b0 = __ldcs(x4 + sp / V);
                const uint4 b1 = kk ? __ldcs(x4 + sp / V + 1) : b0;
                const uint4 c0 = __ldcs(x4 + src2 / V);
                const uint4 c1 = k2s ? __ldcs(x4 + src2 / V + 1) : c0;
                const uint4 w1 = window16<T>(b0, b1, kk);
                const uint4 w2 = window16<T>(c0, c1, k2s);
                // codes [0, a) from w1, [a, V) from the head of w2: w2 moved up by a elements
                const uint32_t a = (uint32_t)a_left;
                const uint4 z = make_uint4(0, 0, 0, 0);
                const uint4 w2s = window16<T>(z, w2, V - a);
                const uint32_t e1 = a * (uint32_t)sizeof(T);   // bytes from w1
                uint32_t m[4];
#pragma unroll
                for (int i = 0; i < 4; i++) {
                    const uint32_t lo = 4 * i;
                    m[i] = e1 >= lo + 4 ? FULL : (e1 <= lo ? 0u : (1u << (8 * (e1 - lo))) - 1u);
                }
                const uint4 w = make_uint4((w1.x & m[0]) | (w2s.x & ~m[0]), (w1.y & m[1]) | (w2s.y & ~m[1]),
                                           (w1.z & m[2]) | (w2s.z & ~m[2]), (w1.w & m[3]) | (w2s.w & ~m[3]));
                __stcs(reinterpret_cast<uint4 *>(dst), code_group<T, QM>(w, q, err));
                done = true;
            }
        }
        if (!done) {
            // element by element: the stream's ragged ends, the capacity edge, three or more runs in
            // one vector, or more than 32 run starts in this step
            for (int h = 0; h < V; h++) {
                const int64_t j = jv + h;
                if (j < 0 || j >= (int64_t)total) continue;
                const uint64_t pos = ab + (uint64_t)(j + (int64_t)d0);
                if (pos >= capacity) continue;
                const uint64_t r = rx_find(koff, rc, nruns, (uint64_t)j);
                const T v = x[(uint64_t)R.rrow[r] * nx + R.x0[r] + ((uint64_t)j - koff[r])];
                out[pos] = (C)code1<T, QM>(v, q, err);
            }
        }
        // the run holding the next step's first code
        if (covered) {
            const uint32_t le = __ballot_sync(FULL, ok && ko <= (uint64_t)max(jend, (int64_t)0));
            rc += 31 - __clz(le | 1u);
        } else {
            rc = rx_find(koff, rc, nruns, (uint64_t)max(jend, (int64_t)0));
        }
    }
}

template <typename T, typename C>
__global__ void __launch_bounds__(256) k_rx_extract(const T *__restrict__ x, const RunsView R, uint64_t nx,
                                                    const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                                    const uint32_t *__restrict__ task_run, roix_scalars *sc,
                                                    C *__restrict__ out, uint64_t capacity, const uint64_t *offset) {
    if (*R.err_snap) return;   // (not get_err: this kernel's own capacity bit must not stop its other CTAs)
    constexpr int V = gr_v<T>();
    const uint64_t nruns = *R.n_runs;
    const uint64_t total = nruns ? koff[nruns] : 0;
    const uint64_t off0 = offset ? *offset : 0;
    const uint64_t ntasks = (total + off0 % V + (uint64_t)RX_TV * V - 1) / ((uint64_t)RX_TV * V);
    const QP q = load_qp(sc);
    uint32_t err = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && off0 + total > capacity) err |= ROIX_ERR_CAPACITY;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t t = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntasks; t += nw) {
        const uint32_t rf = task_run[t];
        if constexpr (sizeof(T) == 4) {
            rx_task<T, C, QM_FLOAT>(x, R, nx, koff, klen, nruns, total, t, rf, off0, out, capacity, q, err);
        } else {
            switch (qmode(q)) {
            case QM_POW2: rx_task<T, C, QM_POW2>(x, R, nx, koff, klen, nruns, total, t, rf, off0, out, capacity, q, err); break;
            case QM_INT: rx_task<T, C, QM_INT>(x, R, nx, koff, klen, nruns, total, t, rf, off0, out, capacity, q, err); break;
            case QM_ONE: rx_task<T, C, QM_ONE>(x, R, nx, koff, klen, nruns, total, t, rf, off0, out, capacity, q, err); break;
            default: rx_task<T, C, QM_FLOAT>(x, R, nx, koff, klen, nruns, total, t, rf, off0, out, capacity, q, err); break;
            }
        }
    }
    if (err) set_err(sc, err);
}

}  // namespace roix

using namespace roix;


uint64_t runx_task_entries(uint64_t n) { return n / (RX_TV * 4) + 2; }

cudaError_t launch_runx(const void *x, int dtype, uint64_t nx, const RunsView &R, uint64_t cap, uint32_t *klen,
                        uint64_t *koff, uint64_t *scan_tmp, uint32_t *task_run, roix_scalars *sc, void *codes,
                        uint64_t capacity, const uint64_t *offset, cudaStream_t st) {
    const int grid = num_sms() * 8;
    k_kept_len<<<grid, 256, 0, st>>>(R, klen, sc);
    cudaError_t e = scan_u64_dev(klen, koff, R.n_runs, cap, scan_tmp, st);
    if (e != cudaSuccess) return e;
    const uint32_t V = dtype == ROIX_U16 ? 8u : 4u;
    k_rx_map<<<grid, 256, 0, st>>>(R, koff, klen, V, offset, task_run);
    // persistent warps: one wave of resident CTAs
    static int occ16 = 0, occ32 = 0;
    if (!occ16) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ16, k_rx_extract<uint16_t, uint16_t>, 256, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ32, k_rx_extract<float, int32_t>, 256, 0);
        if (occ16 < 1) occ16 = 1;
        if (occ32 < 1) occ32 = 1;
    }
    const unsigned pgrid = (unsigned)num_sms() * (dtype == ROIX_U16 ? occ16 : occ32);
    if (dtype == ROIX_U16)
        k_rx_extract<uint16_t, uint16_t><<<pgrid, 256, 0, st>>>((const uint16_t *)x, R, nx, koff, klen, task_run, sc,
                                                               (uint16_t *)codes, capacity, offset);
    else
        k_rx_extract<float, int32_t><<<pgrid, 256, 0, st>>>((const float *)x, R, nx, koff, klen, task_run, sc,
                                                           (int32_t *)codes, capacity, offset);
    k_gather_total<<<1, 1, 0, st>>>(R, koff, sc);
    return cudaGetLastError();
}
