// k_gather.cu -- a1+a8 EXTRACT from the kept x-runs of a6/a7 (roix_extract_runs): never reads K,
// reads x only under kept runs.  The code stream is the concatenation, in run order (= increasing
// linear index, G-17), of the quantised voxels of every run whose component was kept (P:316-334's
// pixel sections, without the gaps): k_kept_len + scan give every run its stream range, k_rx_runs
// fills them.  The pipeline takes this form for uint16 volumes labelled in 3-D and the mask-driven
// roix_extract (k_compact.cu) otherwise; DESIGN.md section 9 compares them.
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


// ---------------------------------------------------------------- run-driven extraction
// k_rx_runs: a warp per batch of 32 consecutive runs (lane k: run b 32 + k; its stream range
// [koff, koff + klen), klen = 0 for a dropped run).  The batch's kept runs are cut into the aligned
// 16-byte output vectors they touch (nv_k of them), numbered through the batch by a warp scan; the
// warp then takes 32 of those vectors per pass, lane t finding its run by a binary search over the
// scan.  A vector is one window of x (two aligned 16-byte loads + a shift), quantised in registers:
// inside its run it is one 16-byte store; at a run end only the run's own codes are stored (the rest
// of that vector belongs to the neighbouring runs, which store their own), code by code.  K is never
// read, x only under kept runs, and every pass keeps 32 vectors' loads in flight whatever the run
// lengths.
template <typename T, typename C, int QM>
__device__ __forceinline__ void rr_batch(const T *__restrict__ x, uint64_t n, const RunsView &R, uint64_t nx,
                                         const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                         uint64_t nruns, uint64_t b, uint64_t off0, C *__restrict__ out,
                                         uint64_t capacity, const QP &q, uint32_t &err) {
    constexpr int V = gr_v<T>();
    const uint32_t lane = lane_id();
    const uint64_t r = b * 32 + lane;
    const bool ok = r < nruns;
    const uint32_t len = ok ? klen[r] : 0u;
    const uint64_t dst = ok ? koff[r] + off0 : 0ull;                          // stream position of its first code
    const uint64_t src = len ? (uint64_t)R.rrow[r] * nx + R.x0[r] : 0ull;    // linear index of its first voxel
    const uint64_t a0 = dst - dst % V;                                         // its first aligned vector
    const uint32_t nv = len ? (uint32_t)((dst + len - a0 + V - 1) / V) : 0u;
    const uint32_t incl = warp_incl_scan(nv);
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    const uint32_t excl = incl - nv;
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const uint64_t ng = n / V;   // whole 16-byte groups of x
    for (uint32_t p0 = 0; p0 < tot; p0 += 32) {
        const uint32_t t = p0 + lane;
        // the lane's run: the last k with excl_k <= t (runs with nv = 0 share their successor's excl)
        uint32_t k = 0;
#pragma unroll
        for (uint32_t bb = 16; bb >= 1; bb >>= 1) {
            const uint32_t e = __shfl_sync(FULL, excl, k + bb);
            if (k + bb < 32 && e <= t) k += bb;
        }
        const uint32_t ek = __shfl_sync(FULL, excl, k), nk = __shfl_sync(FULL, nv, k);
        const uint32_t lk = __shfl_sync(FULL, len, k);
        const uint64_t dk = __shfl_sync(FULL, dst, k), sk = __shfl_sync(FULL, src, k);
        if (t >= tot || t - ek >= nk) continue;
        const uint64_t A = (dk - dk % V) + (uint64_t)V * (t - ek);           // this vector's first position
        const uint32_t lo = A < dk ? (uint32_t)(dk - A) : 0u;                // its codes [lo, hi) belong to run k
        const uint32_t hi = A + V <= dk + lk ? (uint32_t)V : (uint32_t)(dk + lk - A);
        const int64_t spos = (int64_t)(sk + A) - (int64_t)dk;                // source of position A (may be < sk)
        if (spos >= 0 && (uint64_t)spos / V + 2 <= ng && A + V <= capacity) {
            const uint64_t g = (uint64_t)spos / V;
            const uint32_t kk = (uint32_t)((uint64_t)spos % V);
            const uint4 b0 = __ldcs(x4 + g);
            const uint4 b1 = kk ? __ldcs(x4 + g + 1) : b0;
            const uint4 c = code_group<T, QM>(window16<T>(b0, b1, kk), q, err);
            if (lo == 0 && hi == (uint32_t)V) {
                __stcs(reinterpret_cast<uint4 *>(out + A), c);
            } else {
                const uint32_t cw[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
                for (int h = 0; h < V; h++) {
                    if ((uint32_t)h < lo || (uint32_t)h >= hi) continue;
                    uint32_t v;
                    if constexpr (sizeof(C) == 2) v = (h & 1) ? cw[h >> 1] >> 16 : cw[h >> 1] & 0xffffu;
                    else v = cw[h];
                    out[A + h] = (C)v;
                }
            }
        } else {   // the volume's ends or the capacity edge: code by code
            for (uint32_t h = lo; h < hi; h++) {
                if (A + h >= capacity) break;
                out[A + h] = (C)code1<T, QM>(x[(uint64_t)spos + h], q, err);
            }
        }
    }
}

// 8 CTAs per SM (full occupancy: 32 registers, 140 B of spills): the kernel is latency-bound (42 %
// issue at 4 CTAs per SM), and more warps keep more passes in flight -- same box, C4 / C5 extract:
// 4 CTAs 6.65 / 4.06 ms, 5: 6.29 / 3.73, 6: 5.93 / 3.53, 8: 5.50 / 3.25
template <typename T, typename C>
__global__ void __launch_bounds__(256, 8) k_rx_runs(const T *__restrict__ x, uint64_t n, const RunsView R, uint64_t nx,
                                                 const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                                 roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                                                 const uint64_t *offset) {
    if (*R.err_snap) return;
    const uint64_t nruns = *R.n_runs;
    const uint64_t total = nruns ? koff[nruns] : 0;
    const uint64_t off0 = offset ? *offset : 0;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && off0 + total > capacity) err |= ROIX_ERR_CAPACITY;
    const uint64_t nb = (nruns + 31) / 32, nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t b = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < nb; b += nw) {
        if constexpr (sizeof(T) == 4) {
            rr_batch<T, C, QM_FLOAT>(x, n, R, nx, koff, klen, nruns, b, off0, out, capacity, q, err);
        } else {
            switch (qmode(q)) {
            case QM_POW2: rr_batch<T, C, QM_POW2>(x, n, R, nx, koff, klen, nruns, b, off0, out, capacity, q, err); break;
            case QM_INT: rr_batch<T, C, QM_INT>(x, n, R, nx, koff, klen, nruns, b, off0, out, capacity, q, err); break;
            case QM_ONE: rr_batch<T, C, QM_ONE>(x, n, R, nx, koff, klen, nruns, b, off0, out, capacity, q, err); break;
            default: rr_batch<T, C, QM_FLOAT>(x, n, R, nx, koff, klen, nruns, b, off0, out, capacity, q, err); break;
            }
        }
    }
    err = __reduce_or_sync(FULL, err);
    if (err && lane_id() == 0) set_err(sc, err);
}

}  // namespace roix

using namespace roix;



cudaError_t launch_runx(const void *x, int dtype, uint64_t n, uint64_t nx, const RunsView &R, uint64_t cap, uint32_t *klen,
                        uint64_t *koff, uint64_t *scan_tmp, roix_scalars *sc, void *codes,
                        uint64_t capacity, const uint64_t *offset, cudaStream_t st) {
    const int grid = num_sms() * 8;
    k_kept_len<<<grid, 256, 0, st>>>(R, klen, sc);
    cudaError_t e = scan_u64_dev(klen, koff, R.n_runs, cap, scan_tmp, st);
    if (e != cudaSuccess) return e;
    // persistent warps over 32-run batches: one wave of resident CTAs
    static int occ16 = 0, occ32 = 0;
    if (!occ16) {
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ16, k_rx_runs<uint16_t, uint16_t>, 256, 0);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ32, k_rx_runs<float, int32_t>, 256, 0);
        if (occ16 < 1) occ16 = 1;
        if (occ32 < 1) occ32 = 1;
    }
    const unsigned pgrid = (unsigned)num_sms() * (dtype == ROIX_U16 ? occ16 : occ32);
    if (dtype == ROIX_U16)
        k_rx_runs<uint16_t, uint16_t><<<pgrid, 256, 0, st>>>((const uint16_t *)x, n, R, nx, koff, klen, sc,
                                                            (uint16_t *)codes, capacity, offset);
    else
        k_rx_runs<float, int32_t><<<pgrid, 256, 0, st>>>((const float *)x, n, R, nx, koff, klen, sc,
                                                        (int32_t *)codes, capacity, offset);
    k_gather_total<<<1, 1, 0, st>>>(R, koff, sc);
    return cudaGetLastError();
}
