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
template <typename T, typename C, int QM>
__device__ __forceinline__ void gather_runs_w(const T *__restrict__ x, const RunsView &R, uint64_t nx,
                                              const uint64_t *__restrict__ koff, const uint32_t *__restrict__ klen,
                                              roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                                              uint64_t base_off, const QP &q) {
    const uint64_t nruns = *R.n_runs;
    const uint64_t total = nruns ? koff[nruns] : 0;
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t err = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0 && base_off + total > capacity) err |= ROIX_ERR_CAPACITY;
    uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint32_t len = 0, row = 0, x0 = 0;
    uint64_t ko = 0;
    if (r < nruns) {
        len = klen[r];
        ko = koff[r];
        row = R.rrow[r];
        x0 = R.x0[r];
    }
    while (r < nruns) {
        const uint64_t rn = r + nw;
        uint32_t len2 = 0, row2 = 0, x02 = 0;
        uint64_t ko2 = 0;
        if (rn < nruns) {   // prefetch
            len2 = klen[rn];
            ko2 = koff[rn];
            row2 = R.rrow[rn];
            x02 = R.x0[rn];
        }
        if (len) warp_segment<T, C, QM, 2>(x, (uint64_t)row * nx + x0, out, base_off + ko, len, capacity, q, err);
        r = rn;
        len = len2;
        ko = ko2;
        row = row2;
        x0 = x02;
    }
    if (err) set_err(sc, err);
}

template <typename T, typename C>
__global__ void __launch_bounds__(256) k_gather_runs(const T *__restrict__ x, const RunsView R, uint64_t nx,
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
