// scan.cuh -- exclusive prefix sum of uint32 counts in one pass (decoupled look-back: every tile
// publishes its aggregate, then its inclusive prefix, and each tile's first warp sums its
// predecessors' published values 32 at a time).  out[len] receives the total (saturated to uint32 for
// uint32 outputs); the exact uint64 total is kept at scan_total_ptr(tmp, maxlen).  The length may
// live in device memory (scan_u32_dev / scan_u64_dev): elements at or past it are treated as 0 and
// not written.  in and out may alias.
#pragma once
#include "common.cuh"

namespace roix {

constexpr int SCAN_T = 256, SCAN_V = 32, SCAN_TILE = SCAN_T * SCAN_V;

// tiles of a scan of up to maxlen elements (one more than needed, so the tile holding index len exists)
__host__ __device__ inline uint64_t scan_nblocks(uint64_t maxlen) { return maxlen / SCAN_TILE + 1; }
inline uint64_t scan_tmp_elems(uint64_t maxlen) { return scan_nblocks(maxlen) + 2; }
inline const uint64_t *scan_total_ptr(const uint64_t *tmp, uint64_t maxlen) { return tmp + scan_nblocks(maxlen); }

template <typename O>
cudaError_t scan_impl(const uint32_t *in, O *out, const uint64_t *len_dev, uint64_t len, uint64_t maxlen, uint64_t *tmp,
                      cudaStream_t st);

// host-known length; out must hold len + 1 elements
inline cudaError_t scan_u32(const uint32_t *in, uint32_t *out, uint64_t len, uint64_t *tmp, cudaStream_t st) {
    return scan_impl(in, out, nullptr, len, len, tmp, st);
}
// uint64 offsets (totals beyond 2^32); out must hold len + 1 elements
inline cudaError_t scan_u32_u64(const uint32_t *in, uint64_t *out, uint64_t len, uint64_t *tmp, cudaStream_t st) {
    return scan_impl(in, out, nullptr, len, len, tmp, st);
}
// device-resident length (<= maxlen); out must hold maxlen + 1 elements
inline cudaError_t scan_u32_dev(const uint32_t *in, uint32_t *out, const uint64_t *len_dev, uint64_t maxlen,
                                uint64_t *tmp, cudaStream_t st) {
    return scan_impl(in, out, len_dev, 0, maxlen, tmp, st);
}

// device-resident length, uint64 offsets; out must hold maxlen + 1 elements
inline cudaError_t scan_u64_dev(const uint32_t *in, uint64_t *out, const uint64_t *len_dev, uint64_t maxlen,
                                uint64_t *tmp, cudaStream_t st) {
    return scan_impl(in, out, len_dev, 0, maxlen, tmp, st);
}

}  // namespace roix
