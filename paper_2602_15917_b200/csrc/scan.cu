// scan.cu -- the prefix-sum kernels declared in scan.cuh.
#include "scan.cuh"

namespace roix {

__device__ __forceinline__ uint64_t block_sum_u64(uint64_t v, uint64_t *sh) {
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
    if (lane_id() == 0) sh[threadIdx.x >> 5] = v;
    __syncthreads();
    uint64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); w++) t += sh[w];
    __syncthreads();
    return t;
}

__global__ void __launch_bounds__(SCAN_T) k_scan_reduce(const uint32_t *in, const uint64_t *len_dev, uint64_t len,
                                                        uint64_t *tmp) {
    __shared__ uint64_t sh[SCAN_T / 32];
    const uint64_t n = len_dev ? *len_dev : len;
    const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    uint64_t s = 0;
    if (base < n) {
#pragma unroll
        for (int k = 0; k < SCAN_V; k++) {
            uint64_t i = base + (uint64_t)k * SCAN_T + threadIdx.x;
            if (i < n) s += in[i];
        }
    }
    s = block_sum_u64(s, sh);
    if (threadIdx.x == 0) tmp[blockIdx.x] = s;
}

// one CTA: exclusive scan of nb tile sums in place; total at tmp[nb]
__global__ void __launch_bounds__(1024) k_scan_blocks(uint64_t *tmp, uint64_t nb) {
    __shared__ uint64_t sh[32];
    __shared__ uint64_t carry;
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (uint64_t b0 = 0; b0 < nb; b0 += blockDim.x) {
        uint64_t i = b0 + threadIdx.x;
        uint64_t v = i < nb ? tmp[i] : 0;
        uint64_t x = warp_incl_scan(v);
        if (lane_id() == 31) sh[threadIdx.x >> 5] = x;
        __syncthreads();
        if (threadIdx.x < 32) {
            uint64_t w = threadIdx.x < (blockDim.x >> 5) ? sh[threadIdx.x] : 0;
            w = warp_incl_scan(w);
            sh[threadIdx.x] = w;
        }
        __syncthreads();
        uint64_t wpre = (threadIdx.x >> 5) ? sh[(threadIdx.x >> 5) - 1] : 0;
        uint64_t c = carry;
        if (i < nb) tmp[i] = c + wpre + x - v;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = c + wpre + x;
        __syncthreads();
    }
    if (threadIdx.x == 0) tmp[nb] = carry;
}

template <typename O>
__global__ void __launch_bounds__(SCAN_T) k_scan_down(const uint32_t *in, O *out, const uint64_t *len_dev,
                                                      uint64_t len, const uint64_t *tmp, uint64_t nb) {
    __shared__ uint64_t sh[SCAN_T / 32];
    const uint64_t n = len_dev ? *len_dev : len;
    const uint64_t base = (uint64_t)blockIdx.x * SCAN_TILE;
    if (base < n) {
        // thread t owns elements base + t*V .. +V (contiguous) for a simple sequential local scan
        uint32_t v[SCAN_V];
        uint64_t loc = 0;
#pragma unroll
        for (int k = 0; k < SCAN_V; k++) {
            uint64_t i = base + (uint64_t)threadIdx.x * SCAN_V + k;
            v[k] = i < n ? in[i] : 0u;
            loc += v[k];
        }
        uint64_t x = warp_incl_scan(loc);
        if (lane_id() == 31) sh[threadIdx.x >> 5] = x;
        __syncthreads();
        uint64_t wpre = 0;
        for (int w = 0; w < (int)(threadIdx.x >> 5); w++) wpre += sh[w];
        uint64_t run = tmp[blockIdx.x] + wpre + x - loc;
#pragma unroll
        for (int k = 0; k < SCAN_V; k++) {
            uint64_t i = base + (uint64_t)threadIdx.x * SCAN_V + k;
            if (i < n) out[i] = (O)run;
            run += v[k];
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        uint64_t t = tmp[nb];
        out[n] = sizeof(O) == 4 ? (O)(t > 0xffffffffull ? 0xffffffffull : t) : (O)t;
    }
}

template <typename O>
cudaError_t scan_impl(const uint32_t *in, O *out, const uint64_t *len_dev, uint64_t len, uint64_t maxlen, uint64_t *tmp,
                      cudaStream_t st) {
    const uint64_t nb = scan_nblocks(maxlen);
    if (nb == 0) {
        // empty: total 0
        cudaError_t e = cudaMemsetAsync(tmp, 0, 8, st);
        if (e != cudaSuccess) return e;
        return cudaMemsetAsync(out, 0, sizeof(O), st);
    }
    k_scan_reduce<<<(unsigned)nb, SCAN_T, 0, st>>>(in, len_dev, len, tmp);
    k_scan_blocks<<<1, 1024, 0, st>>>(tmp, nb);
    k_scan_down<O><<<(unsigned)nb, SCAN_T, 0, st>>>(in, out, len_dev, len, tmp, nb);
    return cudaGetLastError();
}

template cudaError_t scan_impl<uint32_t>(const uint32_t *, uint32_t *, const uint64_t *, uint64_t, uint64_t, uint64_t *,
                                         cudaStream_t);
template cudaError_t scan_impl<uint64_t>(const uint32_t *, uint64_t *, const uint64_t *, uint64_t, uint64_t, uint64_t *,
                                         cudaStream_t);

}  // namespace roix
