// scan.cu -- the single-pass prefix sum declared in scan.cuh.
#include "scan.cuh"

namespace roix {

constexpr uint64_t ST_AGG = 1ull << 62, ST_PRE = 2ull << 62, ST_VAL = (1ull << 62) - 1;

__device__ __forceinline__ uint64_t ld_state(const uint64_t *p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_state(uint64_t *p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// tmp[0 .. nb): tile states (zeroed by the launcher); tmp[nb]: the total
template <typename O>
__global__ void __launch_bounds__(SCAN_T) k_scan_dlb(const uint32_t *in, O *out, const uint64_t *len_dev, uint64_t len,
                                                     uint64_t *tmp, uint64_t nb) {
    __shared__ uint64_t wsum[SCAN_T / 32];
    __shared__ uint64_t s_pre;
    const uint64_t n = len_dev ? *len_dev : len;
    const uint64_t t = blockIdx.x;
    const uint64_t base = t * SCAN_TILE;
    if (base > n) return;   // nobody waits on tiles past the one holding index n
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    // thread owns elements base + tid*V .. +V (contiguous)
    uint32_t v[SCAN_V];
    uint64_t loc = 0;
#pragma unroll
    for (int k = 0; k < SCAN_V; k++) {
        const uint64_t i = base + (uint64_t)threadIdx.x * SCAN_V + k;
        v[k] = i < n ? in[i] : 0u;
        loc += v[k];
    }
    const uint64_t x = warp_incl_scan(loc);
    if (lane == 31) wsum[warp] = x;
    __syncthreads();
    uint64_t wpre = 0, agg = 0;
#pragma unroll
    for (int w = 0; w < SCAN_T / 32; w++) {
        const uint64_t s = wsum[w];
        if (w < (int)warp) wpre += s;
        agg += s;
    }
    if (warp == 0) {
        uint64_t pre = 0;
        if (t == 0) {
            if (lane == 0) st_state(tmp, ST_PRE | agg);
        } else {
            if (lane == 0) st_state(tmp + t, ST_AGG | agg);
            // look back over the predecessors, 32 at a time, until one has published its prefix
            int64_t j = (int64_t)t - 1;
            while (true) {
                const int64_t idx = j - (int64_t)lane;
                uint64_t sv = ST_PRE;   // before tile 0: a zero prefix
                if (idx >= 0) {
                    do {
                        sv = ld_state(tmp + idx);
                    } while ((sv >> 62) == 0);
                }
                const uint32_t pm = __ballot_sync(FULL, (sv >> 62) == 2);
                const uint32_t lim = pm ? (uint32_t)(__ffs(pm) - 1) : 31u;
                uint64_t add = lane <= lim ? (sv & ST_VAL) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) add += __shfl_xor_sync(FULL, add, d);
                pre += add;
                if (pm) break;
                j -= 32;
            }
            if (lane == 0) st_state(tmp + t, ST_PRE | (pre + agg));
        }
        if (lane == 0) s_pre = pre;
    }
    __syncthreads();
    uint64_t run = s_pre + wpre + x - loc;
#pragma unroll
    for (int k = 0; k < SCAN_V; k++) {
        const uint64_t i = base + (uint64_t)threadIdx.x * SCAN_V + k;
        if (i < n) out[i] = (O)run;
        run += v[k];
    }
    // the tile holding index n writes the total
    if (n - base < SCAN_TILE && threadIdx.x == 0) {
        const uint64_t tot = s_pre + agg;
        out[n] = sizeof(O) == 4 ? (O)(tot > 0xffffffffull ? 0xffffffffull : tot) : (O)tot;
        tmp[nb] = tot;
    }
}

template <typename O>
cudaError_t scan_impl(const uint32_t *in, O *out, const uint64_t *len_dev, uint64_t len, uint64_t maxlen, uint64_t *tmp,
                      cudaStream_t st) {
    const uint64_t nb = scan_nblocks(maxlen);
    cudaError_t e = cudaMemsetAsync(tmp, 0, nb * sizeof(uint64_t), st);
    if (e != cudaSuccess) return e;
    k_scan_dlb<O><<<(unsigned)nb, SCAN_T, 0, st>>>(in, out, len_dev, len, tmp, nb);
    return cudaGetLastError();
}

template cudaError_t scan_impl<uint32_t>(const uint32_t *, uint32_t *, const uint64_t *, uint64_t, uint64_t, uint64_t *,
                                         cudaStream_t);
template cudaError_t scan_impl<uint64_t>(const uint32_t *, uint64_t *, const uint64_t *, uint64_t, uint64_t, uint64_t *,
                                         cudaStream_t);

}  // namespace roix
