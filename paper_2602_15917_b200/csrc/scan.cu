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

// tmp[0 .. nb): tile states (zeroed by the launcher); tmp[nb]: the total.
// A tile is SCAN_T / 32 warps x SCAN_CH chunks of 128 elements; lane l of a warp holds elements
// 4 l .. 4 l + 3 of each of its chunks (one coalesced 16-byte load per chunk when the tile is whole and
// the pointers aligned), so the warp scans chunk by chunk with a running carry.  Large tiles keep the
// look-back chain short (the first wave of tiles resolves its prefixes 32 tiles per round).
template <typename O>
__global__ void __launch_bounds__(SCAN_T) k_scan_dlb(const uint32_t *in, O *out, const uint64_t *len_dev, uint64_t len,
                                                     uint64_t *tmp, uint64_t nb) {
    constexpr int CH = SCAN_TILE / SCAN_T / 4;   // chunks of 128 elements per warp
    __shared__ uint64_t wsum[SCAN_T / 32];
    __shared__ uint64_t s_pre;
    const uint64_t n = len_dev ? *len_dev : len;
    const uint64_t t = blockIdx.x;
    const uint64_t base = t * SCAN_TILE;
    if (base > n) return;   // nobody waits on tiles past the one holding index n
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint64_t wbase = base + (uint64_t)warp * CH * 128;
    const bool whole = base + SCAN_TILE <= n;
    const bool vin = whole && ((uintptr_t)in & 15) == 0;
    uint4 q[CH];
    uint64_t ex[CH];   // exclusive prefix of the lane's four elements inside the warp's region
    uint64_t carry = 0;
#pragma unroll
    for (int c = 0; c < CH; c++) {
        const uint64_t i = wbase + (uint64_t)c * 128 + 4 * lane;
        if (vin) {
            q[c] = reinterpret_cast<const uint4 *>(in + i)[0];
        } else {
            q[c].x = i < n ? in[i] : 0u;
            q[c].y = i + 1 < n ? in[i + 1] : 0u;
            q[c].z = i + 2 < n ? in[i + 2] : 0u;
            q[c].w = i + 3 < n ? in[i + 3] : 0u;
        }
    }
#pragma unroll
    for (int c = 0; c < CH; c++) {
        const uint64_t s4 = (uint64_t)q[c].x + q[c].y + q[c].z + q[c].w;
        const uint64_t inc = warp_incl_scan(s4);
        ex[c] = carry + inc - s4;
        carry += __shfl_sync(FULL, inc, 31);
    }
    if (lane == 31) wsum[warp] = carry;
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
    const uint64_t off = s_pre + wpre;
    const bool vout = whole && ((uintptr_t)out & 15) == 0;
#pragma unroll
    for (int c = 0; c < CH; c++) {
        const uint64_t i = wbase + (uint64_t)c * 128 + 4 * lane;
        const uint64_t r0 = off + ex[c], r1 = r0 + q[c].x, r2 = r1 + q[c].y, r3 = r2 + q[c].z;
        if (vout) {
            if constexpr (sizeof(O) == 4) {
                reinterpret_cast<uint4 *>(out + i)[0] = make_uint4((uint32_t)r0, (uint32_t)r1, (uint32_t)r2, (uint32_t)r3);
            } else {
                ulonglong2 *o2 = reinterpret_cast<ulonglong2 *>(out + i);
                o2[0] = make_ulonglong2(r0, r1);
                o2[1] = make_ulonglong2(r2, r3);
            }
        } else {
            if (i < n) out[i] = (O)r0;
            if (i + 1 < n) out[i + 1] = (O)r1;
            if (i + 2 < n) out[i + 2] = (O)r2;
            if (i + 3 < n) out[i + 3] = (O)r3;
        }
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
