// k_greedy.cu -- NEXT-2: the paper's greedy absolute-error-bounded quantiser (§4.2.3 Steps
// 1-5) on a uint16 sequence D[0..n): groups are the greedy left-to-right maximal runs whose
// intervals [D - E, D + E] intersect, i.e. whose range max - min stays <= 2E; every element of a
// group gets Q = floor((u + l) / 2) = floor((max + min) / 2) of the group, clipped to [0, qmax].
//
// The scan is sequential by definition; its parallel form here rests on forced boundaries: where
// |D[i] - D[i-1]| > 2E no group can hold both i-1 and i, so a group starts at i whatever came before.
// The stretches between forced boundaries are independent greedy problems:
//   k_greedy   thread t owns 32 elements: their forced boundaries, and every stretch starting among
//              them, scanned with Steps 3-4 to the next forced boundary (possibly far beyond the
//              window), writing Q and the group-start bits; the group count is summed per warp
// On noisy data (CT, small E) stretches are a few elements long; a smooth stretch is scanned by one
// thread (the exact, sequential worst case).
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

// One thread per 32-element window.  The window's elements are staged in shared memory (row stride
// 17 words: conflict-free for the threads' data-dependent indices) with 16-byte loads; its forced
// boundaries come from neighbouring elements; every stretch starting in the window is scanned (Steps
// 3-4) from shared memory while it stays in the window and from global memory beyond.  Q of the
// window's own elements is staged and stored with 16-byte stores when the window begins with a forced
// boundary (otherwise its prefix belongs to an earlier thread's stretch and the codes go one by one).
// Group-start bits of the window are OR-ed in once; bits beyond it (long stretches) atomically.
constexpr int GQ_T = 256, GQ_RS = 17;   // threads, shared row stride in 32-bit words (34 halfwords)

__global__ void __launch_bounds__(GQ_T) k_greedy(const uint16_t *__restrict__ D, uint64_t n, uint32_t T, uint32_t qmax,
                                                 uint16_t *__restrict__ Q, uint32_t *__restrict__ G,
                                                 unsigned long long *ngroups) {
    __shared__ uint32_t s_d[GQ_T * GQ_RS];
    __shared__ uint32_t s_q[GQ_T * GQ_RS];
    const uint64_t nw = (n + 31) / 32;
    uint16_t *sd = reinterpret_cast<uint16_t *>(s_d) + threadIdx.x * (2 * GQ_RS);
    uint16_t *sq = reinterpret_cast<uint16_t *>(s_q) + threadIdx.x * (2 * GQ_RS);
    uint64_t count = 0;
    for (uint64_t w0 = (uint64_t)blockIdx.x * GQ_T; w0 < nw; w0 += (uint64_t)gridDim.x * GQ_T) {
        const uint64_t w = w0 + threadIdx.x;
        if (w < nw) {
            const uint64_t i0 = w * 32;
            const uint32_t m = (uint32_t)min((uint64_t)32, n - i0);   // elements in this window
            if (m == 32) {
                const uint4 *src = reinterpret_cast<const uint4 *>(D + i0);
                uint32_t *row = reinterpret_cast<uint32_t *>(sd);
#pragma unroll
                for (int k = 0; k < 4; k++) {
                    const uint4 v = __ldcs(src + k);
                    row[4 * k] = v.x;
                    row[4 * k + 1] = v.y;
                    row[4 * k + 2] = v.z;
                    row[4 * k + 3] = v.w;
                }
            } else {
                for (uint32_t j = 0; j < m; j++) sd[j] = D[i0 + j];
            }
            // forced boundaries of the window: |D[i] - D[i-1]| > 2E (T = floor(2E)), and i = 0
            uint32_t prev = i0 ? D[i0 - 1] : 0u, F = 0;
            for (uint32_t j = 0; j < m; j++) {
                const uint32_t v = sd[j];
                if ((i0 == 0 && j == 0) || (v > prev ? v - prev : prev - v) > T) F |= 1u << j;
                prev = v;
            }
            uint32_t own = 0, starts = F;
            while (starts) {
                const uint32_t b = __ffs(starts) - 1;
                starts &= starts - 1;
                uint64_t i = i0 + b, g0 = i;
                uint32_t mn = sd[b], mx = mn, pv = mn;
                own |= 1u << b;
                count++;
                for (++i; i < n; ++i) {
                    const uint32_t v = i - i0 < 32 ? (uint32_t)sd[i - i0] : (uint32_t)D[i];
                    if ((v > pv ? v - pv : pv - v) > T) break;   // next forced boundary: the stretch ends
                    pv = v;
                    const uint32_t nmn = min(mn, v), nmx = max(mx, v);
                    if (nmx - nmn > T) {   // empty intersection: close [g0, i), open a group at i
                        const uint16_t q = (uint16_t)min((mn + mx) >> 1, qmax);
                        for (uint64_t j = g0; j < i; j++) {
                            if (j - i0 < 32) sq[j - i0] = q;
                            else Q[j] = q;
                        }
                        g0 = i;
                        mn = mx = v;
                        count++;
                        if (i - i0 < 32) own |= 1u << (i - i0);
                        else atomicOr(&G[i >> 5], 1u << (i & 31));
                    } else {
                        mn = nmn;
                        mx = nmx;
                    }
                }
                const uint16_t q = (uint16_t)min((mn + mx) >> 1, qmax);
                for (uint64_t j = g0; j < i; j++) {
                    if (j - i0 < 32) sq[j - i0] = q;
                    else Q[j] = q;
                }
            }
            // this window's codes: positions from its first forced boundary on
            if (F & 1u && m == 32) {
                const uint32_t *row = reinterpret_cast<const uint32_t *>(sq);
                uint4 *dst = reinterpret_cast<uint4 *>(Q + i0);
#pragma unroll
                for (int k = 0; k < 4; k++)
                    __stcs(dst + k, make_uint4(row[4 * k], row[4 * k + 1], row[4 * k + 2], row[4 * k + 3]));
            } else if (F) {
                for (uint32_t j = __ffs(F) - 1; j < m; j++) Q[i0 + j] = sq[j];
            }
            if (own) atomicOr(&G[w], own);
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) count += __shfl_xor_sync(FULL, count, d);
    if (lane_id() == 0 && count) atomicAdd(ngroups, (unsigned long long)count);
}

}  // namespace roix

using namespace roix;

size_t greedy_workspace_bytes(uint64_t n) { return 256; }

cudaError_t launch_greedy(const uint16_t *D, uint64_t n, double E, uint32_t qmax, uint16_t *Q, uint32_t *group_bits,
                          uint64_t *ngroups, void *ws, cudaStream_t st) {
    (void)ws;
    const uint64_t nw = (n + 31) / 32;
    cudaError_t e = cudaMemsetAsync(group_bits, 0, nw * 4, st);
    if (e != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(ngroups, 0, 8, st)) != cudaSuccess) return e;
    if (n == 0) return cudaSuccess;
    // |a - b| > 2E  <=>  |a - b| > floor(2E) for integers
    const double t = floor(2.0 * E);
    const uint32_t T = t >= 65536.0 ? 65536u : (uint32_t)t;
    const unsigned grid = (unsigned)min((nw + GQ_T - 1) / GQ_T, (uint64_t)num_sms() * 8);
    k_greedy<<<grid, GQ_T, 0, st>>>(D, n, T, qmax, Q, group_bits, (unsigned long long *)ngroups);
    return cudaGetLastError();
}
