// k_open2d.cu -- a5 MORPHOLOGICAL CLEANUP for the in-plane cross (se = 4; reading G-11: o =
// dilate(erode(m)), 4-neighbour cross, out-of-image neighbours ignored) on LINEAR words.
//
// The frame stacks (C3: 128 frames of 9 700 x 13 900, the paper's detector) have rows that are
// not whole words (13 900 = 434 words + 12 bits), so a row-by-row form re-aligns every row.  Here the
// opening works directly on the linear bit array: the x-neighbours of the bits of a word are the same
// array shifted by one bit, the y-neighbours the array shifted by +-X bits (two words and a funnel
// shift), and the row / plane structure enters only through four masks per 32-bit window (bits with
// x = 0, x = X-1, y = 0, y = Y-1), where the out-of-image neighbour is ignored (erosion: taken as 1,
// dilation: as 0).  A CTA owns a tile of R rows (R X a multiple of 32, so tiles own whole words):
//   1. the m words of rows r0-2 .. r0+R+1 into shared memory (coalesced 16-byte loads);
//   2. e = m AND its 4 neighbours (or the mask) for rows r0-1 .. r0+R;
//   3. o = e OR its 4 neighbours (AND NOT the mask) for rows r0 .. r0+R-1, stored (whole words, no
//      atomics, no zeroing);
//   4. per row (a warp per row): the x-run count (the fused first step of a6) and the first rs runs
//      (x0, x1) as run records, by ballots over the row's words (runs are sparse).
#include "async.cuh"
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

struct O2L {
    const uint32_t *m;     // binarised slab, linear bits
    uint64_t m_words;
    uint32_t *o;           // opened mask, linear words
    uint64_t rows, ny, nx, n;
    uint32_t R;            // rows per tile
    uint64_t xmag, ymag;   // ceil(2^64 / X), ceil(2^64 / Y): exact floor divisions of values < 2^40 (X, Y < 2^24)
    uint32_t mw, ew, ow;   // words of the m / e / o tile buffers
    uint32_t *row_runs;
    uint2 *run_slots;
    uint32_t rs;
};

__device__ __forceinline__ uint64_t divmag(uint64_t p, uint64_t mag) { return __umul64hi(p, mag); }

// 32 bits of a shared bit array starting at absolute bit P (word 0 of the array = absolute bit base)
__device__ __forceinline__ uint32_t win(const uint32_t *a, int64_t base, int64_t P) {
    const uint64_t i = (uint64_t)(P - base);
    const uint32_t w = (uint32_t)(i >> 5), sh = (uint32_t)(i & 31);
    return sh ? __funnelshift_r(a[w], a[w + 1], sh) : a[w];
}

// bit j of the window at absolute bit P >= 0: x = 0 (st), x = X-1 (en), y = 0 (top), y = Y-1 (bot)
struct Edge {
    uint32_t st, en, top, bot;
};
__device__ __forceinline__ Edge edges(uint64_t P, const O2L &A) {
    const uint64_t ra = divmag(P, A.xmag);
    const uint32_t q = (uint32_t)(P - ra * A.nx);   // x of bit 0
    const uint32_t jb = (uint32_t)A.nx - q;          // first bit of the next row (1 .. X)
    Edge E;
    E.st = (q == 0 ? 1u : 0u) | (jb < 32 ? 1u << jb : 0u);
    E.en = jb - 1 < 32 ? 1u << (jb - 1) : 0u;
    const uint32_t ma = jb >= 32 ? FULL : (1u << jb) - 1u, mb = ~ma;
    const uint64_t ya = ra - divmag(ra, A.ymag) * A.ny;
    const uint64_t yb = ya + 1 == A.ny ? 0 : ya + 1;
    E.top = (ya == 0 ? ma : 0u) | (yb == 0 ? mb : 0u);
    E.bot = (ya == A.ny - 1 ? ma : 0u) | (yb == A.ny - 1 ? mb : 0u);
    return E;
}

__global__ void __launch_bounds__(256) k_open2d_lin(O2L A, roix_scalars *sc) {
    extern __shared__ uint32_t smem[];
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->run_slots = A.rs;   // read by a6 after this launch
    if (get_err(sc)) return;
    const int64_t X = (int64_t)A.nx;
    const int64_t r0 = (int64_t)blockIdx.x * A.R;
    if (r0 >= (int64_t)A.rows) return;
    const int64_t r1 = min((int64_t)A.rows, r0 + (int64_t)A.R);
    const int64_t B0 = r0 * X, B1 = r1 * X;   // this tile's bits (B0 % 32 == 0)
    uint32_t *M = smem;                       // absolute bits [MB, MB + 32 mw)
    uint32_t *E = M + A.mw + 2;               // [EB, EB + 32 ew)
    uint32_t *O = E + A.ew + 2;               // [B0 - 32, ...): O[0] is a zero guard, O[1 + k] = word B0/32 + k
    const int64_t MB = ((B0 - 2 * X - 32) >> 7) << 7;   // floor to 16 bytes (arithmetic shift: may be negative)
    const int64_t EB = ((B0 - X - 32) >> 5) << 5;
    // 1. m words: the part inside the slab by one bulk copy (TMA engine, mbarrier completion), the rest
    // zero (the masks never let those bits count)
    {
        __shared__ uint64_t bar;
        const int64_t w0 = MB >> 5;                                   // multiple of 4
        const int64_t nw = (int64_t)A.mw + 2;
        const int64_t lo = max(w0, (int64_t)0), hi = min(w0 + nw, (int64_t)((A.m_words + 3) & ~3ull));
        const int64_t c0 = lo, c1 = lo + (((hi - lo) > 0 ? (hi - lo) : 0) & ~3ll);   // whole 16-byte units copied
        for (int64_t k = threadIdx.x; k < nw; k += blockDim.x) {
            const int64_t wi = w0 + k;
            if (wi < c0 || wi >= c1) M[k] = (wi >= 0 && (uint64_t)wi < A.m_words) ? __ldg(A.m + wi) : 0u;
        }
        if (threadIdx.x == 0) {
            mbar_init(&bar, 1);
            asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
            if (c1 > c0) {
                mbar_arrive_expect_tx(&bar, (uint32_t)((c1 - c0) * 4));
                bulk_g2s(M + (c0 - w0), A.m + c0, (uint32_t)((c1 - c0) * 4), &bar);
            } else {
                mbar_arrive(&bar);
            }
        }
        __syncthreads();
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    // 2. erosion
    for (uint32_t k = threadIdx.x; k < A.ew + 2; k += blockDim.x) {
        const int64_t P = EB + 32 * (int64_t)k;
        uint32_t e = 0;
        if (P >= 0 && P < (int64_t)A.n) {
            const Edge g = edges((uint64_t)P, A);
            e = win(M, MB, P) & (win(M, MB, P - 1) | g.st) & (win(M, MB, P + 1) | g.en) &
                (win(M, MB, P - X) | g.top) & (win(M, MB, P + X) | g.bot);
        }
        E[k] = e;
    }
    __syncthreads();
    // 3. dilation -> o (whole words of the tile)
    if (threadIdx.x == 0) O[0] = 0u;
    for (uint32_t k = threadIdx.x; k < A.ow; k += blockDim.x) {
        const int64_t P = B0 + 32 * (int64_t)k;
        uint32_t o = 0;
        if (P < B1) {
            const Edge g = edges((uint64_t)P, A);
            o = win(E, EB, P) | (win(E, EB, P - 1) & ~g.st) | (win(E, EB, P + 1) & ~g.en) |
                (win(E, EB, P - X) & ~g.top) | (win(E, EB, P + X) & ~g.bot);
            if (P + 32 > B1) o &= low_mask((uint32_t)(B1 - P));   // past the slab: pad bits 0
            A.o[(uint64_t)P >> 5] = o;
        }
        O[1 + k] = o;
    }
    if (threadIdx.x < 3) O[1 + A.ow + threadIdx.x] = 0u;
    __syncthreads();
    // 4. runs per row: a warp per row, row-local words cut out of the tile's o
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    const uint32_t W = (uint32_t)((X + 31) / 32);
    const uint32_t tail = (uint32_t)(X - 32 * (int64_t)(W - 1));
    for (int64_t r = r0 + warp; r < r1; r += nwarp) {
        const int64_t rb = r * X;   // absolute bit of the row start
        uint32_t runs = 0, ns = 0, ne = 0;
        uint2 *slot = A.run_slots ? A.run_slots + (uint64_t)r * A.rs : nullptr;
        for (uint32_t k0 = 0; k0 < W; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t w = 0, lw = 0, rw = 0;
            if (k < W) {
                w = win(O, B0 - 32, rb + 32 * (int64_t)k);
                if (k == W - 1 && tail < 32) w &= low_mask(tail);
            }
            // neighbours within the row (the row's bits only): from the adjacent lanes / chunks
            lw = __shfl_up_sync(FULL, w, 1);
            rw = __shfl_down_sync(FULL, w, 1);
            if (lane == 0) lw = k0 ? win(O, B0 - 32, rb + 32 * (int64_t)(k0 - 1)) : 0u;
            if (lane == 31) {
                rw = k + 1 < W ? win(O, B0 - 32, rb + 32 * (int64_t)(k + 1)) : 0u;
                if (k + 1 == W - 1 && tail < 32) rw &= low_mask(tail);
            }
            const uint32_t st = w & ~((w << 1) | (lw >> 31)), en = w & ~((w >> 1) | (rw << 31));
            runs += __reduce_add_sync(FULL, __popc(st));
            if (slot && ns < A.rs) {
                uint32_t bs = __ballot_sync(FULL, st != 0);
                while (bs) {
                    const uint32_t l = __ffs(bs) - 1;
                    bs &= bs - 1;
                    for (uint32_t mm = __shfl_sync(FULL, st, l); mm; mm &= mm - 1) {
                        if (lane == 0 && ns < A.rs) slot[ns].x = 32 * (k0 + l) + __ffs(mm) - 1;
                        ns++;
                    }
                }
            }
            if (slot && ne < A.rs) {
                uint32_t be = __ballot_sync(FULL, en != 0);
                while (be) {
                    const uint32_t l = __ffs(be) - 1;
                    be &= be - 1;
                    for (uint32_t mm = __shfl_sync(FULL, en, l); mm; mm &= mm - 1) {
                        if (lane == 0 && ne < A.rs) slot[ne].y = 32 * (k0 + l) + __ffs(mm);
                        ne++;
                    }
                }
            }
        }
        if (lane == 0 && A.row_runs) A.row_runs[r] = runs;
    }
}

}  // namespace roix

using namespace roix;

static uint64_t ceil_div_2_64(uint64_t d) {   // ceil(2^64 / d) for d >= 2
    const unsigned __int128 one = (unsigned __int128)1 << 64;
    return (uint64_t)((one + d - 1) / d);
}

// returns cudaErrorNotSupported when this form does not apply (the caller keeps the row form)
cudaError_t launch_open2d_lin(const uint32_t *m, uint64_t m_words, const roix_geom &g, uint32_t *o_bits,
                              uint32_t *row_runs, uint2 *run_slots, uint32_t rs, roix_scalars *sc, cudaStream_t st) {
    const uint64_t X = g.nx, Y = g.ny, rows = g.nz * g.ny, n = rows * X;
    if (X < 32 || X >= (1u << 24) || Y < 2 || Y >= (1u << 24) || n >= (1ull << 40)) return cudaErrorNotSupported;
    // rows per tile: R X a multiple of 32 (tiles own whole words), at least 16
    uint64_t R0 = 32;
    for (uint64_t t = X; (t & 1) == 0 && R0 > 1; t >>= 1) R0 >>= 1;
    uint64_t R = R0;
    while (R < 16) R += R0;
    O2L A = {};
    A.m = m;
    A.m_words = m_words;
    A.o = o_bits;
    A.rows = rows;
    A.ny = Y;
    A.nx = X;
    A.n = n;
    A.R = (uint32_t)R;
    A.xmag = ceil_div_2_64(X);
    A.ymag = ceil_div_2_64(Y);
    A.mw = (uint32_t)((((R + 4) * X + 288) / 32 + 2 + 3) & ~3ull);
    A.ew = (uint32_t)(((R + 2) * X + 160) / 32 + 2);
    A.ow = (uint32_t)((R * X + 31) / 32);
    A.row_runs = row_runs;
    A.run_slots = row_runs ? run_slots : nullptr;
    A.rs = A.run_slots ? rs : 0;
    const size_t sm = ((size_t)A.mw + 2 + A.ew + 2 + A.ow + 4) * 4;
    if (sm > 200 * 1024) return cudaErrorNotSupported;
    cudaError_t e = cudaFuncSetAttribute(k_open2d_lin, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    if (e != cudaSuccess) return e;
    const unsigned ctas = (unsigned)((rows + R - 1) / R);
    k_open2d_lin<<<ctas, 256, sm, st>>>(A, sc);
    return cudaGetLastError();
}
