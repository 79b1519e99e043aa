// k_morph2d.cu -- a4 BINARISE (Eq. 2) fused with the in-plane a5 opening (reading G-11:
// o = dilate(erode(m)), 4-neighbour cross, out-of-image neighbours ignored) for frame stacks (C3:
// 128 frames of 9 700 x 13 900, the paper's own detector geometry).
//
// x is read once and m never leaves the SM.  A CTA owns a band of rows (a multiple of 32 rows, so its
// first row starts on a word of the linear bit array for any X) and marches along it S = 8 rows per
// step, with the rings of k_open2d in shared memory: m rows (binarised straight from x by the warp
// that owns the row), e rows, o rows.  Before binarising step c0's rows, every warp asks the TMA
// engine to prefetch into L2 the x row it will binarise in the next step (cp.async.bulk.prefetch), so
// the row loads of a step hit L2 while DRAM streams the next step's rows.
// Output: o as linear words with no atomics and no pre-zeroing -- linear word w belongs to the row
// holding its first bit; a row's last word takes the next row's first bits, so rows are written one
// step row behind the o computation (the o ring keeps S + 1 rows).  Per row it also writes the run
// count (row_runs, the first step of a6) and, when run_slots is given, the first RS runs (x0, x1) of
// the row, so the labelling need not re-read o for rows with at most RS runs.
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

constexpr int M2_S = 8;   // warps per CTA = rows per step

struct M2Args {
    const void *x;
    uint64_t rows, ny, nx;
    uint32_t W, WS;                 // row-local words per row; shared row stride (W + 2 guard words)
    uint64_t rows_per_cta;          // multiple of 32
    const roix_frame *frames;       // per-frame raw thresholds (NEXT-3), or null: sc->thr_*
    uint32_t *o;
    uint32_t *row_runs;             // [rows] or null
    uint2 *run_slots;               // [rows * RS] or null: (x0, x1) of the first RS runs of each row
    uint32_t rs;                    // RS
};

template <typename T>
struct Bin;
template <>
struct Bin<uint16_t> {
    uint32_t thr, low;
    static constexpr int VPL = 8;
    __device__ __forceinline__ uint32_t bits(uint4 v) const {
        uint32_t b = 0;
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
            b |= (uint32_t)((w[k] & 0xffffu) >= thr) << (2 * k);
            b |= (uint32_t)((w[k] >> 16) >= thr) << (2 * k + 1);
        }
        return low ? (~b & 0xffu) : b;
    }
    __device__ __forceinline__ uint32_t bit1(uint16_t v) const { return ((uint32_t)v >= thr) ^ low; }
};
template <>
struct Bin<float> {
    float thr;
    uint32_t low;
    static constexpr int VPL = 4;
    __device__ __forceinline__ uint32_t bits(uint4 v) const {
        uint32_t b = (uint32_t)(__uint_as_float(v.x) >= thr) | ((uint32_t)(__uint_as_float(v.y) >= thr) << 1) |
                     ((uint32_t)(__uint_as_float(v.z) >= thr) << 2) | ((uint32_t)(__uint_as_float(v.w) >= thr) << 3);
        return low ? (~b & 0xfu) : b;
    }
    __device__ __forceinline__ uint32_t bit1(float v) const { return (uint32_t)(v >= thr) ^ low; }
};

__device__ __forceinline__ void l2_prefetch(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// the 16-byte-aligned envelope of row r of x (bytes), for the L2 prefetch
template <typename T>
__device__ __forceinline__ void prefetch_row(const T *x, uint64_t r, uint64_t X) {
    const uintptr_t a = (uintptr_t)(x + r * X) & ~(uintptr_t)15;
    const uintptr_t b = ((uintptr_t)(x + (r + 1) * X) + 15) & ~(uintptr_t)15;
    for (uintptr_t p = a; p < b; p += 0xfff0u) {   // bulk sizes are 32-bit, keep each under 64 KB
        const uint32_t len = (uint32_t)min((uintptr_t)0xfff0u, b - p);
        l2_prefetch((const void *)p, len);
    }
}

// Warp: binarise row r of x into dst[0..W) (row-local words, pad bits beyond X = 1: erosion border).
// Lane l takes the 16-byte blocks l, l+32, ... of the row's aligned envelope, U of them in flight.
template <typename T>
__device__ __forceinline__ void bin_row(const T *__restrict__ xrow, uint64_t X, uint32_t W, const Bin<T> &cmp,
                                        uint32_t *dst) {
    constexpr int VPL = Bin<T>::VPL, LPW = 32 / VPL, U = 8;
    const uint32_t lane = lane_id();
    const uint32_t off = (uint32_t)(((uintptr_t)xrow & 15u) / sizeof(T));   // voxels before xrow in its block
    const uint4 *ab = reinterpret_cast<const uint4 *>(xrow - off);
    const uint64_t span = off + X;
    const uint32_t nblk = (uint32_t)((span + VPL - 1) / VPL);
    const uint32_t nA = (uint32_t)((span + 31) / 32);   // aligned-relative words
    // aligned-relative word a holds row bits [32 a - off, 32 a - off + 32); row word k = bits of
    // aligned words k and k+1 shifted by off -- assembled through the row's own destination: the
    // aligned words are written first to dst[-1 ..] when off > 0 (dst[-1] is the guard word)
    uint32_t *adst = off ? dst - 1 : dst;
    for (uint32_t c0 = 0; c0 < nblk; c0 += 32 * U) {
        // all U loads are issued before any is used (U 16-byte loads in flight per lane)
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t blk = c0 + 32 * u + lane;
            const uint64_t p0 = (uint64_t)blk * VPL;
            v[u] = (blk < nblk && p0 >= off && p0 + VPL <= span) ? __ldcs(ab + blk) : make_uint4(0, 0, 0, 0);
        }
        uint32_t b[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t blk = c0 + 32 * u + lane;
            const uint64_t p0 = (uint64_t)blk * VPL;
            b[u] = 0;
            if (blk < nblk) {
                if (p0 >= off && p0 + VPL <= span) {
                    b[u] = cmp.bits(v[u]);
                } else {   // a row end's partial block: the row's own voxels only, pad bits 1
                    const T *e = reinterpret_cast<const T *>(ab + blk);
                    for (int k = 0; k < VPL; k++) {
                        const uint64_t p = p0 + k;
                        b[u] |= (p >= off && p < span ? cmp.bit1(e[k]) : 1u) << k;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            uint32_t w = 0;
#pragma unroll
            for (int i = 0; i < LPW; i++) w |= __shfl_sync(FULL, b[u], (lane * LPW + i) & 31) << (i * VPL);
            const uint32_t a = (c0 + 32 * u) / LPW + lane;
            if (lane < (uint32_t)VPL && a < nA) adst[a] = w;   // 32 blocks = VPL words
        }
    }
    __syncwarp();
    if (off) {
        // row word k = aligned words A[k], A[k+1] (now at dst[k-1], dst[k]) shifted right by off, in
        // place: every lane reads its two words before any lane writes; A[k0+32], overwritten by the
        // previous 32 words' last lane, is carried in a register
        uint32_t carry = 0;
        for (uint32_t k0 = 0; k0 < W; k0 += 32) {
            const uint32_t k = k0 + lane;
            uint32_t lo = 0, hi = FULL;
            if (k < W) {
                lo = (lane == 0 && k0 > 0) ? carry : dst[(int)k - 1];
                hi = k + 1 < nA ? dst[k] : FULL;
            }
            carry = __shfl_sync(FULL, hi, 31);
            __syncwarp();
            if (k < W) dst[k] = __funnelshift_r(lo, hi, off);
            __syncwarp();
        }
        if (lane == 0) dst[-1] = FULL;   // restore the guard
    }
    __syncwarp();
    const uint32_t tail = (uint32_t)(X - 32ull * (W - 1));
    if (lane == 0 && tail < 32) dst[W - 1] |= ~low_mask(tail);
    __syncwarp();
}

template <typename T>
__global__ void __launch_bounds__(256, 2) k_morph2d(M2Args A, roix_scalars *sc) {
    extern __shared__ uint32_t smem[];
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->run_slots = A.rs;   // read by a6 after this launch
    if (get_err(sc)) return;
    constexpr int S = M2_S;
    constexpr uint32_t MS = S + 4, ES = S + 2, OS = S + 1;
    const uint32_t W = A.W, WS = A.WS;
    const int warp = threadIdx.x >> 5;
    const uint32_t lane = lane_id();
    uint32_t *mring = smem;             // [MS][WS]
    uint32_t *ering = mring + MS * WS;  // [ES][WS]
    uint32_t *oring = ering + ES * WS;  // [OS][WS]
    const T *x = static_cast<const T *>(A.x);
    const int64_t Y = A.ny, X = A.nx, rows = A.rows;
    const int64_t r0 = (int64_t)blockIdx.x * A.rows_per_cta;
    const int64_t r1 = min(rows, r0 + (int64_t)A.rows_per_cta);
    if (r0 >= r1) return;
    Bin<T> cmp;
    if constexpr (sizeof(T) == 2) cmp.thr = sc->thr_u16;
    else cmp.thr = sc->thr_f32;
    cmp.low = sc->polarity;
    for (int i = threadIdx.x; i < (int)MS; i += blockDim.x) {
        mring[i * WS] = FULL;
        mring[i * WS + W + 1] = FULL;
    }
    for (int i = threadIdx.x; i < (int)(ES + OS); i += blockDim.x) {   // e and o rows: zero guard words
        ering[i * WS] = 0;
        ering[i * WS + W + 1] = 0;
    }
    __syncthreads();
    auto mrow = [&](int64_t r) { return mring + ((uint32_t)(r - r0 + 2) % MS) * WS + 1; };
    auto erow = [&](int64_t r) { return ering + ((uint32_t)(r - r0 + 2) % ES) * WS + 1; };
    auto orow = [&](int64_t r) { return oring + ((uint32_t)(r - r0 + 1) % OS) * WS + 1; };
    auto load_m = [&](int64_t r) {
        uint32_t *dst = mrow(r);
        if (r < 0 || r >= rows) {
            for (uint32_t k = lane; k < W; k += 32) dst[k] = FULL;
            __syncwarp();
            return;
        }
        Bin<T> c = cmp;
        if (A.frames) c.thr = A.frames[(uint64_t)r / (uint64_t)Y].thr_u16;
        bin_row<T>(x + (uint64_t)r * X, X, W, c, dst);
    };
    const uint32_t tail = (uint32_t)(X - 32ll * (W - 1));
    auto comp_e = [&](int64_t r) {
        uint32_t *dst = erow(r);
        if (r < 0 || r >= rows) {
            for (uint32_t k = lane; k < W; k += 32) dst[k] = 0;
            __syncwarp();
            return;
        }
        const int64_t y = r % Y;
        const uint32_t *c = mrow(r);
        const uint32_t *a = y > 0 ? mrow(r - 1) : c, *b = y < Y - 1 ? mrow(r + 1) : c;   // out of plane: ignored
        for (uint32_t k = lane; k < W; k += 32) {
            const uint32_t w = c[k];
            uint32_t v = w & __funnelshift_l(c[k - 1], w, 1) & __funnelshift_r(w, c[k + 1], 1) & a[k] & b[k];
            if (k == W - 1 && tail < 32) v &= low_mask(tail);
            dst[k] = v;
        }
    };
    // o row r -> linear words it owns (those whose first bit is in the row); the last one takes its
    // high bits from row r + 1 (next: its first word, 0 past the volume)
    auto write_row = [&](int64_t r) {
        const uint32_t *R = orow(r);
        const uint32_t nxt = r + 1 < rows ? orow(r + 1)[0] : 0u;
        const uint64_t Bg = (uint64_t)r * X, Be = Bg + X;
        const uint64_t wa = (Bg + 31) >> 5, wb = (Be + 31) >> 5;   // owned linear words [wa, wb)
        for (uint64_t w = wa + lane; w < wb; w += 32) {
            const uint32_t t = (uint32_t)(32 * w - Bg);             // row-local bit of the word's first bit
            const uint32_t k = t >> 5, s = t & 31;
            uint32_t v = s ? __funnelshift_r(R[k], k + 1 < W ? R[k + 1] : 0u, s) : R[k];
            if (t + 32 > X) v |= nxt << (uint32_t)(X - t);          // X - t in 1..31 here
            A.o[w] = v;
        }
    };
    // prologue: m rows r0-2 .. r0+1, e rows r0-1, r0; prefetch the first step's rows
    if (lane == 0) {
        const int64_t rp = r0 + 2 + warp;
        if (rp < rows) prefetch_row(x, (uint64_t)rp, (uint64_t)X);
    }
    for (int i = warp; i < 4; i += S) load_m(r0 - 2 + i);
    __syncthreads();
    for (int i = warp; i < 2; i += S) comp_e(r0 - 1 + i);
    __syncthreads();
    for (int64_t c0 = r0; c0 < r1; c0 += S) {
        // the rows of the next step go to L2 while this step's rows are binarised
        if (lane == 0) {
            const int64_t rp = c0 + S + 2 + warp;
            if (rp < rows && rp < r1 + 2) prefetch_row(x, (uint64_t)rp, (uint64_t)X);
        }
        load_m(c0 + 2 + warp);
        __syncthreads();
        comp_e(c0 + 1 + warp);
        __syncthreads();
        // o rows c0 .. c0+S-1 (into the o ring), run counts and run slots
        const int64_t r = c0 + warp;
        if (r < r1) {
            const int64_t y = r % Y;
            const uint32_t *c = erow(r);
            const uint32_t *a = y > 0 ? erow(r - 1) : nullptr, *b = y < Y - 1 ? erow(r + 1) : nullptr;
            uint32_t *od = orow(r);
            for (uint32_t k = lane; k < W; k += 32) {
                const uint32_t cw = c[k];
                uint32_t w = cw | __funnelshift_l(c[k - 1], cw, 1) | __funnelshift_r(cw, c[k + 1], 1);
                if (a) w |= a[k];
                if (b) w |= b[k];
                if (k == W - 1 && tail < 32) w &= low_mask(tail);
                od[k] = w;
            }
            __syncwarp();
            // x-runs of the row: starts (set, left clear) and ends (set, right clear; exclusive end =
            // position + 1); the i-th start pairs with the i-th end
            uint32_t runs = 0, nends = 0;   // starts / ends met so far in the row
            for (uint32_t k0 = 0; k0 < W; k0 += 32) {
                const uint32_t k = k0 + lane;
                const uint32_t w = k < W ? od[k] : 0u;
                const uint32_t lw = k < W ? od[(int)k - 1] : 0u, rw = k + 1 < W ? od[k + 1] : 0u;
                const uint32_t starts = w & ~((w << 1) | (lw >> 31));
                const uint32_t ends = w & ~((w >> 1) | (rw << 31));
                const uint32_t ns = __popc(starts), ne = __popc(ends);
                if (A.run_slots && nends < A.rs) {
                    uint32_t is = runs + warp_incl_scan(ns) - ns, ie = nends + warp_incl_scan(ne) - ne;
                    uint2 *slot = A.run_slots + (uint64_t)r * A.rs;
                    for (uint32_t sb = starts; sb && is < A.rs; sb &= sb - 1, is++) slot[is].x = 32 * k + __ffs(sb) - 1;
                    for (uint32_t eb = ends; eb && ie < A.rs; eb &= eb - 1, ie++) slot[ie].y = 32 * k + __ffs(eb);
                }
                runs += __reduce_add_sync(FULL, ns);
                nends += __reduce_add_sync(FULL, ne);
            }
            if (A.row_runs && lane == 0) A.row_runs[r] = runs;
        }
        __syncthreads();
        // linear words of rows c0-1 .. c0+S-2 (each needs the first word of the row after it)
        {
            const int64_t rw = c0 - 1 + warp;
            if (rw >= r0 && rw < r1) write_row(rw);
        }
        // (no barrier needed: the o ring slot of row rw is rewritten S + 1 rows later)
    }
    __syncthreads();
    // the band's last row, when the loop's last step ended on it (the loop writes rows up to c0 + S - 2)
    if (warp == 0 && (r1 - r0) % S == 0) write_row(r1 - 1);
}

}  // namespace roix

using namespace roix;

// a4 + a5 for the in-plane SE (se = 4): one pass over x (see the top of this file)
cudaError_t launch_morph2d(const void *x, int dtype, const roix_geom &g, roix_scalars *sc, uint32_t *o_bits,
                           uint32_t *row_runs, uint2 *run_slots, uint32_t rs, const roix_frame *frames,
                           cudaStream_t st) {
    M2Args A = {};
    A.x = x;
    A.rows = g.nz * g.ny;
    A.ny = g.ny;
    A.nx = g.nx;
    A.W = (uint32_t)((g.nx + 31) / 32);
    A.WS = A.W + 2;
    A.frames = frames;
    A.o = o_bits;
    A.row_runs = row_runs;
    A.run_slots = run_slots;
    A.rs = run_slots ? rs : 0;
    const size_t sm = (size_t)((M2_S + 4) + (M2_S + 2) + (M2_S + 1)) * A.WS * 4;
    if (sm > 220 * 1024) return cudaErrorInvalidConfiguration;
    cudaError_t e;
    int occ = 0;
    if (dtype == ROIX_U16) {
        if ((e = cudaFuncSetAttribute(k_morph2d<uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) !=
                cudaSuccess ||
            (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_morph2d<uint16_t>, 32 * M2_S, sm)) != cudaSuccess)
            return e;
    } else {
        if ((e = cudaFuncSetAttribute(k_morph2d<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)) !=
                cudaSuccess ||
            (e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_morph2d<float>, 32 * M2_S, sm)) != cudaSuccess)
            return e;
    }
    if (occ < 1) occ = 1;
    // one wave of equal bands; each band a multiple of 32 rows (its first row starts on a word)
    const uint64_t slots = (uint64_t)num_sms() * occ;
    uint64_t rpc = (A.rows + slots - 1) / slots;
    rpc = (rpc + 31) / 32 * 32;
    A.rows_per_cta = rpc;
    const unsigned ctas = (unsigned)((A.rows + rpc - 1) / rpc);
    if (dtype == ROIX_U16) k_morph2d<uint16_t><<<ctas, 32 * M2_S, sm, st>>>(A, sc);
    else k_morph2d<float><<<ctas, 32 * M2_S, sm, st>>>(A, sc);
    return cudaGetLastError();
}
