// k_morph.cu -- a4 BINARISE (Eq. 2) and a5 MORPHOLOGICAL CLEANUP (reading G-11: one
// opening o = dilate(erode(m)), radius-1 cross, out-of-volume neighbours ignored).
//
//  k_binarize: a pure stream over x (16-byte loads, one mask word per lane, coalesced 128-byte
//    stores) writing the packed mask m.
//  k_open3d (se = 6): a CTA owns a band of TY rows of every plane of a z-chunk and marches along z
//    with rings of 3 m-planes and 3 e-planes in shared memory; m is re-read only for 2 halo rows per
//    band side and 2 halo planes per chunk side (bits: 1/16 of the input bytes for u16).
//  k_open2d (se = 4, in-plane): a CTA owns a range of rows and marches along them.
// Shared-memory rows: W = ceil(X/32) words plus a guard word on each side (stride WS = W + 2); m rows
// carry guard/pad bits = 1 (erosion border 1), e/o rows 0 (dilation border 0).  Erosion and
// dilation are word-wise AND / OR of the row, its +-1 x-shifts (funnel shifts across the
// neighbouring words) and the neighbouring rows / planes.  Both open kernels count the x-runs of
// every output row (the fused first step of a6 CCL).
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

struct MorphArgs {
    uint64_t nz, ny, nx, z0, gz;
    const uint32_t *m;       // binarised slab, linear bits
    uint64_t m_words;
    uint32_t W, WS;          // words per row, row stride in shared memory
    int TY;                  // 3-D: rows per band
    uint64_t zchunk;         // 3-D: planes per CTA
    uint64_t rows_per_cta;   // 2-D: rows per CTA
    int aligned_out;         // 1: plain stores of whole words; 0: atomicOr into zeroed o
    int async;               // 3-D: rows are whole 16-byte units (X % 128 == 0): cp.async prefetch
    const uint32_t *halo_lo, *halo_hi;
    uint32_t *o;
    uint32_t *row_runs;
};

template <typename T>
struct Cmp;
template <>
struct Cmp<uint16_t> {
    uint32_t thr;
    uint32_t low;
    __device__ Cmp(const roix_scalars *sc) : thr(sc->thr_u16), low(sc->polarity) {}
    static constexpr int VPL = 8;  // voxels per 16-byte load
    __device__ __forceinline__ uint32_t bits(uint4 v) const {
        uint32_t w[4] = {v.x, v.y, v.z, v.w}, b = 0;
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
struct Cmp<float> {
    float thr;
    uint32_t low;
    __device__ Cmp(const roix_scalars *sc) : thr(sc->thr_f32), low(sc->polarity) {}
    static constexpr int VPL = 4;
    __device__ __forceinline__ uint32_t bits(uint4 v) const {
        uint32_t b = (uint32_t)(__uint_as_float(v.x) >= thr) | ((uint32_t)(__uint_as_float(v.y) >= thr) << 1) |
                     ((uint32_t)(__uint_as_float(v.z) >= thr) << 2) | ((uint32_t)(__uint_as_float(v.w) >= thr) << 3);
        return low ? (~b & 0xfu) : b;
    }
    __device__ __forceinline__ uint32_t bit1(float v) const { return (uint32_t)(v >= thr) ^ low; }
};

// Warp-level: binarise one row of X voxels starting at xrow into dst[0..W) (row-local words),
// pad bits beyond X = 1.  stage: W + 2 words of per-warp scratch (used when xrow is not 16-B aligned).
template <typename T>
__device__ void binarize_row(const T *__restrict__ xrow, uint64_t X, uint32_t W, const Cmp<T> &cmp, uint32_t *dst,
                             uint32_t *stage) {
    constexpr int VPL = Cmp<T>::VPL;
    const uint32_t lane = lane_id();
    const uint32_t off = (uint32_t)(((uintptr_t)xrow & 15u) / sizeof(T));  // voxels before xrow in its 16-B block
    const uint4 *ab = reinterpret_cast<const uint4 *>(xrow - off);
    const uint64_t span = off + X;                  // aligned-relative voxel positions [0, span)
    const uint64_t nblk = (span + VPL - 1) / VPL;   // 16-B blocks touched
    uint32_t *out = off ? stage : dst;              // aligned-relative words
    const uint32_t nA = (uint32_t)((span + 31) / 32);
    for (uint64_t c0 = 0; c0 * 32 < nblk; c0 += 4) {
        uint32_t b[4];
#pragma unroll
        for (int u = 0; u < 4; u++) {
            uint64_t blk = (c0 + u) * 32 + lane;
            b[u] = 0;
            if (blk < nblk) {
                uint64_t p0 = blk * VPL;
                if (p0 >= off && p0 + VPL <= span) {
                    b[u] = cmp.bits(__ldcs(ab + blk));
                } else {  // partial block at a row end: scalar loads of the valid voxels only
                    const T *e = reinterpret_cast<const T *>(ab + blk);
                    for (int k = 0; k < VPL; k++) {
                        uint64_t p = p0 + k;
                        uint32_t bit = 1;  // pad (p >= span) and head (p < off, shifted out) bits
                        if (p >= off && p < span) bit = cmp.bit1(e[k]);
                        b[u] |= bit << k;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
            // word j of this chunk = lanes [j*32/VPL, (j+1)*32/VPL)
            uint32_t w = 0;
            constexpr int LPW = 32 / VPL;  // lanes per word
#pragma unroll
            for (int i = 0; i < LPW; i++) {
                uint32_t v = __shfl_sync(FULL, b[u], (lane * LPW + i) & 31);
                w |= v << (i * VPL);
            }
            uint64_t widx = (c0 + u) * VPL + lane;
            if (lane < (uint32_t)VPL && widx < nA) out[widx] = w;
        }
    }
    if (off) {
        __syncwarp();
        for (uint32_t k = lane; k < W; k += 32) {
            uint32_t lo = stage[k], hi = (k + 1 < nA) ? stage[k + 1] : FULL;
            dst[k] = __funnelshift_r(lo, hi, off);
        }
    }
    __syncwarp();
    // pad bits beyond X are 1 (erosion border)
    uint32_t tail = (uint32_t)(X - 32ull * (W - 1));
    if (lane == 0 && tail < 32) dst[W - 1] |= ~low_mask(tail);
    __syncwarp();
}

__device__ __forceinline__ void fill_row(uint32_t *dst, uint32_t W, uint32_t v) {
    for (uint32_t k = lane_id(); k < W; k += 32) dst[k] = v;
    __syncwarp();
}

// erosion of word k of row `c` (guards at [-1] and [W]); up/down/front/back rows
__device__ __forceinline__ uint32_t erode_word(const uint32_t *c, const uint32_t *a, const uint32_t *b,
                                               const uint32_t *f, const uint32_t *g, int k) {
    uint32_t w = c[k];
    uint32_t l = __funnelshift_l(c[k - 1], w, 1);  // bit x <- bit x-1
    uint32_t r = __funnelshift_r(w, c[k + 1], 1);  // bit x <- bit x+1
    uint32_t v = w & l & r & a[k] & b[k];
    if (f) v &= f[k] & g[k];
    return v;
}
__device__ __forceinline__ uint32_t dilate_word(const uint32_t *c, const uint32_t *a, const uint32_t *b,
                                                const uint32_t *f, const uint32_t *g, int k) {
    uint32_t w = c[k];
    uint32_t l = __funnelshift_l(c[k - 1], w, 1);
    uint32_t r = __funnelshift_r(w, c[k + 1], 1);
    uint32_t v = w | l | r | a[k] | b[k];
    if (f) v |= f[k] | g[k];
    return v;
}

// Warp-level: count x-runs of a row given its words (pad bits 0); lanes cover words k = lane + 32 i.
__device__ __forceinline__ uint32_t count_runs_words(uint32_t w, uint32_t &carry) {
    uint32_t prev = __shfl_up_sync(FULL, w, 1);
    if (lane_id() == 0) prev = carry;
    carry = __shfl_sync(FULL, w, 31);
    uint32_t starts = w & ~((w << 1) | (prev >> 31));
    return __popc(starts);
}

__device__ __forceinline__ void write_row_atomic(uint32_t *o, uint64_t bitpos, uint32_t k, uint32_t w) {
    uint64_t b = bitpos + 32ull * k;
    uint32_t sh = (uint32_t)(b & 31);
    if (!w) return;
    atomicOr(&o[b >> 5], w << sh);
    if (sh) atomicOr(&o[(b >> 5) + 1], w >> (32 - sh));
}


// ------------------------------------------------------------------------------------ binarise
// One warp iteration = 32 mask words = 1024 voxels; lane l loads the 16-byte groups c*32 + l
// (c < CH), packs their VPL-bit masks into P = sum_c b_c << (c VPL), then lane j gathers word j from
// the GPW lanes that hold its groups.
template <typename T>
__global__ void __launch_bounds__(256) k_binarize(const T *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                  uint32_t *__restrict__ m) {
    if (get_err(sc)) return;
    constexpr int VPL = Cmp<T>::VPL, CH = 32 / VPL, GPW = 32 / VPL;
    const Cmp<T> cmp(sc);
    const uint32_t lane = lane_id();
    const uint64_t iters = (n + 1023) / 1024;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const uint64_t nwords = (n + 31) / 32;
    for (uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); it < iters; it += wstride) {
        const uint64_t g0 = it * 32 * CH;  // first 16-byte group of the iteration
        uint32_t P = 0;
        if ((it + 1) * 1024 <= n) {
            uint4 v[CH];
#pragma unroll
            for (int c = 0; c < CH; c++) v[c] = __ldcs(x4 + g0 + c * 32 + lane);
#pragma unroll
            for (int c = 0; c < CH; c++) P |= cmp.bits(v[c]) << (c * VPL);
        } else {
            for (int c = 0; c < CH; c++) {
                const uint64_t v0 = (g0 + c * 32 + lane) * VPL;
                uint32_t b = 0;
                if (v0 + VPL <= n) b = cmp.bits(__ldcs(x4 + g0 + c * 32 + lane));
                else
                    for (int k = 0; k < VPL; k++)
                        if (v0 + k < n) b |= cmp.bit1(x[v0 + k]) << k;
                P |= b << (c * VPL);
            }
        }
        // word j = chunk c = j / VPL, groups (j % VPL) * GPW + i of that chunk
        const uint32_t c = lane / VPL, src0 = (lane % VPL) * GPW;
        uint32_t w = 0;
#pragma unroll
        for (int i = 0; i < GPW; i++) {
            uint32_t q = __shfl_sync(FULL, P, src0 + i);
            w |= ((q >> (c * VPL)) & ((1u << VPL) - 1u)) << (i * VPL);
        }
        const uint64_t wi = it * 32 + lane;
        if (wi < nwords) m[wi] = w;
    }
}

// Warp-level: row words of a linear bit array starting at bit `bit0` (X bits), pad bits = 1 (m rows).
__device__ __forceinline__ void load_m_row(const uint32_t *__restrict__ src, uint64_t src_words, uint64_t bit0,
                                           uint64_t X, uint32_t W, uint32_t *dst) {
    const uint32_t sh = (uint32_t)(bit0 & 31);
    const uint64_t w0 = bit0 >> 5;
    const uint32_t tail = (uint32_t)(X - 32ull * (W - 1));
    for (uint32_t k = lane_id(); k < W; k += 32) {
        const uint64_t wi = w0 + k;
        uint32_t v = src[wi];
        if (sh) v = __funnelshift_r(v, (wi + 1 < src_words) ? src[wi + 1] : 0u, sh);
        if (k == W - 1 && tail < 32) v |= ~low_mask(tail);
        dst[k] = v;
    }
}

// ------------------------------------------------------------------------------------ 3-D opening
__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
    unsigned s = (unsigned)__cvta_generic_to_shared(dst);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(src));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

constexpr int MSLOTS = 8, PF = 4;  // m ring slots; planes prefetched ahead (PF + 3 <= MSLOTS)

// Rings: m has MSLOTS plane slots (m(p+1..p+PF) are in flight with cp.async while e(p-1) and o(p-2)
// are computed), e has 3.  Row data starts 4 words into its slot (16-byte aligned for cp.async), with the
// guard words at data[-1] and data[W].  A.async: rows are whole 16-byte units in global memory
// (X % 128 == 0); otherwise rows are loaded synchronously with funnel shifts.
__global__ void __launch_bounds__(256) k_open3d(MorphArgs A, roix_scalars *sc) {
    extern __shared__ __align__(16) uint32_t smem[];
    if (get_err(sc)) return;
    const int TY = A.TY;
    const uint32_t W = A.W, WS = A.WS;             // WS: multiple of 4, >= W + 8
    const int MR = TY + 4, ER = TY + 2;            // m rows y0-2.., e rows y0-1..
    uint32_t *mring = smem;                          // [MSLOTS][MR][WS]
    uint32_t *ering = mring + MSLOTS * MR * WS;      // [3][ER][WS]
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const int64_t y0 = (int64_t)blockIdx.x * TY;
    const int64_t zs = (int64_t)blockIdx.y * A.zchunk;
    const int64_t ze = min((int64_t)A.nz, zs + (int64_t)A.zchunk);
    const int64_t Y = A.ny, X = A.nx;
    if (zs >= ze) return;
    for (int i = threadIdx.x; i < MSLOTS * MR; i += blockDim.x) {
        mring[i * WS + 3] = FULL;
        mring[i * WS + 4 + W] = FULL;
    }
    for (int i = threadIdx.x; i < 3 * ER; i += blockDim.x) {
        ering[i * WS + 3] = 0;
        ering[i * WS + 4 + W] = 0;
    }
    __syncthreads();
    auto mrow = [&](int64_t p, int r) { return mring + (((p + MSLOTS) & (MSLOTS - 1)) * MR + r) * WS + 4; };
    auto erow = [&](int64_t p, int r) { return ering + ((p + 3) % 3 * ER + r) * WS + 4; };
    const uint64_t plane_w = (A.ny * A.nx + 31) / 32;
    const uint32_t tail = (uint32_t)(X - 32ll * (W - 1));
    const bool async = A.async;
    // enqueue the rows of m(p) (cp.async, or synchronous loads in the generic path)
    auto fetch = [&](int64_t p) {
        const int64_t gp = (int64_t)A.z0 + p;
        for (int r = warp; r < MR; r += nw) {
            const int64_t y = y0 - 2 + r;
            uint32_t *dst = mrow(p, r);
            const uint32_t *src;
            uint64_t bit0, swords;
            if (y < 0 || y >= Y || gp < 0 || gp >= (int64_t)A.gz) {
                fill_row(dst, W, FULL);
                continue;
            } else if (p < 0) {
                src = A.halo_lo;
                swords = 2 * plane_w;
                bit0 = (uint64_t)(p + 2) * plane_w * 32 + y * A.nx;
            } else if (p >= (int64_t)A.nz) {
                src = A.halo_hi;
                swords = 2 * plane_w;
                bit0 = (uint64_t)(p - A.nz) * plane_w * 32 + y * A.nx;
            } else {
                src = A.m;
                swords = A.m_words;
                bit0 = ((uint64_t)p * A.ny + y) * A.nx;
            }
            if (async) {
                const uint4 *s4 = reinterpret_cast<const uint4 *>(src + (bit0 >> 5));
                for (uint32_t k = lane_id(); k < W / 4; k += 32) cp_async16(dst + 4 * k, s4 + k);
            } else {
                load_m_row(src, swords, bit0, A.nx, W, dst);
            }
        }
        cp_async_commit();
    };
    for (int k = 0; k < PF; k++) {
        if (zs - 2 + k <= ze + 1) fetch(zs - 2 + k);
        else cp_async_commit();
    }
    for (int64_t p = zs - 2; p <= ze + 1; p++) {
        if (p + PF <= ze + 1) fetch(p + PF);
        else cp_async_commit();     // empty group: keeps the group count uniform
        cp_async_wait<PF>();        // m(p) has landed; m(p+1..p+PF) may still be in flight
        __syncthreads();
        // e(q = p-1), rows y0-1 .. y0+TY
        const int64_t q = p - 1;
        if (q >= zs - 1) {
            const int64_t gq = (int64_t)A.z0 + q;
            const bool qin = gq >= 0 && gq < (int64_t)A.gz;
            for (int r = warp; r < ER; r += nw) {
                const int64_t y = y0 - 1 + r;
                uint32_t *dst = erow(q, r);
                if (!qin || y < 0 || y >= Y) {
                    fill_row(dst, W, 0u);
                    continue;
                }
                const uint32_t *c = mrow(q, r + 1), *a = mrow(q, r), *b = mrow(q, r + 2);
                const uint32_t *f = mrow(q - 1, r + 1), *g = mrow(q + 1, r + 1);
                for (uint32_t k = lane_id(); k < W; k += 32) {
                    uint32_t v = erode_word(c, a, b, f, g, k);
                    if (k == W - 1 && tail < 32) v &= low_mask(tail);
                    dst[k] = v;
                }
            }
        }
        __syncthreads();
        // o(z = p-2), rows y0 .. y0+TY-1
        const int64_t z = p - 2;
        if (z >= zs && z < ze) {
            for (int r = warp; r < TY; r += nw) {
                const int64_t y = y0 + r;
                if (y >= Y) break;
                const uint32_t *c = erow(z, r + 1), *a = erow(z, r), *b = erow(z, r + 2);
                const uint32_t *f = erow(z - 1, r + 1), *g = erow(z + 1, r + 1);
                const uint64_t row = (uint64_t)z * A.ny + y;
                const uint64_t bitpos = row * A.nx;
                uint32_t carry = 0, runs = 0;
                for (uint32_t k0 = 0; k0 < W; k0 += 32) {
                    uint32_t k = k0 + lane_id();
                    uint32_t w = 0;
                    if (k < W) {
                        w = dilate_word(c, a, b, f, g, k);
                        if (k == W - 1 && tail < 32) w &= low_mask(tail);
                    }
                    runs += count_runs_words(w, carry);
                    if (k < W) {
                        if (A.aligned_out) A.o[(bitpos >> 5) + k] = w;
                        else write_row_atomic(A.o, bitpos, k, w);
                    }
                }
                if (A.row_runs) {
#pragma unroll
                    for (int d = 16; d > 0; d >>= 1) runs += __shfl_xor_sync(FULL, runs, d);
                    if (lane_id() == 0) A.row_runs[row] = runs;
                }
            }
        }
        // the next iteration's fetch writes m(p+1+PF) into the slot of m(p+1+PF-MSLOTS), last read
        // by e(p+2+PF-MSLOTS) <= e(p-1), which every warp finished before the barrier above
    }
}

// ------------------------------------------------------------------------------------ 2-D opening
// Rows r = q*Y + y of the slab (q = plane); neighbours only within the same plane.  S = rows per
// step = warps per CTA.  The output rows of a step are contiguous bits [c X, (c+S) X) of o; they are
// assembled from the o rows in shared memory into whole words.
__global__ void __launch_bounds__(256) k_open2d(MorphArgs A, roix_scalars *sc) {
    extern __shared__ uint32_t smem[];
    if (get_err(sc)) return;
    const uint32_t W = A.W, WS = A.WS;
    const int S = blockDim.x >> 5, warp = threadIdx.x >> 5;
    const int MS = S + 4, ES = S + 2;
    uint32_t *mring = smem;            // [MS][WS]
    uint32_t *ering = mring + MS * WS; // [ES][WS]
    uint32_t *orow = ering + ES * WS;  // [S][WS]
    const int64_t Y = A.ny, X = A.nx;
    const int64_t rows = (int64_t)(A.nz * A.ny);
    const int64_t r0 = (int64_t)blockIdx.x * A.rows_per_cta;
    const int64_t r1 = min(rows, r0 + (int64_t)A.rows_per_cta);
    if (r0 >= r1) return;
    for (int i = threadIdx.x; i < MS; i += blockDim.x) {
        mring[i * WS] = FULL;
        mring[i * WS + W + 1] = FULL;
    }
    for (int i = threadIdx.x; i < ES + S; i += blockDim.x) {
        ering[i * WS] = 0;
        ering[i * WS + W + 1] = 0;
    }
    __syncthreads();
    auto mrow = [&](int64_t r) { return mring + ((r % MS + MS) % MS) * WS + 1; };
    auto erow = [&](int64_t r) { return ering + ((r % ES + ES) % ES) * WS + 1; };
    auto load_m = [&](int64_t r) {
        uint32_t *dst = mrow(r);
        if (r < 0 || r >= rows) fill_row(dst, W, FULL);
        else load_m_row(A.m, A.m_words, (uint64_t)r * A.nx, A.nx, W, dst);
    };
    const uint32_t tail = (uint32_t)(X - 32ll * (W - 1));
    auto comp_e = [&](int64_t r) {
        uint32_t *dst = erow(r);
        if (r < 0 || r >= rows) {
            fill_row(dst, W, 0u);
            return;
        }
        const int64_t y = r % Y;
        const uint32_t *c = mrow(r);
        // out-of-plane neighbours are ignored (border 1): use the row itself
        const uint32_t *a = y > 0 ? mrow(r - 1) : c, *b = y < Y - 1 ? mrow(r + 1) : c;
        for (uint32_t k = lane_id(); k < W; k += 32) {
            uint32_t v = erode_word(c, a, b, nullptr, nullptr, k);
            if (k == W - 1 && tail < 32) v &= low_mask(tail);
            dst[k] = v;
        }
    };
    // prologue: m rows r0-2 .. r0+1, e rows r0-1, r0
    for (int i = warp; i < 4; i += S) load_m(r0 - 2 + i);
    __syncthreads();
    for (int i = warp; i < 2; i += S) comp_e(r0 - 1 + i);
    __syncthreads();
    for (int64_t c0 = r0; c0 < r1; c0 += S) {
        load_m(c0 + 2 + warp);
        __syncthreads();
        comp_e(c0 + 1 + warp);
        __syncthreads();
        // o rows c0 .. c0+S-1 into orow, with run counts
        const int64_t r = c0 + warp;
        uint32_t *od = orow + warp * WS + 1;
        if (r < r1) {
            const int64_t y = r % Y;
            const uint32_t *c = erow(r);
            const uint32_t *a = y > 0 ? erow(r - 1) : nullptr, *b = y < Y - 1 ? erow(r + 1) : nullptr;
            uint32_t carry = 0, runs = 0;
            for (uint32_t k0 = 0; k0 < W; k0 += 32) {
                uint32_t k = k0 + lane_id();
                uint32_t w = 0;
                if (k < W) {
                    uint32_t cw = c[k];
                    w = cw | __funnelshift_l(c[k - 1], cw, 1) | __funnelshift_r(cw, c[k + 1], 1);
                    if (a) w |= a[k];
                    if (b) w |= b[k];
                    if (k == W - 1 && tail < 32) w &= low_mask(tail);
                    od[k] = w;
                }
                runs += count_runs_words(w, carry);
            }
            if (A.row_runs) {
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) runs += __shfl_xor_sync(FULL, runs, d);
                if (lane_id() == 0) A.row_runs[r] = runs;
            }
        }
        __syncthreads();
        // assemble bits [c0 X, cend X) into global words
        const int64_t cend = min(r1, c0 + (int64_t)S);
        const uint64_t B0 = (uint64_t)c0 * A.nx, B1 = (uint64_t)cend * A.nx;
        const uint64_t w0 = B0 >> 5, w1 = (B1 + 31) >> 5;
        for (uint64_t wi = w0 + threadIdx.x; wi < w1; wi += blockDim.x) {
            uint64_t lo = max(wi * 32, B0), hi = min(wi * 32 + 32, B1);
            uint32_t val = 0;
            uint64_t pos = lo;
            while (pos < hi) {
                uint64_t rel = pos - B0;
                uint64_t rr = rel / A.nx, col = rel - rr * A.nx;
                uint32_t take = (uint32_t)min((uint64_t)(hi - pos), A.nx - col);
                const uint32_t *src = orow + rr * WS + 1;
                uint32_t cw = (uint32_t)(col >> 5), cs = (uint32_t)(col & 31);
                uint32_t bits = __funnelshift_r(src[cw], src[cw + 1], cs) & low_mask(take);
                val |= bits << (uint32_t)(pos - wi * 32);
                pos += take;
            }
            // a word is owned by this CTA alone when it starts here and either ends here or holds
            // the end of the volume (its remaining bits are pad bits, which must be 0)
            bool whole = lo == wi * 32 && (hi == wi * 32 + 32 || hi == (uint64_t)rows * A.nx);
            if (whole && A.aligned_out) A.o[wi] = val;
            else if (val) atomicOr(&A.o[wi], val);
        }
        __syncthreads();
    }
}

// ------------------------------------------------------------------ halo planes: m packed per plane
template <typename T>
__global__ void __launch_bounds__(256) k_binarize_planes(const T *__restrict__ x, MorphArgs A, uint64_t p0,
                                                         uint64_t np, roix_scalars *sc, uint32_t *out) {
    extern __shared__ uint32_t smem[];
    if (get_err(sc)) return;
    const Cmp<T> cmp(sc);
    const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    uint32_t *row = smem + warp * 2 * A.WS;
    uint32_t *stage = row + A.WS;
    const uint64_t plane_w = (A.ny * A.nx + 31) / 32;
    const uint64_t total = np * A.ny;
    for (uint64_t rr = (uint64_t)blockIdx.x * nw + warp; rr < total; rr += (uint64_t)gridDim.x * nw) {
        uint64_t pl = rr / A.ny, y = rr % A.ny;
        binarize_row(x + ((p0 + pl) * A.ny + y) * A.nx, A.nx, A.W, cmp, row, stage);
        uint32_t tail = (uint32_t)(A.nx - 32ull * (A.W - 1));
        for (uint32_t k = lane_id(); k < A.W; k += 32) {
            uint32_t w = row[k];
            if (k == A.W - 1 && tail < 32) w &= low_mask(tail);
            write_row_atomic(out + pl * plane_w, y * A.nx, k, w);
        }
        __syncwarp();
    }
}

}  // namespace roix

using namespace roix;

template <typename K>
static cudaError_t set_smem(K kern, size_t bytes) {
    return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
}

size_t morph_workspace_bytes(const roix_geom &g) { return ((g.nz * g.ny * g.nx + 31) / 32 + 64) * 4; }

cudaError_t launch_morph(const void *x, int dtype, const roix_geom &g, uint32_t se, const uint32_t *halo_lo,
                         const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs, void *ws,
                         cudaStream_t st) {
    MorphArgs A = {};
    A.nz = g.nz;
    A.ny = g.ny;
    A.nx = g.nx;
    A.z0 = g.z0;
    A.gz = g.gz;
    A.W = (uint32_t)((g.nx + 31) / 32);
    A.WS = A.W + 2;
    A.halo_lo = halo_lo;
    A.halo_hi = halo_hi;
    A.o = o_bits;
    A.row_runs = row_runs;
    const uint64_t n = g.nz * g.ny * g.nx;
    const uint64_t nwords = (n + 31) / 32;
    uint32_t *m = (uint32_t *)ws;
    A.m = m;
    A.m_words = nwords;
    cudaError_t e;
    // a4: stream x -> m
    {
        uint64_t iters = (n + 1023) / 1024;
        uint64_t blocks = (iters + 7) / 8;
        uint64_t cap = (uint64_t)num_sms() * 8;
        if (blocks > cap) blocks = cap;
        if (dtype == ROIX_U16) k_binarize<uint16_t><<<(unsigned)blocks, 256, 0, st>>>((const uint16_t *)x, n, sc, m);
        else k_binarize<float><<<(unsigned)blocks, 256, 0, st>>>((const float *)x, n, sc, m);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    int occ = 0;
    if (se == 6) {
        // band height: the largest of 64/32/16/8 rows whose rings fit ~100 KB (2+ CTAs per SM) and
        // that still gives >= 1.5 CTAs per SM with z-chunks of >= 64 planes
        const uint64_t chunks_max = g.nz >= 128 ? g.nz / 64 : 1;
        A.WS = (A.W + 8 + 3) / 4 * 4;
        A.async = (g.nx % 128 == 0);
        int TY = 64;
        auto smem_of = [&](int ty) { return (size_t)(MSLOTS * (ty + 4) + 3 * (ty + 2)) * A.WS * 4; };
        while (TY > 4 && smem_of(TY) > 72 * 1024) TY /= 2;
        while (TY > 8 && ((g.ny + TY - 1) / TY) * chunks_max < (uint64_t)(1.5 * num_sms())) TY /= 2;
        if ((uint64_t)TY > g.ny) TY = (int)g.ny;
        A.TY = TY;
        size_t sm = smem_of(TY);
        if (sm > 220 * 1024) return cudaErrorInvalidConfiguration;
        if ((e = set_smem(k_open3d, sm)) != cudaSuccess) return e;
        cudaFuncSetAttribute(k_open3d, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_open3d, 256, sm)) != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        uint64_t bands = (g.ny + TY - 1) / TY;
        uint64_t slots = (uint64_t)num_sms() * occ;
        uint64_t chunks = (slots + bands - 1) / bands;
        if (chunks < 1) chunks = 1;
        if (chunks > chunks_max) chunks = chunks_max;
        A.zchunk = (g.nz + chunks - 1) / chunks;
        chunks = (g.nz + A.zchunk - 1) / A.zchunk;
        A.aligned_out = (g.nx % 32 == 0);
        if (!A.aligned_out && (e = cudaMemsetAsync(o_bits, 0, nwords * 4, st)) != cudaSuccess) return e;
        dim3 grid((unsigned)bands, (unsigned)chunks);
        k_open3d<<<grid, 256, sm, st>>>(A, sc);
    } else {
        const int S = 8;
        size_t sm = (size_t)((S + 4) + (S + 2) + S) * A.WS * 4;
        if (sm > 220 * 1024) return cudaErrorInvalidConfiguration;
        if ((e = set_smem(k_open2d, sm)) != cudaSuccess) return e;
        if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_open2d, 32 * S, sm)) != cudaSuccess) return e;
        if (occ < 1) occ = 1;
        const uint64_t rows = g.nz * g.ny;
        uint64_t slots = (uint64_t)num_sms() * occ;
        // rows per CTA: a multiple of 32, so every CTA's bit range starts on a word boundary
        uint64_t rpc = (rows + slots - 1) / slots;
        rpc = (rpc + 31) / 32 * 32;
        A.rows_per_cta = rpc;
        uint64_t ctas = (rows + rpc - 1) / rpc;
        // whole words at every step iff S*X is a multiple of 32 (CTA starts are, see above)
        A.aligned_out = ((uint64_t)S * g.nx) % 32 == 0;
        if (!A.aligned_out && (e = cudaMemsetAsync(o_bits, 0, nwords * 4, st)) != cudaSuccess) return e;
        k_open2d<<<(unsigned)ctas, 32 * S, sm, st>>>(A, sc);
    }
    return cudaGetLastError();
}

cudaError_t launch_binarize_planes(const void *x, int dtype, const roix_geom &g, uint64_t p0, uint64_t np,
                                   roix_scalars *sc, uint32_t *m_bits, cudaStream_t st) {
    MorphArgs A = {};
    A.nz = g.nz;
    A.ny = g.ny;
    A.nx = g.nx;
    A.W = (uint32_t)((g.nx + 31) / 32);
    A.WS = A.W + 2;
    const uint64_t plane_w = (g.ny * g.nx + 31) / 32;
    cudaError_t e = cudaMemsetAsync(m_bits, 0, np * plane_w * 4, st);
    if (e != cudaSuccess) return e;
    size_t sm = (size_t)8 * 2 * A.WS * 4;
    uint64_t rows = np * g.ny;
    unsigned blocks = (unsigned)((rows + 7) / 8 < 1024 ? (rows + 7) / 8 : 1024);
    if (blocks == 0) return cudaSuccess;
    if (dtype == ROIX_U16) {
        if ((e = set_smem(k_binarize_planes<uint16_t>, sm)) != cudaSuccess) return e;
        k_binarize_planes<uint16_t><<<blocks, 256, sm, st>>>((const uint16_t *)x, A, p0, np, sc, m_bits);
    } else {
        if ((e = set_smem(k_binarize_planes<float>, sm)) != cudaSuccess) return e;
        k_binarize_planes<float><<<blocks, 256, sm, st>>>((const float *)x, A, p0, np, sc, m_bits);
    }
    return cudaGetLastError();
}
