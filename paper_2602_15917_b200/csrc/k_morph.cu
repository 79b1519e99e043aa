// k_morph.cu -- a4 BINARISE (Eq. 2) and a5 MORPHOLOGICAL CLEANUP (reading G-11: one
// opening o = dilate(erode(m)), radius-1 cross, out-of-volume neighbours ignored).
//
//  k_binarize: a pure stream over x (16-byte loads, one mask word per lane, coalesced 128-byte
//    stores) writing the packed mask m.
//  k_open3d (se = 6): a CTA owns a band of TY rows of every plane of a z-chunk and marches along z
//    with rings of 3 m-planes and 3 e-planes in shared memory; m is re-read only for 2 halo rows per
//    band side and 2 halo planes per chunk side (bits: 1/16 of the input bytes for u16).
//  k_open2d_w (se = 4, in-plane, 32 <= X < 16 K): a warp owns a range of rows, each row whole in
//    registers; the slab is cut into chunks of planes, binarised on the caller's stream and opened on
//    a second stream, so the (issue-bound) opening of one chunk overlaps the (HBM-bound) binarisation
//    of the next.
//  k_open2d (se = 4, other widths): a CTA owns a range of rows and marches along them.
// Shared-memory rows: W = ceil(X/32) words plus a guard word on each side (stride WS = W + 2); m rows
// carry guard/pad bits = 1 (erosion border 1), e/o rows 0 (dilation border 0).  Erosion and
// dilation are word-wise AND / OR of the row, its +-1 x-shifts (funnel shifts across the
// neighbouring words) and the neighbouring rows / planes.  Both open kernels count the x-runs of
// every output row (the fused first step of a6 CCL).
#include <cstdlib>
#include <mutex>

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
    const uint32_t *halo_lo, *halo_hi;
    uint32_t *o;
    uint32_t *row_runs;
    uint2 *run_slots;        // [rows * rs] or null: (x0, x1) of the first rs x-runs of every output row
    uint32_t rs;
    int64_t row_lo, row_hi;  // 2-D register-row opening: the rows (whole planes) this launch reads and writes
    int64_t z_lo, z_hi;      // 3-D whole-row opening: the planes this launch writes
};

template <typename T>
struct Cmp;
template <>
struct Cmp<uint16_t> {
    uint32_t thr;
    uint32_t low;
    uint32_t t2, keep;   // SWAR compare: (thr mod 2^15) in both halves; mask selecting | (thr < 2^15) or &
    __device__ Cmp(const roix_scalars *sc) : low(sc->polarity) { set_thr(sc->thr_u16); }
    __device__ __forceinline__ void set_thr(uint32_t t) {
        thr = t;
        t2 = (t & 0x7fffu) * 0x00010001u;
        keep = t < 0x8000u ? FULL : 0u;
    }
    static constexpr int VPL = 8;  // voxels per 16-byte load
    // x >= thr for both 16-bit halves of w, exact for every uint16 x and thr <= 0xffff: with x = 2^15 xh
    // + xl, s = (x | 2^15) - tl has bit 15 = [xl >= tl] (no borrow leaves the half), and
    // x >= thr = xh | [xl >= tl] when th = 0, xh & [xl >= tl] when th = 1.  Flags at bits 15 and 31.
    __device__ __forceinline__ uint32_t ge2(uint32_t w) const {
        const uint32_t sv = (w | 0x80008000u) - t2;
        return ((w & sv) | ((w | sv) & keep)) & 0x80008000u;
    }
    __device__ __forceinline__ uint32_t bits(uint4 v) const {
        if (thr > 0xffffu) return low ? 0xffu : 0u;
        // byte 1 / byte 3 of each flag word hold the voxels' flags at their top bit; one multiply moves
        // four byte-top bits to bits 28..31 (partial products land on distinct bits: no carries)
        const uint32_t r01 = __byte_perm(ge2(v.x), ge2(v.y), 0x7531), r23 = __byte_perm(ge2(v.z), ge2(v.w), 0x7531);
        const uint32_t b = ((r01 * 0x00204081u) >> 28) | (((r23 * 0x00204081u) >> 28) << 4);
        return low ? (~b & 0xffu) : b;
    }
    __device__ __forceinline__ uint32_t bit1(uint16_t v) const { return ((uint32_t)v >= thr) ^ low; }
};
template <>
struct Cmp<float> {
    float thr;
    uint32_t low;
    __device__ Cmp(const roix_scalars *sc) : thr(sc->thr_f32), low(sc->polarity) {}
    __device__ __forceinline__ void set_thr(float t) { thr = t; }
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
// NEXT-3 per-frame thresholds (uint16 frame stacks): voxel v of plane p = v / A compares against
// frames[p].thr_u16.  A warp iteration covers 1024 voxels, so for A >= 1024 it meets at most one plane
// boundary b1: a 16-byte group uses the threshold of its plane, a group straddling b1 goes voxel by
// voxel; A < 1024 (tiny frames) divides per voxel.
struct FrameThr {
    const roix_frame *f;
    uint64_t A;
};

__device__ __forceinline__ uint32_t u16_of(uint4 v, int k) {
    const uint32_t w = k < 2 ? v.x : k < 4 ? v.y : k < 6 ? v.z : v.w;
    return (k & 1) ? w >> 16 : w & 0xffffu;
}

template <typename T, bool FR>
__device__ __forceinline__ uint32_t group_bits(const Cmp<T> &cmp, uint4 vec, uint64_t v0, const FrameThr &F,
                                               uint64_t p0, uint64_t b1, uint32_t t0, uint32_t t1) {
    if constexpr (!FR) {
        return cmp.bits(vec);
    } else {
        constexpr int VPL = Cmp<T>::VPL;
        Cmp<T> c = cmp;
        if (F.A >= 1024) {
            if (v0 + VPL <= b1 || v0 >= b1) {
                c.set_thr(v0 < b1 ? t0 : t1);
                return c.bits(vec);
            }
            uint32_t b = 0;
            for (int k = 0; k < VPL; k++) b |= ((u16_of(vec, k) >= (v0 + k < b1 ? t0 : t1)) ^ c.low) << k;
            return b;
        }
        uint32_t b = 0;
        for (int k = 0; k < VPL; k++) b |= ((u16_of(vec, k) >= F.f[(v0 + k) / F.A].thr_u16) ^ c.low) << k;
        return b;
    }
}

template <typename T, bool FR>
__device__ __forceinline__ uint32_t voxel_bit(const Cmp<T> &cmp, T val, uint64_t v, const FrameThr &F) {
    if constexpr (!FR) {
        return cmp.bit1(val);
    } else {
        return ((uint32_t)val >= F.f[v / F.A].thr_u16) ^ cmp.low;
    }
}

// One warp iteration = 32 mask words = 1024 voxels; lane l loads the 16-byte groups c*32 + l
// (c < CH), packs their VPL-bit masks into P = sum_c b_c << (c VPL), then lane j gathers word j from
// the GPW lanes that hold its groups.
template <typename T, bool FR = false>
__global__ void __launch_bounds__(256) k_binarize(const T *__restrict__ x, uint64_t n, roix_scalars *sc,
                                                  uint32_t *__restrict__ m, int skip_if_resolved, FrameThr F) {
    if (get_err(sc)) return;
    if (skip_if_resolved && sc->spec_state == 2) return;   // the fused pass already produced m
    constexpr int VPL = Cmp<T>::VPL, CH = 32 / VPL, GPW = 32 / VPL;
    const Cmp<T> cmp(sc);
    const uint32_t lane = lane_id();
    const uint64_t iters = (n + 1023) / 1024;
    const uint64_t wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const uint64_t nwords = (n + 31) / 32;
    // the next iteration's loads are issued before this one is binarised (two iterations in flight)
    uint64_t it = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint4 nxt[CH];
    auto prefetch = [&](uint64_t j) {
        if (j < iters && (j + 1) * 1024 <= n) {
#pragma unroll
            for (int c = 0; c < CH; c++) nxt[c] = __ldcs(x4 + j * 32 * CH + c * 32 + lane);
        }
    };
    prefetch(it);
    for (; it < iters; it += wstride) {
        const uint64_t g0 = it * 32 * CH;  // first 16-byte group of the iteration
        uint4 v[CH];
#pragma unroll
        for (int c = 0; c < CH; c++) v[c] = nxt[c];
        prefetch(it + wstride);
        uint64_t p0 = 0, b1 = ~0ull;
        uint32_t t0 = 0, t1 = 0;
        if constexpr (FR) {
            if (F.A >= 1024) {
                p0 = it * 1024 / F.A;
                b1 = (p0 + 1) * F.A;
                t0 = F.f[p0].thr_u16;
                t1 = b1 < n ? F.f[p0 + 1].thr_u16 : t0;
            }
        }
        uint32_t P = 0;
        if ((it + 1) * 1024 <= n) {
#pragma unroll
            for (int c = 0; c < CH; c++)
                P |= group_bits<T, FR>(cmp, v[c], (g0 + c * 32 + lane) * VPL, F, p0, b1, t0, t1) << (c * VPL);
        } else {
            for (int c = 0; c < CH; c++) {
                const uint64_t v0 = (g0 + c * 32 + lane) * VPL;
                uint32_t b = 0;
                if (v0 + VPL <= n) b = group_bits<T, FR>(cmp, __ldcs(x4 + g0 + c * 32 + lane), v0, F, p0, b1, t0, t1);
                else
                    for (int k = 0; k < VPL; k++)
                        if (v0 + k < n) b |= voxel_bit<T, FR>(cmp, x[v0 + k], v0 + k, F) << k;
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
// Four lane-iterations' loads are issued before any is used (a long row otherwise waits on one
// global-load latency per 32 words).
__device__ __forceinline__ void load_m_row(const uint32_t *__restrict__ src, uint64_t src_words, uint64_t bit0,
                                           uint64_t X, uint32_t W, uint32_t *dst) {
    constexpr int U = 4;
    const uint32_t sh = (uint32_t)(bit0 & 31);
    const uint64_t w0 = bit0 >> 5;
    const uint32_t tail = (uint32_t)(X - 32ull * (W - 1));
    const uint32_t *row = src + w0;
    // words of the row readable past its first one (32-bit from here on)
    const uint32_t avail = (uint32_t)min(src_words - w0, (uint64_t)W + 1);
    for (uint32_t k0 = lane_id(); k0 < W; k0 += 32 * U) {
        uint32_t v[U], nx[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t k = k0 + 32 * u;
            v[u] = k < W ? row[k] : 0u;
            nx[u] = (k < W && sh && k + 1 < avail) ? row[k + 1] : 0u;
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint32_t k = k0 + 32 * u;
            if (k >= W) break;
            uint32_t val = sh ? __funnelshift_r(v[u], nx[u], sh) : v[u];
            if (k == W - 1 && tail < 32) val |= ~low_mask(tail);
            dst[k] = val;
        }
    }
}

// ------------------------------------------------------- 3-D opening, whole-row warps (X % 32 == 0)
// A warp owns S = 32 / L row segments; segment s holds RY consecutive rows of one plane and its lane
// sl the KW consecutive words [KW sl, KW sl + KW) of each row (W = L KW words per row: every row is
// complete inside its segment, so no x-halo).  The warp marches along z over its z-chunk keeping in
// registers m of planes p-1, p, p+1 (rows yb-2 .. yb+RY+1) and e of planes p-2, p-1, p (rows yb-1 ..
// yb+RY).  The three slots of each ring rotate by renaming (the z-loop is unrolled by 3), so there
// are no register moves.  x-neighbour words come from the adjacent lanes (one shfl each way per
// row), y-neighbours from the adjacent register rows, z-neighbours from the other slots.  Each
// segment also writes the x-run count of every output row (the first step of a6 CCL) with a plain
// store: a row belongs to exactly one warp.
template <int KW>
struct WordsT;
template <>
struct WordsT<1> {
    static __device__ __forceinline__ void ld(const uint32_t *p, uint32_t (&w)[1]) { w[0] = __ldg(p); }
    static __device__ __forceinline__ void st(uint32_t *p, const uint32_t (&w)[1]) { *p = w[0]; }
};
template <>
struct WordsT<2> {
    static __device__ __forceinline__ void ld(const uint32_t *p, uint32_t (&w)[2]) {
        const uint2 v = __ldg(reinterpret_cast<const uint2 *>(p));
        w[0] = v.x;
        w[1] = v.y;
    }
    static __device__ __forceinline__ void st(uint32_t *p, const uint32_t (&w)[2]) {
        *reinterpret_cast<uint2 *>(p) = make_uint2(w[0], w[1]);
    }
};
template <>
struct WordsT<4> {
    static __device__ __forceinline__ void ld(const uint32_t *p, uint32_t (&w)[4]) {
        const uint4 v = __ldg(reinterpret_cast<const uint4 *>(p));
        w[0] = v.x;
        w[1] = v.y;
        w[2] = v.z;
        w[3] = v.w;
    }
    static __device__ __forceinline__ void st(uint32_t *p, const uint32_t (&w)[4]) {
        *reinterpret_cast<uint4 *>(p) = make_uint4(w[0], w[1], w[2], w[3]);
    }
};

// bit x <- bit x-1 (l) and bit x <- bit x+1 (r) of the lane's KW words; `pad` enters at the row ends
template <int L, int KW>
__device__ __forceinline__ void xnbr(const uint32_t (&c)[KW], uint32_t sl, uint32_t pad, uint32_t (&l)[KW],
                                     uint32_t (&r)[KW]) {
    uint32_t left = __shfl_up_sync(FULL, c[KW - 1], 1, L);
    uint32_t right = __shfl_down_sync(FULL, c[0], 1, L);
    if (sl == 0) left = pad;
    if (sl == L - 1) right = pad;
#pragma unroll
    for (int i = 0; i < KW; i++) {
        l[i] = __funnelshift_l(i ? c[i - 1] : left, c[i], 1);
        r[i] = __funnelshift_r(c[i], i < KW - 1 ? c[i + 1] : right, 1);
    }
}

template <int L>
__device__ __forceinline__ uint32_t seg_sum(uint32_t v) {
    if constexpr (L == 32) {
        return __reduce_add_sync(FULL, v);
    } else {
#pragma unroll
        for (int d = L / 2; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
        return v;
    }
}

template <int L, int KW, int RY>
__global__ void __launch_bounds__(256, (KW == 1 ? 3 : (KW == 2 ? 2 : 1))) k_open3d_rows(MorphArgs A, roix_scalars *sc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->run_slots = 0;   // no run records from this form
    if (get_err(sc)) return;
    constexpr int S = 32 / L, MR = RY + 4, ER = RY + 2;
    using WT = WordsT<KW>;
    const uint32_t lane = lane_id(), sl = lane & (L - 1), seg = lane / L;
    const int Y = (int)A.ny;
    const uint32_t W = L * KW;
    const uint32_t tiles_y = (uint32_t)((A.ny + S * RY - 1) / (S * RY));
    const uint32_t task = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t cz = task / tiles_y;
    const int yb = (int)((task - cz * tiles_y) * (S * RY) + seg * RY);   // this segment's first row
    const int nz = (int)A.nz;
    const int zs = (int)A.z_lo + (int)(cz * A.zchunk);   // planes [z_lo, z_hi) of this launch
    if (zs >= (int)A.z_hi) return;
    const int ze = min((int)A.z_hi, zs + (int)A.zchunk);
    const uint64_t plane_w = A.ny * (uint64_t)W;
    const int64_t gz = (int64_t)A.gz, z0 = (int64_t)A.z0;
    const int roff = (yb - 2) * (int)W + (int)(KW * sl);   // word offset of slot row 0 in its plane
    uint32_t vm = 0;   // bit j: m row yb-2+j is inside the plane
#pragma unroll
    for (int j = 0; j < MR; j++)
        if (yb - 2 + j >= 0 && yb - 2 + j < Y) vm |= 1u << j;
    const uint32_t ve = vm >> 1;   // bit i: e row yb-1+i is inside the plane

    uint32_t m[3][MR][KW], e[3][ER][KW];
    auto load = [&](int p, uint32_t (&dst)[MR][KW]) {
        const int64_t gp = z0 + p;
        const uint32_t *pb = nullptr;
        if (gp >= 0 && gp < gz) {
            if (p < 0) pb = A.halo_lo + (uint64_t)(p + 2) * plane_w;
            else if (p >= nz) pb = A.halo_hi + (uint64_t)(p - nz) * plane_w;
            else pb = A.m + (uint64_t)p * plane_w;
        }
#pragma unroll
        for (int j = 0; j < MR; j++) {
            if (pb && ((vm >> j) & 1)) {
                WT::ld(pb + roff + j * (int)W, dst[j]);
            } else {
#pragma unroll
                for (int i = 0; i < KW; i++) dst[j][i] = FULL;
            }
        }
    };
    // e(p) into E from m(p-1) = MP, m(p) = MC, m(p+1) = MN
    auto erode = [&](int p, const uint32_t (&MP)[MR][KW], const uint32_t (&MC)[MR][KW],
                     const uint32_t (&MN)[MR][KW], uint32_t (&E)[ER][KW]) {
        const int64_t gp = z0 + p;
        const bool pin = gp >= 0 && gp < gz;
#pragma unroll
        for (int r = 0; r < ER; r++) {
            uint32_t l[KW], rr[KW];
            xnbr<L, KW>(MC[r + 1], sl, FULL, l, rr);
            const bool live = pin && ((ve >> r) & 1);
#pragma unroll
            for (int i = 0; i < KW; i++) {
                const uint32_t v = MC[r + 1][i] & l[i] & rr[i] & MC[r][i] & MC[r + 2][i] & MP[r + 1][i] & MN[r + 1][i];
                E[r][i] = live ? v : 0u;
            }
        }
    };
    // o(q) from e(q-1) = EP, e(q) = EC, e(q+1) = EN; stores o and the run counts of its rows
    auto dilate = [&](int q, const uint32_t (&EP)[ER][KW], const uint32_t (&EC)[ER][KW],
                      const uint32_t (&EN)[ER][KW]) {
        uint32_t *ob = A.o + (uint64_t)q * plane_w + roff + 2 * W;
        const uint64_t rbase = (uint64_t)q * A.ny + yb;
#pragma unroll
        for (int j = 0; j < RY; j++) {
            uint32_t l[KW], rr[KW], o[KW];
            xnbr<L, KW>(EC[j + 1], sl, 0u, l, rr);
#pragma unroll
            for (int i = 0; i < KW; i++)
                o[i] = EC[j + 1][i] | l[i] | rr[i] | EC[j][i] | EC[j + 2][i] | EP[j + 1][i] | EN[j + 1][i];
            // run starts: set bits whose left neighbour is clear
            uint32_t left = __shfl_up_sync(FULL, o[KW - 1], 1, L);
            if (sl == 0) left = 0u;
            uint32_t cnt = 0;
#pragma unroll
            for (int i = 0; i < KW; i++) cnt += __popc(o[i] & ~__funnelshift_l(i ? o[i - 1] : left, o[i], 1));
            cnt = seg_sum<L>(cnt);
            if (yb + j < Y) {
                WT::st(ob + j * (int)W, o);
                if (sl == 0 && A.row_runs) A.row_runs[rbase + j] = cnt;
            }
        }
    };
#pragma unroll
    for (int s = 0; s < 3; s++)
#pragma unroll
        for (int r = 0; r < ER; r++)
#pragma unroll
            for (int i = 0; i < KW; i++) e[s][r][i] = 0u;
    load(zs - 2, m[0]);
    load(zs - 1, m[1]);
    load(zs, m[2]);
    // step p: e(p) from m(p-1..p+1); m(p+2) into the freed slot; o(p-1) from e(p-2..p)
#define ROIX_OPEN_STEP(A0, A1, A2)                                  \
    {                                                               \
        if (p > ze) break;                                          \
        erode(p, m[A0], m[A1], m[A2], e[A2]);                       \
        if (p + 2 <= ze + 1) load(p + 2, m[A0]);                    \
        if (p - 1 >= zs) dilate(p - 1, e[A0], e[A1], e[A2]);        \
        p++;                                                        \
    }
    for (int p = zs - 1;;) {
        ROIX_OPEN_STEP(0, 1, 2)
        ROIX_OPEN_STEP(1, 2, 0)
        ROIX_OPEN_STEP(2, 0, 1)
    }
#undef ROIX_OPEN_STEP
}

// ----------------------------------------------------------------- 3-D opening, warp-register form
// No shared memory and no block barriers: every warp owns a pencil of RY rows x 32 words (lanes)
// and marches along z keeping the m and e words of 3 planes in registers.  Lanes 0 and 31 hold the
// halo words of the pencil (the words left and right of its 30 output words): e and o bits next to
// the output words only depend on their adjacent bits, which are exact.  Rows y-2, y-1 / y+RY,
// y+RY+1 are the pencil's y-halo (re-read from L1/L2).  Neighbours in x come from the adjacent
// lanes (__shfl), in y from the neighbouring register, in z from the previous/next plane registers.
template <int RY>
__global__ void __launch_bounds__(256, 3) k_open3d_reg(MorphArgs A, roix_scalars *sc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->run_slots = 0;   // no run records from this form
    if (get_err(sc)) return;
    constexpr int MRW = RY + 4, ERW = RY + 2;
    const uint32_t lane = lane_id();
    const int Y = (int)A.ny;
    const uint32_t W = A.W;
    const uint32_t npx = (W + 29) / 30;                       // pencils across a row
    const uint32_t nry = (uint32_t)((A.ny + RY - 1) / RY);     // row groups
    const uint32_t task = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    const uint32_t per_chunk = npx * nry;
    const uint32_t cz = task / per_chunk;
    const uint32_t rem = task - cz * per_chunk;
    const int yb = (int)(rem / npx) * RY;
    const int kw = (int)(rem % npx) * 30 + (int)lane - 1;   // this lane's word column
    const int nz = (int)A.nz;
    const int zs = (int)(cz * A.zchunk);
    if (zs >= nz) return;
    const int ze = min(nz, zs + (int)A.zchunk);
    const bool in_x = kw >= 0 && kw < (int)W;
    const uint32_t tail = (uint32_t)(A.nx - 32ull * (W - 1));
    const uint32_t padm = (kw == (int)W - 1 && tail < 32) ? ~low_mask(tail) : 0u;   // pad bits of the last word
    const bool out_lane = lane >= 1 && lane <= 30 && in_x;
    const uint64_t plane_w = (A.ny * A.nx + 31) / 32;
    const bool aligned = (A.nx & 31) == 0;
    const int64_t gz = (int64_t)A.gz, z0 = (int64_t)A.z0;
    // per-lane offsets (in words) of the pencil's rows inside a plane, and their validity
    const uint32_t wpr = (uint32_t)(A.nx >> 5);   // words per row when aligned
    uint32_t roff[MRW];
    uint32_t vmask = 0;   // bit j: row yb-2+j exists and the lane's column is inside the row
#pragma unroll
    for (int j = 0; j < MRW; j++) {
        const int y = yb - 2 + j;
        roff[j] = (uint32_t)max(y, 0) * wpr + (uint32_t)max(kw, 0);
        if (in_x && y >= 0 && y < Y) vmask |= 1u << j;
    }

    auto load_plane = [&](int p, uint32_t (&mw)[MRW]) {
        const int64_t gp = z0 + p;
        if (gp < 0 || gp >= gz) {
#pragma unroll
            for (int j = 0; j < MRW; j++) mw[j] = FULL;
            return;
        }
        if (aligned && p >= 0 && p < nz) {   // common case: one load per row
            const uint32_t *base = A.m + (uint64_t)p * plane_w;
#pragma unroll
            for (int j = 0; j < MRW; j++) mw[j] = ((vmask >> j) & 1) ? (__ldg(base + roff[j]) | padm) : FULL;
            return;
        }
        // halo planes / unaligned rows: generic bit addressing
        const uint32_t *src;
        uint64_t pb, sw;
        if (p < 0) {
            src = A.halo_lo;
            pb = (uint64_t)(p + 2) * plane_w * 32;
            sw = 2 * plane_w;
        } else if (p >= nz) {
            src = A.halo_hi;
            pb = (uint64_t)(p - nz) * plane_w * 32;
            sw = 2 * plane_w;
        } else {
            src = A.m;
            pb = (uint64_t)p * A.ny * A.nx;
            sw = A.m_words;
        }
#pragma unroll
        for (int j = 0; j < MRW; j++) {
            uint32_t v = FULL;
            if ((vmask >> j) & 1) {
                const uint64_t b = pb + (uint64_t)(yb - 2 + j) * A.nx + 32ull * kw;
                const uint64_t wi = b >> 5;
                const uint32_t sh = (uint32_t)(b & 31);
                v = __ldg(src + wi);
                if (sh) v = __funnelshift_r(v, wi + 1 < sw ? __ldg(src + wi + 1) : 0u, sh);
                v |= padm;
            }
            mw[j] = v;
        }
    };

    uint32_t m0[MRW], m1[MRW], m2[MRW], mn[MRW];   // m of planes p-2, p-1, p; mn: plane p+1 in flight
    uint32_t e0[ERW], e1[ERW], e2[ERW];            // e of planes p-3, p-2, p-1
#pragma unroll
    for (int j = 0; j < MRW; j++) m0[j] = FULL;
    load_plane(zs - 2, m1);
    load_plane(zs - 1, m2);
    load_plane(zs, mn);
#pragma unroll
    for (int j = 0; j < ERW; j++) e0[j] = e1[j] = e2[j] = 0u;
    // e rows yb-1+j exist iff bit j+1 of vmask (same column, row offset by one)
    const uint32_t emask = vmask >> 1;
    uint32_t *const o_base = A.o;
    for (int p = zs; p <= ze + 1; p++) {
#pragma unroll
        for (int j = 0; j < MRW; j++) {
            m0[j] = m1[j];
            m1[j] = m2[j];
            m2[j] = mn[j];
        }
        if (p + 1 <= ze + 1) load_plane(p + 1, mn);   // prefetch: consumed in the next iteration
#pragma unroll
        for (int j = 0; j < ERW; j++) {
            e0[j] = e1[j];
            e1[j] = e2[j];
        }
        // e(p-1), rows yb-1+j
        const int64_t gq = z0 + p - 1;
        const bool qin = gq >= 0 && gq < gz;
#pragma unroll
        for (int j = 0; j < ERW; j++) {
            const uint32_t c = m1[j + 1];
            const uint32_t lw = __shfl_up_sync(FULL, c, 1), rw = __shfl_down_sync(FULL, c, 1);
            const uint32_t l = __funnelshift_l(lane == 0 ? FULL : lw, c, 1);
            const uint32_t r = __funnelshift_r(c, lane == 31 ? FULL : rw, 1);
            const uint32_t v = c & l & r & m1[j] & m1[j + 2] & m0[j + 1] & m2[j + 1];
            e2[j] = (qin && ((emask >> j) & 1)) ? (v & ~padm) : 0u;
        }
        // o(p-2), rows yb+j
        const int z = p - 2;
        if (z >= zs) {
            uint32_t *orow = o_base + (uint64_t)z * plane_w;
#pragma unroll
            for (int j = 0; j < RY; j++) {
                const uint32_t c = e1[j + 1];
                const uint32_t lw = __shfl_up_sync(FULL, c, 1), rw = __shfl_down_sync(FULL, c, 1);
                uint32_t o = c | e1[j] | e1[j + 2] | e0[j + 1] | e2[j + 1];
                o |= __funnelshift_l(lane == 0 ? 0u : lw, c, 1) | __funnelshift_r(c, lane == 31 ? 0u : rw, 1);
                o &= ~padm;
                const int y = yb + j;
                const uint32_t prev = __shfl_up_sync(FULL, o, 1);
                const bool live = y < Y;
                uint32_t cnt = 0;
                if (out_lane && live) {
                    if (aligned) orow[roff[j + 2]] = o;
                    else write_row_atomic(A.o, ((uint64_t)z * A.ny + y) * A.nx, (uint32_t)kw, o);
                    cnt = __popc(o & ~((o << 1) | ((kw > 0) ? (prev >> 31) : 0u)));
                }
                cnt = __reduce_add_sync(FULL, cnt);
                if (lane == 0 && cnt && live && A.row_runs) atomicAdd(&A.row_runs[(uint64_t)z * A.ny + y], cnt);
            }
        }
    }
}

// ------------------------------------------------------------------------------------ 2-D opening
// Rows r = q*Y + y of the slab (q = plane); neighbours only within the same plane.  S = rows per
// step = warps per CTA.  The output rows of a step are contiguous bits [c X, (c+S) X) of o; they are
// assembled from the o rows in shared memory into whole words.
// Warp: the x-runs (x0, x1 exclusive) of a row of W words in shared memory (guard words 0 at [-1] and
// [W]) into slot[0 ..), for a row known to hold at most the slots' count: words with a run start or
// end are found by ballot, their bits walked in order.
__device__ __forceinline__ void row_slots(const uint32_t *od, uint32_t W, uint2 *slot) {
    const uint32_t lane = lane_id();
    uint32_t ns = 0, ne = 0;
    for (uint32_t k0 = 0; k0 < W; k0 += 32) {
        const uint32_t k = k0 + lane;
        const uint32_t w = k < W ? od[k] : 0u;
        const uint32_t lw = k < W ? od[(int)k - 1] : 0u, rw = k + 1 < W ? od[k + 1] : 0u;
        const uint32_t st = w & ~((w << 1) | (lw >> 31)), en = w & ~((w >> 1) | (rw << 31));
        uint32_t bs = __ballot_sync(FULL, st != 0), be = __ballot_sync(FULL, en != 0);
        while (bs) {
            const uint32_t l = __ffs(bs) - 1;
            bs &= bs - 1;
            uint32_t m = __shfl_sync(FULL, st, l);
            while (m) {
                if (lane == 0) slot[ns].x = 32 * (k0 + l) + __ffs(m) - 1;
                m &= m - 1;
                ns++;
            }
        }
        while (be) {
            const uint32_t l = __ffs(be) - 1;
            be &= be - 1;
            uint32_t m = __shfl_sync(FULL, en, l);
            while (m) {
                if (lane == 0) slot[ne].y = 32 * (k0 + l) + __ffs(m);
                m &= m - 1;
                ne++;
            }
        }
    }
}

__global__ void __launch_bounds__(256) k_open2d(MorphArgs A, roix_scalars *sc) {
    extern __shared__ uint32_t smem[];
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->run_slots = A.rs;   // read by a6 after this launch
    if (get_err(sc)) return;
    const uint32_t W = A.W, WS = A.WS;
    constexpr int S = 8;                          // warps per CTA (launched with 256 threads)
    constexpr uint32_t MS = S + 4, ES = S + 2;    // ring slots: constant moduli compile to multiply-shifts
    const int warp = threadIdx.x >> 5;
    uint32_t *mring = smem;            // [MS][WS]
    uint32_t *ering = mring + MS * WS; // [ES][WS]
    uint32_t *orow = ering + ES * WS;  // [S + 1][WS]: ring of o rows (the previous step's last row stays)
    const int64_t Y = A.ny, X = A.nx;
    const int64_t rows = (int64_t)(A.nz * A.ny);
    const int64_t r0 = (int64_t)blockIdx.x * A.rows_per_cta;
    const int64_t r1 = min(rows, r0 + (int64_t)A.rows_per_cta);
    if (r0 >= r1) return;
    for (int i = threadIdx.x; i < (int)MS; i += blockDim.x) {
        mring[i * WS] = FULL;
        mring[i * WS + W + 1] = FULL;
    }
    for (int i = threadIdx.x; i < (int)ES + S + 1; i += blockDim.x) {   // e rows and o rows: zero pad words
        ering[i * WS] = 0;
        ering[i * WS + W + 1] = 0;
    }
    __syncthreads();
    // ring slot of row r >= r0 - 2: from the (32-bit) distance to r0 - 2, constant modulus
    auto mrow = [&](int64_t r) { return mring + ((uint32_t)(r - r0 + 2) % MS) * WS + 1; };
    auto erow = [&](int64_t r) { return ering + ((uint32_t)(r - r0 + 2) % ES) * WS + 1; };
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
        auto orow_of = [&](int64_t rr) { return orow + ((uint32_t)(rr - r0 + 1) % (uint32_t)(S + 1)) * WS + 1; };
        uint32_t *od = orow_of(r);
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
                __syncwarp();
                if (A.rs && runs && runs <= A.rs) row_slots(od, W, A.run_slots + (uint64_t)r * A.rs);
            }
        }
        __syncthreads();
        // write row r (warp w) at global bit r X with plain stores, no zeroing: a word shared by two rows
        // belongs to the later row, which takes the earlier row's tail bits from the o ring (the band
        // starts and ends on word boundaries, so no word is shared between CTAs)
        if (r < r1) {
            const uint64_t Bg = (uint64_t)r * A.nx, Be = Bg + A.nx;
            const uint32_t sh = (uint32_t)(Bg & 31), esh = (uint32_t)(Be & 31);
            const uint64_t wf = Bg >> 5;
            const uint32_t nwo = (uint32_t)(((Be - 1) >> 5) - wf + 1);   // output words the row touches
            uint32_t *dst = A.o + wf;
            if (X < 32) {   // a word may hold several short rows: OR the shared words into a zeroed o
                for (uint32_t j = lane_id(); j < nwo; j += 32) {
                    const uint32_t val = sh == 0 ? od[j] : (j == 0 ? od[0] << sh : __funnelshift_r(od[j - 1], od[j], 32 - sh));
                    const bool whole = (j > 0 || sh == 0) && (j + 1 < nwo || esh == 0);
                    if (whole) dst[j] = val;
                    else if (val) atomicOr(&dst[j], val);
                }
            }
            const uint32_t nown = X < 32 ? 0u : (esh == 0 || r + 1 == rows) ? nwo : nwo - 1;   // the last: row r+1's
            uint32_t tail = 0;   // row r-1's last sh bits (the low bits of word 0)
            if (sh && nown) {
                const uint32_t *pr = orow_of(r - 1);
                const uint32_t b = (uint32_t)(X - sh), a = b >> 5;
                tail = __funnelshift_r(pr[a], pr[a + 1], b & 31) & low_mask(sh);
            }
            for (uint32_t j = lane_id(); j < nown; j += 32) {
                // output word j = row bits [32 j - sh, 32 j - sh + 32)
                const uint32_t val = sh == 0 ? od[j] : (j == 0 ? (od[0] << sh) | tail : __funnelshift_r(od[j - 1], od[j], 32 - sh));
                dst[j] = val;
            }
        }
        __syncthreads();
    }
}

// ------------------------------------------------------- 2-D opening, register rows (32 <= X < 16 K)
// One warp per range of consecutive rows [ra, rb) of the slab (ra, rb multiples of 32, so row ra starts
// on a word boundary and no output word is shared between warps); the whole row is in registers: lane
// l holds words k = l + 32 j (j < J, W + 1 <= 32 J), so every global load and store is coalesced and
// no block barrier is involved.  The warp marches along the rows keeping m of rows s-2, s-1, s and e
// of rows s-3, s-2, s-1; x-neighbour words come from the adjacent lane (one shfl per word and
// direction; lane 0 / 31 take the previous / next chunk's).  In-plane borders: erosion takes a missing
// row or word as all ones, dilation as all zeros (G-11), so rows of other planes are never read (the
// rows past the slab ends are never used unsubstituted).  The output row (X bits at bit p X) is written
// as whole words: the word shared with the next row is held in a register and completed by that row.
// Each row also gets its run count and its first rs run records (a6 reads them instead of the mask for
// rows with at most rs runs).
// Since 32 (J - 1) <= W < 32 J, only the last two chunks hold pad words (k >= W - 1).
//
// Chunks where some word holds two starts or two ends are recorded after the row (their start / end
// bits and running counts parked in shared memory): ranks from ballots of the per-lane counts
// (count >= i for i = 1 .. max), then each lane writes its own bits in order.
template <int J>
__global__ void __launch_bounds__(128, J <= 14 ? 4 : 3) k_open2d_w(MorphArgs A, roix_scalars *sc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) sc->run_slots = A.rs;   // read by a6 after this launch
    if (get_err(sc)) return;
    const uint32_t lane = lane_id();
    const int64_t rows = (int64_t)(A.nz * A.ny);
    const uint64_t X = A.nx, Y = A.ny;
    const uint32_t W = A.W;
    const uint64_t gw = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t ra = A.row_lo + (int64_t)(gw * A.rows_per_cta), rb = min(A.row_hi, ra + (int64_t)A.rows_per_cta);
    if (ra >= rb) return;
    const uint32_t sl = (lane + 31) & 31, sr = (lane + 1) & 31;
    const bool l0 = lane == 0, l31 = lane == 31;
    const uint32_t lt = (1u << lane) - 1u;
    const uint32_t rsl = A.row_runs ? A.rs : 0u;   // run records per row (0: none)
    __shared__ uint32_t park[4][2 * 32 * J];
    __shared__ uint2 park_base[4][J];
    uint32_t *const pst = park[threadIdx.x >> 5], *const pen = pst + 32 * J;
    uint2 *const pbase = park_base[threadIdx.x >> 5];
    // m pads (ones past X) of the last two chunks; e / o take the complement as a keep mask
    uint32_t padA, padB;
    {
        const uint32_t tail = (uint32_t)(X - 32ull * (W - 1));
        auto pad = [&](uint32_t k) { return k >= W ? FULL : (k == W - 1 && tail < 32) ? ~low_mask(tail) : 0u; };
        padA = J >= 2 ? pad(lane + 32 * (J - 2)) : 0u;
        padB = pad(lane + 32 * (J - 1));
    }
    auto padm = [&](int j) -> uint32_t { return j == J - 1 ? padB : j == J - 2 ? padA : 0u; };
    uint32_t raw[J], m0[J], m1[J], m2[J], e0[J], e1[J], e2[J];
    auto issue = [&](int64_t s) {   // raw words k <= W of m row s (one coalesced load per chunk)
        if (s < A.row_lo || s >= A.row_hi) return;   // other planes: never used unsubstituted
        const uint32_t *src = A.m + (((uint64_t)s * X) >> 5);
#pragma unroll
        for (int j = 0; j < J; j++) {
            const uint32_t k = lane + 32 * j;
            if (j + 2 < J || k <= W) raw[j] = __ldg(src + k);
        }
    };
#pragma unroll
    for (int j = 0; j < J; j++) raw[j] = m0[j] = m1[j] = FULL, e0[j] = e1[j] = 0u;
    uint64_t ys = (uint64_t)((ra - 2 + 2 * (int64_t)Y) % (int64_t)Y);   // plane row of s (valid for s >= 0)
    uint32_t carry = 0;
    issue(ra - 2);
#pragma unroll 1
    for (int64_t s = ra - 2; s <= rb + 1; s++) {
        // m row s: funnel of the raw word and the next (the next lane's)
        {
            const uint32_t sh = s >= 0 ? (uint32_t)(((uint64_t)s * X) & 31) : 0u;
            uint32_t nxt = __shfl_sync(FULL, raw[0], sr);
#pragma unroll
            for (int j = 0; j < J; j++) {
                const uint32_t cur = nxt;
                if (j + 1 < J) nxt = __shfl_sync(FULL, raw[j + 1], sr);
                const uint32_t nx = l31 ? (j + 1 < J ? nxt : 0u) : cur;
                m2[j] = __funnelshift_r(raw[j], nx, sh) | padm(j);
            }
        }
        issue(s + 1);
        // e row q = s - 1 from m rows s-2, s-1, s (plane borders: the missing row is all ones)
        const uint64_t yq = ys == 0 ? Y - 1 : ys - 1;
        {
            const uint32_t tm = yq == 0 ? FULL : 0u, bm = yq == Y - 1 ? FULL : 0u;
            uint32_t lrot = __shfl_sync(FULL, m1[0], sl), rrot = __shfl_sync(FULL, m1[0], sr), prevl = FULL;
#pragma unroll
            for (int j = 0; j < J; j++) {
                const uint32_t c = m1[j];
                const uint32_t lw = l0 ? prevl : lrot;
                prevl = lrot;
                uint32_t rw = rrot;
                if (j + 1 < J) {
                    lrot = __shfl_sync(FULL, m1[j + 1], sl);
                    rrot = __shfl_sync(FULL, m1[j + 1], sr);
                    if (l31) rw = rrot;
                } else if (l31) {
                    rw = FULL;
                }
                const uint32_t v = c & __funnelshift_l(lw, c, 1) & __funnelshift_r(c, rw, 1);
                e2[j] = v & (m0[j] | tm) & (m2[j] | bm) & ~padm(j);
            }
        }
        // o row p = s - 2 from e rows s-3, s-2, s-1 (plane borders: the missing row is all zeros)
        const int64_t p = s - 2;
        if (p >= ra) {
            const uint64_t yp = yq == 0 ? Y - 1 : yq - 1;
            const uint32_t tk = yp == 0 ? 0u : FULL, bk = yp == Y - 1 ? 0u : FULL;
            // store: output word t = row bits [32 t - sh, 32 t - sh + 32) at global word wf + t
            const uint64_t B = (uint64_t)p * X, Be = B + X;
            const uint32_t sh = (uint32_t)(B & 31), esh = (uint32_t)(Be & 31);
            const uint64_t wf = B >> 5;
            const uint32_t nwo = (uint32_t)(((Be - 1) >> 5) - wf + 1);
            const bool defer = esh != 0 && p + 1 < rows;   // the last word is completed by row p + 1
            const uint32_t nst = defer ? nwo - 1 : nwo, tl = nwo - 1;
            uint32_t *dst = A.o + wf;
            uint32_t cv = 0;
            uint32_t bs = 0, be = 0;   // starts / ends of the row so far (warp-uniform)
            uint32_t multi = 0;        // chunks parked for the multi-bit record pass
            uint32_t *slot = rsl ? reinterpret_cast<uint32_t *>(A.run_slots + (uint64_t)p * rsl) : nullptr;
            uint32_t lrot = __shfl_sync(FULL, e1[0], sl), rrot = __shfl_sync(FULL, e1[0], sr), prevl = 0u;
            uint32_t prevo = 0u;   // lane 31's o word of the previous chunk
#pragma unroll
            for (int j = 0; j < J; j++) {
                const uint32_t c = e1[j];
                const uint32_t lw = l0 ? prevl : lrot;
                prevl = lrot;
                uint32_t rw = rrot;
                if (j + 1 < J) {
                    lrot = __shfl_sync(FULL, e1[j + 1], sl);
                    rrot = __shfl_sync(FULL, e1[j + 1], sr);
                    if (l31) rw = rrot;
                } else if (l31) {
                    rw = 0u;
                }
                uint32_t v = c | __funnelshift_l(lw, c, 1) | __funnelshift_r(c, rw, 1) | (e0[j] & tk) | (e2[j] & bk);
                v &= ~padm(j);
                const uint32_t orot = __shfl_sync(FULL, v, sl);
                const uint32_t ol = l0 ? prevo : orot;
                prevo = orot;
                const uint32_t t = lane + 32 * j;
                uint32_t val = __funnelshift_l(ol, v, sh);
                if (j == 0 && t == 0) val |= carry;
                if (t < nst) dst[t] = val;
                if (j + 2 >= J && t == tl) cv = val;
                // run starts / exclusive ends of the chunk: records (speculative: the row may turn out
                // to have more than rs runs, then a6 ignores them) and the running counts
                const uint32_t b1 = (v << 1) | (ol >> 31);
                const uint32_t st = v & ~b1, en = ~v & b1;
                if (__any_sync(FULL, (st | en) != 0)) {
                    if (__any_sync(FULL, (st & (st - 1)) | (en & (en - 1)))) {
                        pst[t] = st;
                        pen[t] = en;
                        if (lane == 0) pbase[j] = make_uint2(bs, be);
                        multi |= 1u << j;
                        bs += __reduce_add_sync(FULL, __popc(st));
                        be += __reduce_add_sync(FULL, __popc(en));
                    } else {
                        const uint32_t bS = __ballot_sync(FULL, st != 0), bE = __ballot_sync(FULL, en != 0);
                        if (slot) {
                            const uint32_t is = bs + __popc(bS & lt), ie = be + __popc(bE & lt);
                            if (st && is < rsl) slot[2 * is] = 32 * t + __ffs(st) - 1;
                            if (en && ie < rsl) slot[2 * ie + 1] = 32 * t + __ffs(en) - 1;
                        }
                        bs += __popc(bS);
                        be += __popc(bE);
                    }
                }
            }
            carry = defer ? __shfl_sync(FULL, cv, tl & 31) : 0u;
            if (A.row_runs && lane == 0) A.row_runs[p] = bs;
            if (multi && slot && bs <= rsl) {   // rows with more runs than records never use them
                __syncwarp();
                for (uint32_t mk = multi; mk; mk &= mk - 1) {
                    const uint32_t j = __ffs(mk) - 1, t = lane + 32 * j;
                    const uint32_t st = pst[t], en = pen[t];
                    const uint2 base = pbase[j];
                    const uint32_t cs = __popc(st), ce = __popc(en);
                    const uint32_t cmax = __reduce_max_sync(FULL, max(cs, ce));
                    uint32_t ps = 0, pe = 0;
                    for (uint32_t i = 1; i <= cmax; i++) {
                        ps += __popc(__ballot_sync(FULL, cs >= i) & lt);
                        pe += __popc(__ballot_sync(FULL, ce >= i) & lt);
                    }
                    uint32_t i = base.x + ps;
                    for (uint32_t mm = st; mm && i < rsl; mm &= mm - 1) slot[2 * i++] = 32 * t + __ffs(mm) - 1;
                    i = base.y + pe;
                    for (uint32_t mm = en; mm && i < rsl; mm &= mm - 1) slot[2 * i++ + 1] = 32 * t + __ffs(mm) - 1;
                }
                __syncwarp();
            }
        }
#pragma unroll
        for (int j = 0; j < J; j++) {
            m0[j] = m1[j];
            m1[j] = m2[j];
            e0[j] = e1[j];
            e1[j] = e2[j];
        }
        ys = ys + 1 == Y ? 0 : ys + 1;
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

// a4 on planes [p0, p1) of the slab: x -> m (linear bits; the range starts on a word boundary), at most
// `per_sm` CTAs per SM
static cudaError_t binarize_range(const void *x, int dtype, uint64_t p0, uint64_t p1, const roix_geom &g,
                                  roix_scalars *sc, uint32_t *m, int prebinarized, const roix_frame *frames,
                                  uint32_t per_sm, cudaStream_t st) {
    const uint64_t A = g.ny * g.nx, v0 = p0 * A, n = (p1 - p0) * A;
    if (!n) return cudaSuccess;
    uint64_t iters = (n + 1023) / 1024;
    uint64_t blocks = (iters + 7) / 8;
    const uint64_t cap = (uint64_t)num_sms() * per_sm;
    if (blocks > cap) blocks = cap;
    uint32_t *mm = m + v0 / 32;
    if (frames) {
        const FrameThr F = {frames + p0, A};
        k_binarize<uint16_t, true><<<(unsigned)blocks, 256, 0, st>>>((const uint16_t *)x + v0, n, sc, mm, 0, F);
    } else if (dtype == ROIX_U16) {
        k_binarize<uint16_t><<<(unsigned)blocks, 256, 0, st>>>((const uint16_t *)x + v0, n, sc, mm, prebinarized,
                                                                FrameThr{nullptr, A});
    } else {
        k_binarize<float><<<(unsigned)blocks, 256, 0, st>>>((const float *)x + v0, n, sc, mm, prebinarized,
                                                             FrameThr{nullptr, A});
    }
    return cudaGetLastError();
}

// the register-row opening on rows [r0, r1) (whole planes, r0 X a multiple of 32)
static cudaError_t open2d_w_rows(MorphArgs A, int64_t r0, int64_t r1, uint32_t warps_target, roix_scalars *sc,
                                 cudaStream_t st) {
    const uint32_t J = (A.W + 1 + 31) / 32;
    const void *fn = nullptr;
    switch (J) {
#define ROIX_O2W(JJ) \
    case JJ: fn = (const void *)k_open2d_w<JJ>; break;
        ROIX_O2W(1) ROIX_O2W(2) ROIX_O2W(3) ROIX_O2W(4) ROIX_O2W(5) ROIX_O2W(6) ROIX_O2W(7) ROIX_O2W(8)
        ROIX_O2W(9) ROIX_O2W(10) ROIX_O2W(11) ROIX_O2W(12) ROIX_O2W(13) ROIX_O2W(14) ROIX_O2W(15) ROIX_O2W(16)
#undef ROIX_O2W
    default: return cudaErrorInvalidConfiguration;
    }
    const uint64_t rows = (uint64_t)(r1 - r0);
    if (!rows) return cudaSuccess;
    uint64_t rpw = (rows + warps_target - 1) / warps_target;
    rpw = (rpw + 31) / 32 * 32;   // every warp's rows start on a word boundary
    A.rows_per_cta = rpw;
    A.row_lo = r0;
    A.row_hi = r1;
    const uint64_t nw = (rows + rpw - 1) / rpw;
    void *args[] = {&A, &sc};
    return cudaLaunchKernel(fn, dim3((unsigned)((nw + 3) / 4)), dim3(128), args, 0, st);
}

// a4 + a5 for the in-plane SE with the register-row opening: the slab is cut into chunks of whole
// planes (each starting on a word boundary); chunk c is binarised on the caller's stream and opened on
// a second stream as soon as its mask is complete, so the opening of chunk c (issue-bound, little
// memory traffic) runs beside the binarisation of chunk c + 1 (HBM-bound) -- in-plane openings of
// different planes are independent.  The second stream forks from and joins the caller's stream with
// events, so the whole call stays one stream-ordered operation (and one CUDA-graph capture).
struct SideStream {
    std::mutex lock;   // one caller's fork ... join sequence at a time (the events are shared)
    cudaStream_t s = nullptr;
    cudaEvent_t fork = nullptr, join = nullptr, ready[16] = {};
};

static cudaError_t side_stream(SideStream **out) {
    static SideStream side[64];
    static std::once_flag once[64];
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    if (dev < 0 || dev >= 64) return cudaErrorInvalidDevice;
    SideStream &S = side[dev];
    std::call_once(once[dev], [&S, &e] {
        if ((e = cudaStreamCreateWithFlags(&S.s, cudaStreamNonBlocking)) != cudaSuccess) return;
        if ((e = cudaEventCreateWithFlags(&S.fork, cudaEventDisableTiming)) != cudaSuccess) return;
        if ((e = cudaEventCreateWithFlags(&S.join, cudaEventDisableTiming)) != cudaSuccess) return;
        for (auto &ev : S.ready)
            if ((e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming)) != cudaSuccess) return;
    });
    if (e != cudaSuccess) return e;
    if (!S.s) return cudaErrorNotReady;
    *out = &S;
    return cudaSuccess;
}

static uint64_t gcd_u64(uint64_t a, uint64_t b) {
    while (b) {
        const uint64_t t = a % b;
        a = b;
        b = t;
    }
    return a;
}

// Plane chunks of the two-stream a4 + a5 (mirrored by pipeline.morph_chunks): in-plane SE: 8 chunks,
// each starting on a word boundary; 3-D SE: 16 chunks of >= 8 planes, at least 3 (X = 32 W: every
// plane starts on a word).  Only slabs of >= 2^30 voxels are chunked.
constexpr int se_in_plane = 4;
static uint64_t chunk_planes(const roix_geom &g, uint32_t se) {
    const uint64_t Z = g.nz;
    if (se == 6) return max((uint64_t)8, (Z + 15) / 16);
    const uint64_t PA = g.ny * g.nx;
    const uint64_t quantum = 32 / gcd_u64(PA % 32 ? PA % 32 : 32, 32);   // planes per word-aligned step
    const uint64_t cp = (Z + 7) / 8;
    return (cp + quantum - 1) / quantum * quantum;
}
static int morph_chunks(const roix_geom &g, uint32_t se, int prebinarized) {
    if (prebinarized || g.nz * g.ny * g.nx < (1ull << 30)) return 1;
    const uint64_t cp = chunk_planes(g, se), nch = (g.nz + cp - 1) / cp;
    return (int)(nch >= (se == 6 ? 3u : 2u) ? nch : 1);
}

static cudaError_t open2d_pipelined(const void *x, int dtype, const roix_geom &g, MorphArgs A, roix_scalars *sc,
                                    const roix_frame *frames, int nchunks, cudaStream_t st) {
    cudaError_t e;
    const uint64_t Z = g.nz, Y = g.ny;
    // measured at C3 (chunks, binarisation CTAs per SM, opening warps per SM): (8, 4, 24) 7.62 ms for
    // a4 + a5; (8, 2, 8) 9.22, (8, 1, 16) 14.5 (the binarisation needs its warps), (8, 8, 16) 7.69,
    // (16, 4, 16) 7.93; one chunk (no overlap) 8.53; a high-priority stream for either side: no gain
    // with the SWAR binarisation (fewer issue slots): 3 binarisation CTAs per SM 7.37 ms, 4: 7.55, 2: 8.52;
    // opening warps per SM 24: 7.41, >= 48 (32 rows per warp, the minimum, at C3): 7.21
    constexpr int k_bps = 3, k_wt = 64;
    const uint64_t nch = (uint64_t)nchunks, cp = chunk_planes(g, se_in_plane);
    if (nch < 2) {   // one chunk: plain sequence on the caller's stream
        uint32_t *m = const_cast<uint32_t *>(A.m);
        if ((e = binarize_range(x, dtype, 0, Z, g, sc, m, 0, frames, 8, st)) != cudaSuccess) return e;
        return open2d_w_rows(A, 0, (int64_t)(Z * Y), (uint32_t)num_sms() * 16, sc, st);
    }
    SideStream *S = nullptr;
    if ((e = side_stream(&S)) != cudaSuccess) return e;
    std::lock_guard<std::mutex> guard(S->lock);
    if ((e = cudaEventRecord(S->fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(S->s, S->fork, 0)) != cudaSuccess) return e;
    for (uint64_t c = 0; c < nch; c++) {
        const uint64_t p0 = c * cp, p1 = min(Z, p0 + cp);
        // the binarisation (4 CTAs per SM) leaves room on every SM for the previous chunk's opening
        if ((e = binarize_range(x, dtype, p0, p1, g, sc, const_cast<uint32_t *>(A.m), 0, frames, (uint32_t)k_bps, st)) !=
            cudaSuccess)
            return e;
        cudaEvent_t ev = S->ready[c % 16];
        if ((e = cudaEventRecord(ev, st)) != cudaSuccess) return e;
        if ((e = cudaStreamWaitEvent(S->s, ev, 0)) != cudaSuccess) return e;
        if ((e = open2d_w_rows(A, (int64_t)(p0 * Y), (int64_t)(p1 * Y), (uint32_t)num_sms() * k_wt, sc, S->s)) !=
            cudaSuccess)
            return e;
    }
    if ((e = cudaEventRecord(S->join, S->s)) != cudaSuccess) return e;
    return cudaStreamWaitEvent(st, S->join, 0);
}

// the whole-row 3-D opening on planes [z0, z1) of the slab (reads m planes z0-2 .. z1+1)
static cudaError_t open3d_rows_range(MorphArgs A, int64_t z0, int64_t z1, uint64_t target_warps, uint32_t threads,
                                     roix_scalars *sc, cudaStream_t st) {
    const uint32_t Wd = A.W;
    const uint32_t L = Wd < 32 ? Wd : 32, KW = Wd / L;
    const uint32_t RY = KW == 4 ? 2 : 4;
    const uint64_t nzc = (uint64_t)(z1 - z0);
    if (!nzc) return cudaSuccess;
    // whole-row warps: S = 32 / L segments of RY rows each
    const uint64_t tiles_y = (A.ny + (32 / L) * RY - 1) / ((32 / L) * RY);
    uint64_t chunks = (target_warps + tiles_y - 1) / tiles_y;
    const uint64_t cmax = nzc >= 16 ? nzc / 8 : 1;   // >= 8 planes per warp (3 halo planes re-read)
    if (chunks > cmax) chunks = cmax;
    if (chunks < 1) chunks = 1;
    A.zchunk = (nzc + chunks - 1) / chunks;
    chunks = (nzc + A.zchunk - 1) / A.zchunk;
    A.z_lo = z0;
    A.z_hi = z1;
    const uint32_t wpb = threads / 32;
    const unsigned blocks = (unsigned)((tiles_y * chunks + wpb - 1) / wpb);
#define ROIX_OPEN_ROWS(LL, KK, RR) k_open3d_rows<LL, KK, RR><<<blocks, threads, 0, st>>>(A, sc)
    switch (Wd) {
    case 1: ROIX_OPEN_ROWS(1, 1, 4); break;
    case 2: ROIX_OPEN_ROWS(2, 1, 4); break;
    case 4: ROIX_OPEN_ROWS(4, 1, 4); break;
    case 8: ROIX_OPEN_ROWS(8, 1, 4); break;
    case 16: ROIX_OPEN_ROWS(16, 1, 4); break;
    case 32: ROIX_OPEN_ROWS(32, 1, 4); break;
    case 64: ROIX_OPEN_ROWS(32, 2, 4); break;
    default: ROIX_OPEN_ROWS(32, 4, 2); break;
    }
#undef ROIX_OPEN_ROWS
    return cudaGetLastError();
}

// a4 + a5 for the 3-D SE with the whole-row opening: chunks of planes binarised on the caller's stream;
// chunk c is opened on the second stream once chunk c + 1 is binarised too (its last rows need the two
// planes after it), beside the binarisation of chunk c + 2.
static cudaError_t open3d_pipelined(const void *x, int dtype, const roix_geom &g, MorphArgs A, roix_scalars *sc,
                                    const roix_frame *frames, int nchunks, cudaStream_t st) {
    cudaError_t e;
    const uint64_t Z = g.nz;
    uint32_t *m = const_cast<uint32_t *>(A.m);
    // measured (chunks, binarisation CTAs per SM, opening warps per SM, opening CTA threads), a4 + a5
    // in ms at C4 / C5: one chunk 3.71 / 14.76; (16, 4, 48, 128) 3.37 / 13.24; (8, 4, 48, 128) 3.35 /
    // 13.63; (8, 2, 48, 256) 3.75 / 14.88 (a 256-thread opening CTA does not fit beside 4 binarisation
    // CTAs); (8, 6, 48, 128) 3.78 / 15.55
    // with the SWAR binarisation: 3 binarisation CTAs per SM: C4 3.22 / C5 12.80 ms; 4: 3.37 / 13.25;
    // 2: 3.55 / 14.01
    constexpr int k_bps = 3, k_wt = 64, k_thr = 128;   // opening warps per SM: 32 / 48 / 64 within noise
    const uint64_t nch = (uint64_t)nchunks, cp = chunk_planes(g, 6);
    SideStream *S = nullptr;
    if ((e = side_stream(&S)) != cudaSuccess) return e;
    std::lock_guard<std::mutex> guard(S->lock);
    if ((e = cudaEventRecord(S->fork, st)) != cudaSuccess) return e;
    if ((e = cudaStreamWaitEvent(S->s, S->fork, 0)) != cudaSuccess) return e;
    for (uint64_t c = 0; c <= nch; c++) {
        if (c < nch) {
            const uint64_t p0 = c * cp, p1 = min(Z, p0 + cp);
            if ((e = binarize_range(x, dtype, p0, p1, g, sc, m, 0, frames, (uint32_t)k_bps, st)) != cudaSuccess)
                return e;
            if ((e = cudaEventRecord(S->ready[c % 16], st)) != cudaSuccess) return e;
            if ((e = cudaStreamWaitEvent(S->s, S->ready[c % 16], 0)) != cudaSuccess) return e;
        }
        if (c >= 1) {   // chunk c - 1: its planes and the two after them are binarised
            const uint64_t q0 = (c - 1) * cp, q1 = min(Z, q0 + cp);
            if ((e = open3d_rows_range(A, (int64_t)q0, (int64_t)q1, (uint64_t)num_sms() * k_wt, (uint32_t)k_thr, sc,
                                       S->s)) != cudaSuccess)
                return e;
        }
    }
    if ((e = cudaEventRecord(S->join, S->s)) != cudaSuccess) return e;
    return cudaStreamWaitEvent(st, S->join, 0);
}

size_t morph_workspace_bytes(const roix_geom &g) { return ((g.nz * g.ny * g.nx + 31) / 32 + 64) * 4; }

cudaError_t launch_morph(const void *x, int dtype, const roix_geom &g, uint32_t se, const uint32_t *halo_lo,
                         const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs, void *ws,
                         int prebinarized, cudaStream_t st, const roix_frame *frames, uint2 *run_slots,
                         uint32_t rs) {
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
    A.run_slots = row_runs ? run_slots : nullptr;
    A.rs = A.run_slots ? rs : 0;
    A.z_lo = 0;
    A.z_hi = (int64_t)g.nz;
    const uint64_t n = g.nz * g.ny * g.nx;
    const uint64_t nwords = (n + 31) / 32;
    uint32_t *m = (uint32_t *)ws;
    A.m = m;
    A.m_words = nwords;
    cudaError_t e;
    // in-plane SE: binarise + open in one pass over x (m stays on chip)
    // a4: stream x -> m (after a fused speculative pass: resolve its window, binarise only on a miss)
    if (prebinarized && (e = launch_spec_resolve(x, dtype, g, sc, ws, st)) != cudaSuccess) return e;
    const uint32_t Wd = A.W;
    // plane chunks on two streams pay from ~1 G voxels (C1 / C2: the extra launches cost more than
    // the overlap gains)
    const int nchunks = morph_chunks(g, se, prebinarized);
    const bool o2w = se != 6 && g.nx >= 32 && Wd + 1 <= 32 * 16 && !prebinarized;   // register-row 2-D opening
    if (o2w) return open2d_pipelined(x, dtype, g, A, sc, frames, nchunks, st);
    const bool rows_kernel = g.nx % 32 == 0 && (Wd <= 32 ? (Wd & (Wd - 1)) == 0 : (Wd == 64 || Wd == 128));
    if (se == 6 && rows_kernel && nchunks > 1) return open3d_pipelined(x, dtype, g, A, sc, frames, nchunks, st);
    if ((e = binarize_range(x, dtype, 0, g.nz, g, sc, m, prebinarized, frames, 8, st)) != cudaSuccess) return e;
    int occ = 0;
    if (se == 6 && rows_kernel) {
        if ((e = open3d_rows_range(A, 0, (int64_t)g.nz, (uint64_t)num_sms() * 48, 256, sc, st)) != cudaSuccess) return e;
    } else if (se == 6) {
        // general rows (X % 32 != 0 or other widths): 30-word pencils with halo lanes
        constexpr int RY = 4;
        const uint64_t npx = (A.W + 29) / 30, nry = (g.ny + RY - 1) / RY;
        const uint64_t per_chunk = npx * nry;
        const uint64_t target_warps = (uint64_t)num_sms() * 64;
        uint64_t chunks = (target_warps + per_chunk - 1) / per_chunk;
        const uint64_t cmax = g.nz >= 16 ? g.nz / 8 : 1;   // >= 8 planes per warp (4 halo planes re-read from L2)
        if (chunks > cmax) chunks = cmax;
        if (chunks < 1) chunks = 1;
        A.zchunk = (g.nz + chunks - 1) / chunks;
        chunks = (g.nz + A.zchunk - 1) / A.zchunk;
        A.aligned_out = (g.nx % 32 == 0);
        if (!A.aligned_out && (e = cudaMemsetAsync(o_bits, 0, nwords * 4, st)) != cudaSuccess) return e;
        if (row_runs && (e = cudaMemsetAsync(row_runs, 0, g.nz * g.ny * 4, st)) != cudaSuccess) return e;
        const uint64_t tasks = per_chunk * chunks;
        k_open3d_reg<RY><<<(unsigned)((tasks + 7) / 8), 256, 0, st>>>(A, sc);
    } else {
        const int S = 8;
        size_t sm = (size_t)((S + 4) + (S + 2) + S + 1) * A.WS * 4;
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
        if (g.nx < 32 && (e = cudaMemsetAsync(o_bits, 0, nwords * 4, st)) != cudaSuccess) return e;
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
