// k_compact.cu -- a1+a8 EXTRACT: uniform error-bounded quantisation (BJ north_star, G-2..G-4) of the
// kept voxels, compacted into a dense code stream in increasing linear index (G-17); the paper's
// analogue is the pixel section P(i) of every ROI row.
//
// Work units: a chunk = 1024 voxels (32 mask words of K), a group = 32 chunks (32 K voxels).
//   pass 1  k_ck_count: a warp per group reads the group's 4 KB of K with coalesced 16-byte loads and
//           writes every chunk's kept count (uint16) and the group total;
//   scan    group totals -> uint64 group offsets;
//   pass 2  k_ck_extract: a warp per group, looping over its non-empty chunks only (the counts say
//           which; the next chunk's K word is loaded before the current chunk is processed).
// In pass 2 the chunk is 32 lanes x J slots of 16-byte groups of x (u16: 8 voxels, J = 4; fp32: 4
// voxels, J = 8): slot j of lane l is 16-byte group 32 j + l, so every load instruction is one
// coalesced 512-byte line run.  x is loaded only for groups with a kept voxel (DRAM reads x only
// under kept sectors), quantised in registers, and stored straight to the code stream -- no shared
// memory, no block barrier:
//   * a fully kept group whose output position P is 16-byte aligned: one 16-byte store;
//   * a fully kept group with P = 8A + d (d != 0) whose successor group is also fully kept: it writes
//     the aligned output vector that holds its last d codes and the successor's first 8 - d codes
//     (the successor's codes come from the next lane with shfl; one funnel shift + word selects);
//   * every other kept voxel (partial groups: the two ends of each x-run; the ends of a chunk) is
//     stored element by element.
// So almost every code leaves in a 16-byte store of a warp-contiguous line, and the element path
// costs O(runs), not O(voxels).
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace roix {

constexpr int CK_VOX = 1024;            // voxels per chunk
constexpr int CK_WORDS = CK_VOX / 32;   // mask words per chunk
constexpr int CK_G = 32;                // chunks per group (one warp task)
constexpr int CK_THREADS = 256;

struct CkWS {
    uint16_t *ccnt;      // [nchunks]: kept voxels per chunk
    uint32_t *gcnt;      // [ngroups]: kept voxels per group
    uint64_t *goff;      // [ngroups + 1]: exclusive offsets (totals exceed 2^32 at C3-C5)
    uint64_t *scan_tmp;
    uint32_t *err_snap;  // the error word before extraction (its own errors must not stop it)
};

static size_t ck_carve(void *base, uint64_t n, CkWS *w) {
    const uint64_t nchunks = (n + CK_VOX - 1) / CK_VOX, ngroups = (nchunks + CK_G - 1) / CK_G;
    auto al = [](size_t v) { return (v + 255) & ~(size_t)255; };
    const size_t a = al((nchunks + 1) * 2), b = al((ngroups + 1) * 4), c = al((ngroups + 1) * 8),
                 d = al(scan_tmp_elems(ngroups) * 8);
    if (w) {
        char *p = (char *)base;
        w->ccnt = (uint16_t *)p;
        w->gcnt = (uint32_t *)(p + a);
        w->goff = (uint64_t *)(p + a + b);
        w->scan_tmp = (uint64_t *)(p + a + b + c);
        w->err_snap = (uint32_t *)(p + a + b + c + d);
    }
    return a + b + c + d + 256;
}

// ------------------------------------------------------------------------------------- pass 1
// Warp per group: load i (0..7) of lane l covers 16 bytes = words 4 (32 i + l) .. +3 of the group,
// i.e. chunk 4 i + l / 8; eight lanes share a chunk and reduce with shfl_xor.
__global__ void __launch_bounds__(CK_THREADS) k_ck_count(const uint32_t *__restrict__ K, uint64_t n, uint64_t nchunks,
                                                         uint64_t ngroups, CkWS w, const roix_scalars *sc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *w.err_snap = sc->err;
    const uint64_t nwords = (n + 31) / 32;
    const uint32_t lane = lane_id();
    const uint64_t nw = (uint64_t)gridDim.x * (CK_THREADS / 32);
    for (uint64_t g = (uint64_t)blockIdx.x * (CK_THREADS / 32) + (threadIdx.x >> 5); g < ngroups; g += nw) {
        const uint64_t w0 = g * (CK_G * CK_WORDS);
        uint4 v[8];
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const uint64_t wi = w0 + 4ull * (32 * i + lane);
            if (wi + 4 <= nwords) v[i] = __ldcs(reinterpret_cast<const uint4 *>(K + wi));
            else {
                v[i].x = wi < nwords ? K[wi] : 0u;
                v[i].y = wi + 1 < nwords ? K[wi + 1] : 0u;
                v[i].z = wi + 2 < nwords ? K[wi + 2] : 0u;
                v[i].w = 0u;
            }
        }
        uint32_t mine = 0;
#pragma unroll
        for (int i = 0; i < 8; i++) {
            uint32_t c = __popc(v[i].x) + __popc(v[i].y) + __popc(v[i].z) + __popc(v[i].w);
            c += __shfl_xor_sync(FULL, c, 1);
            c += __shfl_xor_sync(FULL, c, 2);
            c += __shfl_xor_sync(FULL, c, 4);
            const uint32_t t = __shfl_sync(FULL, c, 8 * (lane & 3));   // chunk 4 i + (lane & 3)
            if ((lane >> 2) == (uint32_t)i) mine = t;
        }
        const uint64_t c = g * CK_G + lane;
        if (c < nchunks) w.ccnt[c] = (uint16_t)mine;
        const uint32_t tot = __reduce_add_sync(FULL, mine);
        if (lane == 0) w.gcnt[g] = tot;
    }
}

// ------------------------------------------------------------------------------------- pass 2
// Halfword shift of the 16 halfwords S = (W[0..7]) by sh halfwords (0..8): returns S[sh .. sh+8) as
// four words.  First by sh & 1 halfword (funnel shifts), then by sh >> 1 words (two select levels).
__device__ __forceinline__ uint4 shift_hw(const uint32_t (&W)[8], uint32_t sh) {
    const uint32_t f = (sh & 1u) * 16u;
    uint32_t V[7];
#pragma unroll
    for (int i = 0; i < 7; i++) V[i] = __funnelshift_r(W[i], W[i + 1], f);
    const uint32_t s = sh >> 1, b0 = s & 1u, b1 = s & 2u;
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t t = b0 ? V[k + 1] : V[k];
        const uint32_t u = b0 ? V[k + 3] : V[k + 2];
        o[k] = b1 ? u : t;
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

template <typename T>
struct CkTraits;
template <>
struct CkTraits<uint16_t> {
    static constexpr int VPG = 8, J = 4;      // voxels per 16-byte group; slots per lane
};
template <>
struct CkTraits<float> {
    static constexpr int VPG = 4, J = 8;
};

// the 16-byte group of codes of one 16-byte group of x (u16 -> 8 uint16 codes, fp32 -> 4 int32)
template <typename T, int QM>
__device__ __forceinline__ uint4 quant16(uint4 d, const QP &q, uint32_t &err) {
    if constexpr (sizeof(T) == 2) {
        return make_uint4(code_pair_u16_m<QM>(d.x, q, err), code_pair_u16_m<QM>(d.y, q, err),
                          code_pair_u16_m<QM>(d.z, q, err), code_pair_u16_m<QM>(d.w, q, err));
    } else {
        return make_uint4((uint32_t)code_f32(__uint_as_float(d.x), q, err), (uint32_t)code_f32(__uint_as_float(d.y), q, err),
                          (uint32_t)code_f32(__uint_as_float(d.z), q, err), (uint32_t)code_f32(__uint_as_float(d.w), q, err));
    }
}

template <typename C>
__device__ __forceinline__ uint32_t code_k(const uint4 &e, int k) {   // k static
    if constexpr (sizeof(C) == 2) {
        const uint32_t wd = (k >> 1) == 0 ? e.x : (k >> 1) == 1 ? e.y : (k >> 1) == 2 ? e.z : e.w;
        return (k & 1) ? (wd >> 16) : (wd & 0xffffu);
    } else {
        return k == 0 ? e.x : k == 1 ? e.y : k == 2 ? e.z : e.w;
    }
}

// A fully kept chunk (every voxel kept: the interior of long runs, most of C3 / C4): group g's codes
// go to cbase + V g, one misalignment d for the whole chunk, so every aligned output vector is a fixed
// shift of two neighbouring groups -- no flags, no scans; only the chunk's first and last vectors
// (shared with the neighbouring chunks) go element by element.
template <typename T, typename C, int QM>
__device__ __noinline__ void ck_full(const T *__restrict__ x, uint64_t c, uint64_t cbase, C *__restrict__ out,
                                     const QP q, uint32_t &err) {
    constexpr int VPG = CkTraits<T>::VPG, J = CkTraits<T>::J;
    const uint32_t lane = lane_id();
    const uint64_t v0 = c * CK_VOX;
    uint4 e[J];
#pragma unroll
    for (int j = 0; j < J; j++) e[j] = __ldcs(reinterpret_cast<const uint4 *>(x + v0 + (uint64_t)(32 * j + lane) * VPG));
    const uint32_t d = (uint32_t)(cbase % VPG);
    const uint64_t ab = cbase - d;
#pragma unroll
    for (int j = 0; j < J; j++) e[j] = quant16<T, QM>(e[j], q, err);
#pragma unroll
    for (int j = 0; j < J; j++) {
        const uint32_t g = 32 * j + lane;
        if (d == 0) {
            __stcs(reinterpret_cast<uint4 *>(out + ab + (uint64_t)VPG * g), e[j]);
            continue;
        }
        // the vector after group g's first code: g's last d codes, then g+1's first VPG - d
        const uint4 ns = (lane == 0 && j + 1 < J) ? e[j + 1 < J ? j + 1 : j] : e[j];
        uint4 ne;
        ne.x = __shfl_sync(FULL, ns.x, (lane + 1) & 31);
        ne.y = __shfl_sync(FULL, ns.y, (lane + 1) & 31);
        ne.z = __shfl_sync(FULL, ns.z, (lane + 1) & 31);
        ne.w = __shfl_sync(FULL, ns.w, (lane + 1) & 31);
        if (!(lane == 31 && j == J - 1)) {
            const uint32_t W8[8] = {e[j].x, e[j].y, e[j].z, e[j].w, ne.x, ne.y, ne.z, ne.w};
            __stcs(reinterpret_cast<uint4 *>(out + ab + (uint64_t)VPG * (g + 1)),
                   shift_hw(W8, (VPG - d) * (uint32_t)(sizeof(C) / 2)));
        } else {   // the chunk's last group: its next group is in the next chunk
#pragma unroll
            for (int k = 0; k < VPG; k++)
                if ((uint32_t)k >= VPG - d) out[ab + (uint64_t)VPG * g + d + k] = (C)code_k<C>(e[j], k);
        }
        if (g == 0) {   // the chunk's first vector: its first VPG - d codes
#pragma unroll
            for (int k = 0; k < VPG; k++)
                if ((uint32_t)k < VPG - d) out[ab + d + k] = (C)code_k<C>(e[j], k);
        }
    }
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void ck_chunk(const T *__restrict__ x, uint64_t n, uint64_t c, uint32_t kw, uint64_t cbase,
                                         uint32_t ccount, C *__restrict__ out, uint64_t capacity, const QP &q,
                                         uint32_t &err) {
    constexpr int VPG = CkTraits<T>::VPG, J = CkTraits<T>::J;
    constexpr int GPW = 32 / VPG;                 // 16-byte groups per mask word
    constexpr uint32_t GM = (1u << VPG) - 1u;     // a full group's mask
    const uint32_t lane = lane_id();
    const uint64_t v0 = c * CK_VOX;
    if (cbase + ccount > capacity) err |= ROIX_ERR_CAPACITY;
    // masks of the lane's groups (slot j = group 32 j + lane)
    uint32_t mb[J];
#pragma unroll
    for (int j = 0; j < J; j++)
        mb[j] = (__shfl_sync(FULL, kw, j * (32 / GPW) + lane / GPW) >> ((lane % GPW) * VPG)) & GM;
    // x only under kept groups
    uint4 e[J];
    const bool whole = v0 + CK_VOX <= n;
#pragma unroll
    for (int j = 0; j < J; j++) {
        e[j] = make_uint4(0, 0, 0, 0);
        const uint64_t gv = v0 + (uint64_t)(32 * j + lane) * VPG;
        if (mb[j]) {
            if (whole) e[j] = __ldcs(reinterpret_cast<const uint4 *>(x + gv));
            else {   // the volume's last chunk: no 16-byte load past n
                uint32_t wd[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                for (int k = 0; k < VPG; k++) {
                    if (gv + k >= n) break;
                    uint32_t b;
                    if constexpr (sizeof(T) == 2) b = (uint32_t)x[gv + k] << (16 * (k & 1));
                    else b = __float_as_uint(x[gv + k]);
                    wd[sizeof(T) == 2 ? k >> 1 : k] |= b;
                }
                e[j] = make_uint4(wd[0], wd[1], wd[2], wd[3]);
            }
        }
    }
    // chunk-relative exclusive prefix of every group (order: slot-major, lane-minor), two slots
    // per 32-bit word (16-bit fields: a chunk holds at most 1024 codes)
    uint32_t pre[J];
    {
        uint32_t run = 0;
#pragma unroll
        for (int j = 0; j < J; j += 2) {
            const uint32_t c0 = __popc(mb[j]), c1 = __popc(mb[j + 1]);
            const uint32_t pk = c0 | (c1 << 16);
            const uint32_t inc = warp_incl_scan(pk);
            const uint32_t tot = __shfl_sync(FULL, inc, 31);
            pre[j] = run + (inc & 0xffffu) - c0;
            run += tot & 0xffffu;
            pre[j + 1] = run + (inc >> 16) - c1;
            run += tot >> 16;
        }
    }
    // quantise (only kept groups carry data; the rest stay zero and are never stored)
#pragma unroll
    for (int j = 0; j < J; j++)
        if (mb[j]) e[j] = quant16<T, QM>(e[j], q, err);
    // neighbours in output order: next of (j, l) is (j, l+1), or (j+1, 0) for l = 31; prev likewise
#pragma unroll
    for (int j = 0; j < J; j++) {
        if (__ballot_sync(FULL, mb[j]) == 0) continue;   // warp-uniform skip of an empty slot row
        const uint32_t nsrc = (lane + 1) & 31u, psrc = (lane + 31) & 31u;
        // value lane 0 offers to lane 31 is slot j+1's; value lane 31 offers to lane 0 is slot j-1's
        const uint32_t mb_next_src = (lane == 0) ? (j + 1 < J ? mb[j + 1 < J ? j + 1 : j] : 0u) : mb[j];
        const uint32_t mb_prev_src = (lane == 31) ? (j > 0 ? mb[j > 0 ? j - 1 : j] : 0u) : mb[j];
        const uint32_t nmb = __shfl_sync(FULL, mb_next_src, nsrc);
        const uint32_t pmb = __shfl_sync(FULL, mb_prev_src, psrc);
        const uint4 ns = (lane == 0 && j + 1 < J) ? e[j + 1 < J ? j + 1 : j] : e[j];
        uint4 ne;
        ne.x = __shfl_sync(FULL, ns.x, nsrc);
        ne.y = __shfl_sync(FULL, ns.y, nsrc);
        ne.z = __shfl_sync(FULL, ns.z, nsrc);
        ne.w = __shfl_sync(FULL, ns.w, nsrc);
        // lane 31's next / lane 0's prev outside the chunk: treated as not fully kept
        const uint32_t m = mb[j];
        if (!m) continue;
        const uint64_t P = cbase + pre[j];
        // a fully kept neighbour in the chunk shares an aligned output vector with this group; it is
        // stored as a vector when it lies below the capacity (both lanes evaluate the same test)
        const uint64_t Ah = P - (P % VPG);   // the aligned vector holding P
        const bool next_full = nmb == GM && !(lane == 31 && j + 1 >= J) && Ah + 2 * VPG <= capacity;
        const bool prev_full = pmb == GM && !(lane == 0 && j == 0) && Ah + VPG <= capacity;
        uint32_t em;   // codes stored element by element
        if (m == GM) {
            const uint32_t d = (uint32_t)(P % VPG);
            if (d == 0) {
                if (P + VPG <= capacity) __stcs(reinterpret_cast<uint4 *>(out + P), e[j]);
                em = P + VPG <= capacity ? 0u : GM;
            } else {
                const uint32_t head = (1u << (VPG - d)) - 1u;   // codes in the aligned vector before P's
                em = (prev_full ? 0u : head) | (next_full ? 0u : (GM & ~head));
                if (next_full) {   // aligned vector: our last d codes, then the next group's first VPG - d
                    const uint32_t W[8] = {e[j].x, e[j].y, e[j].z, e[j].w, ne.x, ne.y, ne.z, ne.w};
                    const uint32_t sh = (VPG - d) * (uint32_t)(sizeof(C) / 2);   // halfwords: u16 8-d, fp32 2(4-d)
                    __stcs(reinterpret_cast<uint4 *>(out + Ah + VPG), shift_hw(W, sh));
                }
            }
        } else {
            em = m;
        }
        if (em) {
            C *const ob = out + P;   // the group's kept codes go to P, P + 1, ... (32-bit offsets)
            if (P + VPG <= capacity) {
#pragma unroll
                for (int k = 0; k < VPG; k++)
                    if ((em >> k) & 1u) ob[__popc(m & ((1u << k) - 1u))] = (C)code_k<C>(e[j], k);
            } else {
#pragma unroll
                for (int k = 0; k < VPG; k++) {
                    if (!((em >> k) & 1u)) continue;
                    const uint64_t dst = P + __popc(m & ((1u << k) - 1u));
                    if (dst < capacity) out[dst] = (C)code_k<C>(e[j], k);
                }
            }
        }
    }
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void ck_group(const T *__restrict__ x, uint64_t n, const uint32_t *__restrict__ K,
                                         uint64_t nchunks, const CkWS &w, uint64_t g, uint32_t part, uint32_t cpp,
                                         uint64_t off0, C *__restrict__ out, uint64_t capacity, const QP &q,
                                         uint32_t &err) {
    const uint64_t gbase = w.goff[g];
    if (w.goff[g + 1] == gbase) return;   // no kept voxel in 32 K voxels (background)
    const uint32_t lane = lane_id();
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t c0 = g * CK_G;
    const uint32_t cc = c0 + lane < nchunks ? (uint32_t)w.ccnt[c0 + lane] : 0u;
    const uint32_t excl = warp_incl_scan(cc) - cc;
    // this task's chunks: [part cpp, (part + 1) cpp) of the group (small volumes split groups)
    const uint32_t pm = cpp >= 32 ? FULL : (((1u << cpp) - 1u) << (part * cpp));
    uint32_t rem = __ballot_sync(FULL, cc != 0) & pm;
    if (!rem) return;
    auto ldk = [&](int k) -> uint32_t {
        const uint64_t wi = (c0 + k) * CK_WORDS + lane;
        return wi < nwords ? __ldcs(K + wi) : 0u;
    };
    int k = __ffs(rem) - 1;
    uint32_t kw = ldk(k);
    while (k >= 0) {
        rem &= rem - 1;
        const int kn = rem ? __ffs(rem) - 1 : -1;
        const uint32_t kw_next = kn >= 0 ? ldk(kn) : 0u;   // in flight while this chunk is processed
        const uint64_t cbase = off0 + gbase + __shfl_sync(FULL, excl, k);
        const uint32_t ccount = __shfl_sync(FULL, cc, k);
        if (ccount == CK_VOX && (c0 + k + 1) * CK_VOX <= n && cbase + CK_VOX <= capacity)
            ck_full<T, C, QM>(x, c0 + k, cbase, out, q, err);
        else
            ck_chunk<T, C, QM>(x, n, c0 + k, kw, cbase, ccount, out, capacity, q, err);
        k = kn;
        kw = kw_next;
    }
}

template <typename T, typename C>
__global__ void __launch_bounds__(CK_THREADS, sizeof(T) == 2 ? 4 : 3)
    k_ck_extract(const T *__restrict__ x, uint64_t n, const uint32_t *__restrict__ K, uint64_t nchunks,
                 uint64_t ngroups, uint32_t parts, CkWS w, roix_scalars *sc, C *__restrict__ out,
                 uint64_t capacity, const uint64_t *offset) {
    if (*w.err_snap) return;
    const uint64_t t = (uint64_t)blockIdx.x * (CK_THREADS / 32) + (threadIdx.x >> 5);
    const uint64_t g = t / parts;
    if (g >= ngroups) return;
    const uint32_t part = (uint32_t)(t % parts), cpp = CK_G / parts;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t off0 = offset ? *offset : 0ull;
    if constexpr (sizeof(T) == 4) {
        ck_group<T, C, QM_FLOAT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err);
    } else {
        switch (qmode(q)) {   // uniform over the launch: one quantiser body per mode
        case QM_POW2: ck_group<T, C, QM_POW2>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        case QM_INT: ck_group<T, C, QM_INT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        case QM_ONE: ck_group<T, C, QM_ONE>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        default: ck_group<T, C, QM_FLOAT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        }
    }
    err = __reduce_or_sync(FULL, err);
    if (err && lane_id() == 0) set_err(sc, err);
}

__global__ void k_ck_total(const uint64_t *total, const uint32_t *err_snap, roix_scalars *sc) {
    if (*err_snap == 0) sc->count += *total;
}

}  // namespace roix

using namespace roix;

size_t compact_workspace_bytes(uint64_t n) { return ck_carve(nullptr, n, nullptr); }

cudaError_t launch_compact(const void *x, int dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                           void *codes, uint64_t capacity, const uint64_t *offset, void *ws, cudaStream_t st) {
    CkWS w;
    ck_carve(ws, n, &w);
    const uint64_t nchunks = (n + CK_VOX - 1) / CK_VOX, ngroups = (nchunks + CK_G - 1) / CK_G;
    const uint64_t wpc = CK_THREADS / 32;
    uint64_t g1 = (ngroups + wpc - 1) / wpc;
    const uint64_t cap1 = (uint64_t)num_sms() * 8;
    k_ck_count<<<(unsigned)(g1 < cap1 ? (g1 ? g1 : 1) : cap1), CK_THREADS, 0, st>>>(keep_bits, n, nchunks, ngroups, w,
                                                                                  sc);
    cudaError_t e = scan_u32_u64(w.gcnt, w.goff, ngroups, w.scan_tmp, st);
    if (e != cudaSuccess) return e;
    // warp tasks: a group, or a part of one when there are too few groups to fill the GPU
    uint32_t parts = 1;
    while (parts < (uint32_t)CK_G && ngroups * parts < (uint64_t)num_sms() * 64) parts *= 2;
    const uint64_t tasks = ngroups * parts;
    const unsigned g2 = (unsigned)((tasks + wpc - 1) / wpc);
    if (g2) {
        if (dtype == ROIX_F32)
            k_ck_extract<float, int32_t><<<g2, CK_THREADS, 0, st>>>((const float *)x, n, keep_bits, nchunks, ngroups,
                                                                    parts, w, sc, (int32_t *)codes, capacity, offset);
        else
            k_ck_extract<uint16_t, uint16_t><<<g2, CK_THREADS, 0, st>>>((const uint16_t *)x, n, keep_bits, nchunks,
                                                                        ngroups, parts, w, sc, (uint16_t *)codes,
                                                                        capacity, offset);
    }
    k_ck_total<<<1, 1, 0, st>>>(scan_total_ptr(w.scan_tmp, ngroups), w.err_snap, sc);
    return cudaGetLastError();
}
