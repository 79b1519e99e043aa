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

// code k (runtime, 0 <= k < VPG) of a 16-byte group of codes
template <typename C>
__device__ __forceinline__ uint32_t code_at(const uint4 &e, uint32_t k) {
    if constexpr (sizeof(C) == 2) {
        const uint32_t h = k >> 1;
        const uint32_t lo = h & 1u ? e.y : e.x, hi = h & 1u ? e.w : e.z;
        const uint32_t wd = h & 2u ? hi : lo;
        return (wd >> ((k & 1u) * 16u)) & 0xffffu;
    } else {
        const uint32_t lo = k & 1u ? e.y : e.x, hi = k & 1u ? e.w : e.z;
        return k & 2u ? hi : lo;
    }
}

// The aligned output vector holding the last d codes of a fully kept group a and the first VPG - d
// codes of the next fully kept group b: elements [VPG - d, 2 VPG - d) of (a, b).
template <int SH>   // shift in halfwords, 1..7
__device__ __forceinline__ uint4 shift_c(const uint4 &a, const uint4 &b) {
    const uint32_t W[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    constexpr int w0 = SH >> 1;
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; k++) o[k] = (SH & 1) ? __funnelshift_r(W[w0 + k], W[w0 + k + 1], 16) : W[w0 + k];
    return make_uint4(o[0], o[1], o[2], o[3]);
}
// branch-free (lanes of a warp may hold different d): a halfword funnel step, then two word selects
template <typename C>
__device__ __forceinline__ uint4 pair_vector(const uint4 &a, const uint4 &b, uint32_t d) {
    const uint32_t sh = sizeof(C) == 2 ? 8u - d : 2u * (4u - d);   // shift in halfwords
    const uint32_t W[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t f = (sh & 1u) * 16u;
    uint32_t V[7];
#pragma unroll
    for (int i = 0; i < 7; i++) V[i] = __funnelshift_r(W[i], W[i + 1], f);
    const uint32_t s = sh >> 1;
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t t = (s & 1u) ? V[k + 1] : V[k];
        const uint32_t u = (s & 1u) ? V[k + 3] : V[k + 2];
        o[k] = (s & 2u) ? u : t;
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

template <typename T, int J>
__device__ __forceinline__ void ck_masks(uint32_t kw, uint32_t (&mb)[J]) {
    constexpr int VPG = CkTraits<T>::VPG, GPW = 32 / VPG;
    const uint32_t lane = lane_id();
#pragma unroll
    for (int j = 0; j < J; j++)
        mb[j] = (__shfl_sync(FULL, kw, j * (32 / GPW) + lane / GPW) >> ((lane % GPW) * VPG)) & ((1u << VPG) - 1u);
}

// x of the kept 16-byte groups of chunk c (zero elsewhere)
template <typename T, int J>
__device__ __forceinline__ void ck_load(const T *__restrict__ x, uint64_t n, uint64_t c, const uint32_t (&mb)[J],
                                        uint4 (&e)[J]) {
    constexpr int VPG = CkTraits<T>::VPG;
    const uint32_t lane = lane_id();
    const uint64_t v0 = c * CK_VOX;
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
}

template <typename T, typename C, int QM, int J>
__device__ __forceinline__ void ck_chunk(const uint32_t (&mb)[J], uint4 (&e)[J], uint64_t cbase, uint32_t ccount,
                                         C *__restrict__ out, uint64_t capacity, const QP &q, uint32_t &err) {
    constexpr int VPG = CkTraits<T>::VPG;
    constexpr uint32_t GM = (1u << VPG) - 1u;     // a full group's mask
    const uint32_t lane = lane_id();
    if (cbase + ccount > capacity) err |= ROIX_ERR_CAPACITY;
    // output positions relative to the aligned vector holding the chunk's first code
    const uint32_t d0 = (uint32_t)(cbase % VPG);
    const uint64_t ab = cbase - d0;
    C *ob = out + ab;
    const uint32_t caprel = capacity <= ab ? 0u : (uint32_t)min(capacity - ab, (uint64_t)0xffff0000u);
    // chunk-relative exclusive prefix of every group (slot-major, lane-minor order), two slots per
    // 32-bit word (16-bit fields: a chunk holds at most 1024 codes)
    uint32_t pos[J];
    {
        uint32_t run = d0;
#pragma unroll
        for (int j = 0; j < J; j += 2) {
            const uint32_t c0 = __popc(mb[j]), c1 = __popc(mb[j + 1]);
            const uint32_t inc = warp_incl_scan(c0 | (c1 << 16));
            const uint32_t tot = __shfl_sync(FULL, inc, 31);
            pos[j] = run + (inc & 0xffffu) - c0;
            run += tot & 0xffffu;
            pos[j + 1] = run + (inc >> 16) - c1;
            run += tot >> 16;
        }
    }
#pragma unroll
    for (int j = 0; j < J; j++)
        if (mb[j]) e[j] = quant16<T, QM>(e[j], q, err);
    uint32_t F[J];   // lanes whose group in slot j is fully kept
#pragma unroll
    for (int j = 0; j < J; j++) F[j] = __ballot_sync(FULL, mb[j] == GM);
#pragma unroll
    for (int j = 0; j < J; j++) {
        if (__ballot_sync(FULL, mb[j]) == 0) continue;   // warp-uniform skip of an empty slot row
        const uint32_t m = mb[j];
        const bool full = m == GM;
        // neighbours in output order: next of (j, l) is (j, l+1), or (j+1, 0) for l = 31; the chunk's
        // first and last group have none (their shared vectors go element by element)
        const bool next_full = lane < 31 ? (F[j] >> (lane + 1)) & 1u : (j + 1 < J ? F[j + 1 < J ? j + 1 : j] & 1u : 0u);
        const bool prev_full = lane > 0 ? (F[j] >> (lane - 1)) & 1u : (j > 0 ? F[j > 0 ? j - 1 : j] >> 31 : 0u);
        const uint32_t p = pos[j], d = p % VPG, A = p - d;
        const bool vec_own = full && d == 0 && A + VPG <= caprel;
        const bool vec_next = full && d != 0 && next_full && A + 2 * VPG <= caprel;
        const bool by_prev = full && d != 0 && prev_full && A + VPG <= caprel;   // prev wrote vector A
        if (__ballot_sync(FULL, vec_next)) {
            const uint32_t nsrc = (lane + 1) & 31u;
            const uint4 ns = (lane == 0 && j + 1 < J) ? e[j + 1 < J ? j + 1 : j] : e[j];
            uint4 ne;
            ne.x = __shfl_sync(FULL, ns.x, nsrc);
            ne.y = __shfl_sync(FULL, ns.y, nsrc);
            ne.z = __shfl_sync(FULL, ns.z, nsrc);
            ne.w = __shfl_sync(FULL, ns.w, nsrc);
            if (vec_next) __stcs(reinterpret_cast<uint4 *>(ob + A + VPG), pair_vector<C>(e[j], ne, d));
        }
        if (vec_own) __stcs(reinterpret_cast<uint4 *>(ob + A), e[j]);
        uint32_t em = m;   // codes stored element by element
        if (full) {
            const uint32_t head = (1u << (VPG - d)) - 1u;   // codes in vector A
            em = vec_own ? 0u : d == 0 ? GM : ((by_prev ? 0u : head) | (vec_next ? 0u : GM & ~head));
        }
        if (em) {
#pragma unroll
            for (int k = 0; k < VPG; k++) {
                const uint32_t dst = p + __popc(m & ((1u << k) - 1u));
                if (((em >> k) & 1u) && dst < caprel) ob[dst] = (C)code_at<C>(e[j], (uint32_t)k);
            }
        }
    }
}

// one warp task: chunks [part * cpp, (part + 1) * cpp) of group g, non-empty ones only; the next
// chunk's x (u16: double-buffered) and the one after's K word are in flight while a chunk is processed
template <typename T, typename C, int QM>
__device__ __forceinline__ void ck_task(const T *__restrict__ x, uint64_t n, const uint32_t *__restrict__ K,
                                        uint64_t nchunks, const CkWS &w, uint64_t g, uint32_t part, uint32_t cpp,
                                        uint64_t off0, C *__restrict__ out, uint64_t capacity, const QP &q,
                                        uint32_t &err) {
    constexpr int J = CkTraits<T>::J;
    const uint64_t gbase = w.goff[g];
    if (w.goff[g + 1] == gbase) return;   // no kept voxel in 32 K voxels (background)
    const uint32_t lane = lane_id();
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t c0 = g * CK_G;
    const uint32_t cc = c0 + lane < nchunks ? (uint32_t)w.ccnt[c0 + lane] : 0u;
    const uint32_t excl = warp_incl_scan(cc) - cc;
    const uint32_t pm = cpp >= 32 ? FULL : (((1u << cpp) - 1u) << (part * cpp));
    uint32_t rem = __ballot_sync(FULL, cc != 0) & pm;
    if (!rem) return;
    auto ldk = [&](int k) -> uint32_t {
        if (k < 0) return 0u;
        const uint64_t wi = (c0 + k) * CK_WORDS + lane;
        return wi < nwords ? __ldcs(K + wi) : 0u;
    };
    auto nextk = [&](uint32_t &r) -> int {
        const int k = r ? __ffs(r) - 1 : -1;
        if (r) r &= r - 1;
        return k;
    };
    // the K word of the chunk after next is in flight while a chunk is processed (per-group L2
    // prefetches of the next chunk's x were measured and did not pay: the kernel is issue-bound)
    int k = nextk(rem);
    const uint32_t kw = ldk(k);
    int kn = nextk(rem);
    uint32_t kwn = ldk(kn);
    uint32_t mb[J], mbn[J];
    uint4 e[J];
    ck_masks<T, J>(kw, mb);
    ck_load<T, J>(x, n, c0 + k, mb, e);
    ck_masks<T, J>(kwn, mbn);
    while (k >= 0) {
        const int knn = nextk(rem);
        const uint32_t kwnn = ldk(knn);   // arrives while chunk k is processed
        const uint64_t cbase = off0 + gbase + __shfl_sync(FULL, excl, k);
        const uint32_t ccount = __shfl_sync(FULL, cc, k);
        ck_chunk<T, C, QM, J>(mb, e, cbase, ccount, out, capacity, q, err);
        if (kn >= 0) {
#pragma unroll
            for (int j = 0; j < J; j++) mb[j] = mbn[j];
            ck_load<T, J>(x, n, c0 + kn, mb, e);
        }
        ck_masks<T, J>(kwnn, mbn);
        k = kn;
        kn = knn;
    }
}

template <typename T, typename C>
__global__ void __launch_bounds__(CK_THREADS, sizeof(T) == 2 ? 4 : 3)
    k_ck_extract(const T *__restrict__ x, uint64_t n, const uint32_t *__restrict__ K, uint64_t nchunks,
                 uint64_t ngroups, uint32_t parts, CkWS w, roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                 const uint64_t *offset) {
    if (*w.err_snap) return;
    const uint64_t t = (uint64_t)blockIdx.x * (CK_THREADS / 32) + (threadIdx.x >> 5);
    const uint64_t g = t / parts;
    if (g >= ngroups) return;
    const uint32_t part = (uint32_t)(t % parts), cpp = CK_G / parts;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t off0 = offset ? *offset : 0ull;
    if constexpr (sizeof(T) == 4) {
        ck_task<T, C, QM_FLOAT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err);
    } else {
        switch (qmode(q)) {   // uniform over the launch: one quantiser body per mode
        case QM_POW2: ck_task<T, C, QM_POW2>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        case QM_INT: ck_task<T, C, QM_INT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        case QM_ONE: ck_task<T, C, QM_ONE>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
        default: ck_task<T, C, QM_FLOAT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err); break;
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
    const uint64_t want = (uint64_t)num_sms() * 96;
    while (parts < (uint32_t)CK_G && ngroups * parts < want) parts *= 2;
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
