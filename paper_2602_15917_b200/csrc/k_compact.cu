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

// Per-warp shared staging of one chunk: the quantised 16-byte groups in source order, every group's
// mask and output position (chunk-relative), and for every aligned output vector the group holding
// its first code.
template <typename T>
struct CkStage {
    static constexpr int NG = 32 * CkTraits<T>::J;          // groups per chunk
    static constexpr int NV = CK_VOX / CkTraits<T>::VPG + 2; // output vectors per chunk (with the shared ends)
    uint4 codes[NG + 1];
    uint16_t pos[NG + 1];
    uint8_t mask[NG + 1];
    uint8_t vgroup[NV];
};

// elements [sb, sb + V) of the 2V elements (a, b): branch-free (lanes may differ)
template <typename C>
__device__ __forceinline__ uint4 window_el(const uint4 &a, const uint4 &b, uint32_t sb) {
    const uint32_t sh = sb * (uint32_t)(sizeof(C) / 2);   // in halfwords, 0..7
    const uint32_t W[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    const uint32_t f = (sh & 1u) * 16u;
    uint32_t Vv[7];
#pragma unroll
    for (int i = 0; i < 7; i++) Vv[i] = __funnelshift_r(W[i], W[i + 1], f);
    const uint32_t s = sh >> 1;
    uint32_t o[4];
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const uint32_t t = (s & 1u) ? Vv[k + 1] : Vv[k];
        const uint32_t u = (s & 1u) ? Vv[k + 3] : Vv[k + 2];
        o[k] = (s & 2u) ? u : t;
    }
    return make_uint4(o[0], o[1], o[2], o[3]);
}

// position of the (r+1)-th set bit of an 8-bit mask (r < popc(m))
__device__ __forceinline__ uint32_t sel8(uint32_t m, uint32_t r) {
    for (uint32_t i = 0; i < r; i++) m &= m - 1;
    return __ffs(m) - 1;
}

// Output-driven chunk: (A) the lane's groups are quantised and staged in shared memory with their
// masks and positions, and every aligned output vector learns which group holds its first code;
// (B) lane i writes output vectors i, i+32, ...: a vector whose 8 (fp32: 4) codes come from
// consecutive kept voxels is one 16-byte window of the staged codes and one 16-byte store; (C) the
// rest -- vectors across a run end, the two vectors the chunk shares with its neighbours, the
// capacity edge -- are written code by code, eight lanes per vector.
template <typename T, typename C, int QM, int J>
__device__ __forceinline__ void ck_chunk(const uint32_t (&mb)[J], uint4 (&e)[J], uint64_t cbase, uint32_t ccount,
                                         C *__restrict__ out, uint64_t capacity, const QP &q, uint32_t &err,
                                         CkStage<T> &S) {
    constexpr int V = CkTraits<T>::VPG;   // codes per 16-byte vector = voxels per 16-byte group
    constexpr int NG = CkStage<T>::NG;
    constexpr uint32_t GM = (1u << V) - 1u;
    const uint32_t lane = lane_id();
    if (cbase + ccount > capacity) err |= ROIX_ERR_CAPACITY;
    const uint32_t d0 = (uint32_t)(cbase % V);
    const uint64_t ab = cbase - d0;
    C *ob = out + ab;
    const uint32_t caprel = capacity <= ab ? 0u : (uint32_t)min(capacity - ab, (uint64_t)0xffff0000u);
    // (A) positions (two slots per scan word: 16-bit fields), staging, vector -> group table
    uint32_t run = 0;
#pragma unroll
    for (int j = 0; j < J; j += 2) {
        const uint32_t c0 = __popc(mb[j]), c1 = __popc(mb[j + 1]);
        const uint32_t inc = warp_incl_scan(c0 | (c1 << 16));
        const uint32_t tot = __shfl_sync(FULL, inc, 31);
        const uint32_t p0 = run + (inc & 0xffffu) - c0;
        run += tot & 0xffffu;
        const uint32_t p1 = run + (inc >> 16) - c1;
        run += tot >> 16;
        const uint32_t pp[2] = {p0, p1}, cc[2] = {c0, c1};
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int jj = j + h;
            const uint32_t g = 32 * jj + lane;
            S.pos[g] = (uint16_t)pp[h];
            S.mask[g] = (uint8_t)mb[jj];
            if (mb[jj]) {
                S.codes[g] = quant16<T, QM>(e[jj], q, err);
                // vectors whose first code (position V v - d0) is one of this group's codes
                const uint32_t lo = pp[h] + d0, hi = pp[h] + cc[h] + d0;   // [lo, hi) in vector-space codes
                for (uint32_t v = (lo + V - 1) / V; v * V < hi; v++) S.vgroup[v] = (uint8_t)g;
            }
        }
    }
    if (lane == 0) {
        S.pos[NG] = (uint16_t)ccount;
        S.mask[NG] = 0;
    }
    __syncwarp();
    // (B) the vectors of this chunk: [0, nv) in vector space; vector v holds codes V v - d0 ..
    const uint32_t nv = (d0 + ccount + V - 1) / V;
    uint32_t slow_bits = 0;   // per 32-vector round: this lane's vector goes element by element
    for (uint32_t t = 0; t * 32 < nv; t++) {
        const uint32_t v = 32 * t + lane;
        bool slow = false;
        if (v < nv) {
            const int32_t s0 = (int32_t)(V * v) - (int32_t)d0;   // chunk code index of the first code
            bool fast = s0 >= 0 && (uint32_t)s0 + V <= ccount && V * v + V <= caprel;
            if (fast) {
                const uint32_t g = S.vgroup[v];
                const uint32_t r = (uint32_t)s0 - S.pos[g];
                const uint32_t m = S.mask[g];
                const uint32_t sb = m == GM ? r : sel8(m, r);
                const uint32_t win = ((m | ((uint32_t)S.mask[g + 1] << V)) >> sb) & GM;
                if (win == GM) {
                    const uint4 a = S.codes[g];
                    const uint4 b = sb ? S.codes[g + 1] : a;
                    __stcs(reinterpret_cast<uint4 *>(ob + V * v), sb ? window_el<C>(a, b, sb) : a);
                } else {
                    fast = false;
                }
            }
            slow = !fast;
        }
        slow_bits |= (uint32_t)(__ballot_sync(FULL, slow) != 0) << t;
    }
    // (C) slow vectors, eight (fp32: four) lanes per vector, one code each
    constexpr int LPV = V;                 // lanes per vector
    constexpr int VPR = 32 / LPV;          // vectors per round
    for (uint32_t t = 0; t * 32 < nv; t++) {
        if (!((slow_bits >> t) & 1u)) continue;
        // recompute which vectors of round t are slow (same predicate as above)
        const uint32_t v = 32 * t + lane;
        bool slow = false;
        if (v < nv) {
            const int32_t s0 = (int32_t)(V * v) - (int32_t)d0;
            bool fast = s0 >= 0 && (uint32_t)s0 + V <= ccount && V * v + V <= caprel;
            if (fast) {
                const uint32_t g = S.vgroup[v];
                const uint32_t r = (uint32_t)s0 - S.pos[g];
                const uint32_t m = S.mask[g];
                const uint32_t sb = m == GM ? r : sel8(m, r);
                fast = (((m | ((uint32_t)S.mask[g + 1] << V)) >> sb) & GM) == GM;
            }
            slow = !fast;
        }
        uint32_t sm = __ballot_sync(FULL, slow);
        while (sm) {
            // up to VPR slow vectors per pass: sub-lane h of slot k handles code h of vector k
            const uint32_t k = lane / LPV, h = lane % LPV;
            uint32_t pick = sm;
            for (uint32_t i = 0; i < k && pick; i++) pick &= pick - 1;
            const bool has = pick != 0;
            const uint32_t vv = has ? 32 * t + (__ffs(pick) - 1) : 0u;
            for (uint32_t i = 0; i < VPR && sm; i++) sm &= sm - 1;
            if (!has) continue;
            const int32_t c = (int32_t)(V * vv + h) - (int32_t)d0;   // chunk code index
            if (c < 0 || (uint32_t)c >= ccount || V * vv + h >= caprel) continue;
            // the group holding code c: the last group with pos <= c (binary search over NG + 1)
            uint32_t lo = 0, hi = NG;
#pragma unroll
            for (int it = 0; it < 9; it++) {
                if (hi - lo <= 1) break;
                const uint32_t mid = (lo + hi) >> 1;
                if (S.pos[mid] <= (uint32_t)c) lo = mid;
                else hi = mid;
            }
            const uint32_t m = S.mask[lo];
            const uint32_t sb = sel8(m, (uint32_t)c - S.pos[lo]);
            const uint4 cv = S.codes[lo];
            ob[V * vv + h] = (C)code_at<C>(cv, sb);
        }
    }
    __syncwarp();   // the staging is rewritten by the next chunk
}

// one warp task: chunks [part * cpp, (part + 1) * cpp) of group g, non-empty ones only; the next
// chunk's x (u16: double-buffered) and the one after's K word are in flight while a chunk is processed
template <typename T, typename C, int QM>
__device__ __forceinline__ void ck_task(const T *__restrict__ x, uint64_t n, const uint32_t *__restrict__ K,
                                        uint64_t nchunks, const CkWS &w, uint64_t g, uint32_t part, uint32_t cpp,
                                        uint64_t off0, C *__restrict__ out, uint64_t capacity, const QP &q,
                                        uint32_t &err, CkStage<T> &S) {
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
        ck_chunk<T, C, QM, J>(mb, e, cbase, ccount, out, capacity, q, err, S);
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
    __shared__ CkStage<T> stage[CK_THREADS / 32];
    if (*w.err_snap) return;
    const uint64_t t = (uint64_t)blockIdx.x * (CK_THREADS / 32) + (threadIdx.x >> 5);
    const uint64_t g = t / parts;
    if (g >= ngroups) return;
    CkStage<T> &S = stage[threadIdx.x >> 5];
    const uint32_t part = (uint32_t)(t % parts), cpp = CK_G / parts;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t off0 = offset ? *offset : 0ull;
    if constexpr (sizeof(T) == 4) {
        ck_task<T, C, QM_FLOAT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err, S);
    } else {
        switch (qmode(q)) {   // uniform over the launch: one quantiser body per mode
        case QM_POW2: ck_task<T, C, QM_POW2>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err, S); break;
        case QM_INT: ck_task<T, C, QM_INT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err, S); break;
        case QM_ONE: ck_task<T, C, QM_ONE>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err, S); break;
        default: ck_task<T, C, QM_FLOAT>(x, n, K, nchunks, w, g, part, cpp, off0, out, capacity, q, err, S); break;
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
