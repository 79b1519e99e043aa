// k_extract.cu -- a1+a8 EXTRACT: uniform error-bounded quantisation (BJ north_star, G-2..G-4) of the
// kept voxels, compacted into a dense code stream in increasing linear index (G-17).
//
// Tiles of 8192 voxels (256 mask words).  Pass 1 counts the kept voxels of every tile (reads K:
// N/8 bytes), a scan turns the counts into output offsets, pass 2 quantises each tile's kept voxels
// into a shared-memory staging buffer and stores them contiguously with 16-byte stores.  (A single
// pass with a decoupled look-back was measured first: with ~1200 tiles in flight the look-back
// walked back hundreds of tiles and serialised the CTAs; the extra N/8-byte read costs far less.)
// x is loaded only for the 16-byte groups of voxels whose mask byte (u16) / nibble (fp32) is
// non-zero, so DRAM reads x only under kept 32-byte sectors.
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"
#include "segment.cuh"

namespace roix {

constexpr int EX_THREADS = 256;
constexpr int EX_WORDS = 256;            // mask words per tile
constexpr int EX_TILE = EX_WORDS * 32;   // voxels per tile

struct ExWS {
    uint32_t *tcount;   // [ntiles]: per-tile counts
    uint64_t *toff;     // [ntiles + 1]: exclusive offsets (scan output; totals exceed 2^32 at C3-C5)
    uint64_t *scan_tmp; // scan workspace
    uint32_t *err_snap;
};

static size_t ex_carve(void *base, uint64_t n, ExWS *w) {
    uint64_t ntiles = (n + EX_TILE - 1) / EX_TILE;
    size_t a = (((ntiles + 1) * 4) + 255) & ~(size_t)255;
    size_t a2 = (((ntiles + 1) * 8) + 255) & ~(size_t)255;
    size_t b = ((scan_tmp_elems(ntiles) * 8) + 255) & ~(size_t)255;
    if (w) {
        w->tcount = (uint32_t *)base;
        w->toff = (uint64_t *)((char *)base + a);
        w->scan_tmp = (uint64_t *)((char *)base + a + a2);
        w->err_snap = (uint32_t *)((char *)base + a + a2 + b);
    }
    return a + a2 + b + 256;
}

// pass 1: kept voxels per tile -- one warp per tile (256 words = 32 lanes x 2 x 16-byte loads),
// two tiles in flight per warp; also snapshots the error word for pass 2
__global__ void __launch_bounds__(EX_THREADS) k_extract_count(const uint32_t *__restrict__ K, uint64_t n,
                                                              uint64_t ntiles, ExWS w, const roix_scalars *sc) {
    const uint64_t nwords = (n + 31) / 32;
    if (blockIdx.x == 0 && threadIdx.x == 0) *w.err_snap = sc->err;
    const uint64_t wpg = (uint64_t)gridDim.x * (EX_THREADS / 32);
    const uint32_t lane = lane_id();
    const uint4 *K4 = reinterpret_cast<const uint4 *>(K);
    constexpr int U = 4;   // tiles per warp iteration: their 2 U 16-byte loads are issued together
    for (uint64_t t0 = (uint64_t)blockIdx.x * (EX_THREADS / 32) + (threadIdx.x >> 5); t0 < ntiles; t0 += U * wpg) {
        uint4 v[U][2];
#pragma unroll
        for (int u = 0; u < U; u++)
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint64_t wi = (t0 + u * wpg) * EX_WORDS + (h * 32 + lane) * 4;   // first word of the load
                v[u][h] = (t0 + u * wpg < ntiles && wi + 4 <= nwords) ? __ldcs(K4 + wi / 4) : make_uint4(0, 0, 0, 0);
            }
#pragma unroll
        for (int u = 0; u < U; u++) {
            const uint64_t t = t0 + u * wpg;
            if (t >= ntiles) break;
            uint32_t c = 0;
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const uint64_t wi = t * EX_WORDS + (h * 32 + lane) * 4;
                if (wi + 4 <= nwords) c += __popc(v[u][h].x) + __popc(v[u][h].y) + __popc(v[u][h].z) + __popc(v[u][h].w);
                else
                    for (uint64_t k = wi; k < nwords && k < wi + 4; k++) c += __popc(K[k]);
            }
            c = __reduce_add_sync(FULL, c);
            if (lane == 0) w.tcount[t] = c;
        }
    }
}

// ------------------------------------------------------------- segment tiles (the default pass 2)
// Per tile of 8192 voxels (one CTA, thread t <-> mask word t): the kept voxels form a few segments
// (pieces of x-runs).  Their starts / ends come from the mask words (bit tricks, carries between words
// through the warp and through shared memory), two block scans give each segment its voxel range and
// its output offset in the tile; then the threads walk the tile's output in 16-byte-aligned groups of
// V codes, find each group's segment by binary search in shared memory, and copy-quantise it with one
// or two 16-byte loads of x and one 16-byte store -- work proportional to the kept voxels, no divergent
// per-word paths.  Groups across a segment boundary (and the ragged ends) go element by element.
constexpr int ES_MAXSEG = EX_TILE / 2;   // alternating bits: at most 4096 segments in a tile

__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t *wsum, uint32_t &total) {
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t incl = warp_incl_scan(v);
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int k = 0; k < EX_THREADS / 32; k++) {
        const uint32_t t = wsum[k];
        if (k < (int)warp) pre += t;
        tot += t;
    }
    __syncthreads();
    total = tot;
    return pre + incl - v;
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void extract_seg_tile(const T *__restrict__ x, uint64_t n, const uint32_t *__restrict__ K,
                                                 const ExWS &w, roix_scalars *sc, C *__restrict__ out,
                                                 uint64_t capacity, const uint64_t *offset, uint16_t *s_start,
                                                 uint16_t *s_end, uint16_t *s_off, uint32_t *s_edge, uint32_t *wsum) {
    constexpr int V = gr_v<T>();
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    const uint64_t tile = blockIdx.x;
    const uint64_t t0 = w.toff[tile], cnt = w.toff[tile + 1] - t0;
    if (cnt == 0) return;   // empty tile (background)
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t wi = tile * EX_WORDS + tid;
    uint32_t word = wi < nwords ? K[wi] : 0u;
    if (wi == nwords - 1 && (n & 31)) word &= low_mask((uint32_t)(n & 31));   // pad bits
    // neighbouring words' edge bits (tile edges count as background)
    if (lane == 0) s_edge[warp] = word;              // first word of each warp
    if (lane == 31) s_edge[8 + warp] = word;         // last word of each warp
    __syncthreads();
    uint32_t prev = __shfl_up_sync(FULL, word, 1), next = __shfl_down_sync(FULL, word, 1);
    if (lane == 0) prev = warp ? s_edge[8 + warp - 1] : 0u;
    if (lane == 31) next = warp < EX_THREADS / 32 - 1 ? s_edge[warp + 1] : 0u;
    const uint32_t st = word & ~((word << 1) | (prev >> 31));
    const uint32_t en = word & ~((word >> 1) | (next << 31));
    uint32_t nseg;
    const uint32_t both = block_excl_scan(__popc(st) | (__popc(en) << 16), wsum, nseg);
    nseg &= 0xffffu;
    {
        uint32_t ps = both & 0xffffu, pe = both >> 16, m = st;
        while (m) {
            const uint32_t b = __ffs(m) - 1;
            m &= m - 1;
            s_start[ps++] = (uint16_t)(32 * tid + b);
        }
        m = en;
        while (m) {
            const uint32_t b = __ffs(m) - 1;
            m &= m - 1;
            s_end[pe++] = (uint16_t)(32 * tid + b + 1);
        }
    }
    __syncthreads();
    // output offsets of the segments: thread t sums a contiguous chunk of them
    const uint32_t per = (nseg + EX_THREADS - 1) / EX_THREADS;
    const uint32_t k0 = min(nseg, tid * per), k1 = min(nseg, k0 + per);
    uint32_t loc = 0;
    for (uint32_t k = k0; k < k1; k++) loc += s_end[k] - s_start[k];
    uint32_t tot;
    uint32_t run = block_excl_scan(loc, wsum, tot);
    for (uint32_t k = k0; k < k1; k++) {
        s_off[k] = (uint16_t)run;
        run += s_end[k] - s_start[k];
    }
    if (tid == 0) s_off[nseg] = (uint16_t)tot;   // == cnt (<= 8192: fits 16 bits? 8192 does)
    __syncthreads();
    // output groups, aligned in the global stream
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t base = (offset ? *offset : 0) + t0;
    if (tid == 0 && base + cnt > capacity) err |= ROIX_ERR_CAPACITY;
    const int64_t jg0 = -(int64_t)(base % V);   // group g covers tile outputs [jg0 + g V, jg0 + g V + V)
    const uint64_t ngroups = (uint64_t)((int64_t)cnt - jg0 + V - 1) / V;
    const T *xt = x + tile * (uint64_t)EX_TILE;
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const uint64_t vt0 = tile * (uint64_t)EX_TILE;   // first voxel of the tile
    for (uint64_t g = tid; g < ngroups; g += EX_THREADS) {
        const int64_t jg = jg0 + (int64_t)(g * V);
        const uint32_t jl = (uint32_t)max(jg, (int64_t)0);
        int lo = 0, hi = (int)nseg;   // segment of output jl: the largest k with s_off[k] <= jl
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (s_off[mid] <= jl) lo = mid;
            else hi = mid;
        }
        const uint32_t k = lo;
        const uint64_t p = base + (uint64_t)jg;   // output position of the group's first slot
        const bool whole = jg >= 0 && (uint64_t)jg + V <= cnt && s_off[k + 1] >= (uint32_t)jg + V;
        if (whole) {
            const uint64_t v = vt0 + s_start[k] + ((uint32_t)jg - s_off[k]);   // voxel of the group's first code
            const uint32_t kk = (uint32_t)(v % V);
            const uint4 b0 = __ldcs(x4 + v / V);
            const uint4 b1 = kk ? __ldcs(x4 + v / V + 1) : b0;
            const uint4 cv = code_group<T, QM>(window16<T>(b0, b1, kk), q, err);
            if (p + V <= capacity) {
                __stcs(reinterpret_cast<uint4 *>(out + p), cv);
            } else {
                const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                for (int e = 0; e < V; e++)
                    if (p + e < capacity) out[p + e] = (C)(sizeof(C) == 2 ? (cw[e >> 1] >> ((e & 1) * 16)) & 0xffffu : cw[e]);
            }
        } else {
            // a group across segment boundaries (or a ragged end): find every element's voxel first,
            // then issue the V loads together
            uint32_t ks = k, src[V];
            bool ok[V];
#pragma unroll
            for (int e = 0; e < V; e++) {
                const int64_t j = jg + e;
                ok[e] = j >= 0 && (uint64_t)j < cnt;
                src[e] = 0;
                if (ok[e]) {
                    while (s_off[ks + 1] <= (uint32_t)j) ks++;
                    src[e] = s_start[ks] + ((uint32_t)j - s_off[ks]);
                }
            }
            T v[V];
#pragma unroll
            for (int e = 0; e < V; e++) v[e] = ok[e] ? xt[src[e]] : (T)0;
#pragma unroll
            for (int e = 0; e < V; e++)
                if (ok[e] && p + e < capacity) out[p + e] = (C)code1<T, QM>(v[e], q, err);
        }
    }
    if (err) set_err(sc, err);
}

template <typename T, typename C>
__global__ void __launch_bounds__(EX_THREADS) k_extract_seg(const T *__restrict__ x, uint64_t n, uint64_t ntiles,
                                                            const uint32_t *__restrict__ K, ExWS w, roix_scalars *sc,
                                                            C *__restrict__ out, uint64_t capacity,
                                                            const uint64_t *offset) {
    __shared__ uint16_t s_start[ES_MAXSEG], s_end[ES_MAXSEG], s_off[ES_MAXSEG + 1];
    __shared__ uint32_t s_edge[16], wsum[EX_THREADS / 32];
    if (*w.err_snap) return;
    const QP q = load_qp(sc);
    if constexpr (sizeof(T) == 4) {
        extract_seg_tile<T, C, QM_FLOAT>(x, n, K, w, sc, out, capacity, offset, s_start, s_end, s_off, s_edge, wsum);
    } else {
        switch (qmode(q)) {
        case QM_POW2: extract_seg_tile<T, C, QM_POW2>(x, n, K, w, sc, out, capacity, offset, s_start, s_end, s_off, s_edge, wsum); break;
        case QM_INT: extract_seg_tile<T, C, QM_INT>(x, n, K, w, sc, out, capacity, offset, s_start, s_end, s_off, s_edge, wsum); break;
        case QM_ONE: extract_seg_tile<T, C, QM_ONE>(x, n, K, w, sc, out, capacity, offset, s_start, s_end, s_off, s_edge, wsum); break;
        default: extract_seg_tile<T, C, QM_FLOAT>(x, n, K, w, sc, out, capacity, offset, s_start, s_end, s_off, s_edge, wsum); break;
        }
    }
}

// count: total kept voxels (scan total) added to sc->count
__global__ void k_extract_total(const uint64_t *total, const ExWS w, roix_scalars *sc) {
    if (*w.err_snap == 0) sc->count += *total;
}

}  // namespace roix

using namespace roix;

size_t compact_workspace_bytes(uint64_t n);
cudaError_t launch_compact(const void *x, int dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                           void *codes, uint64_t capacity, const uint64_t *offset, void *ws, cudaStream_t st);

size_t extract_workspace_bytes(uint64_t n) {
    const size_t a = ex_carve(nullptr, n, nullptr), b = compact_workspace_bytes(n);
    return a > b ? a : b;
}

cudaError_t launch_extract(const void *x, int dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                           void *codes, uint64_t capacity, const uint64_t *offset, void *ws, cudaStream_t st) {
    // u16: per-chunk warps (k_compact.cu); fp32: the segment tiles below (C2: 0.15 vs 0.36 ms)
    if (dtype == ROIX_U16) return launch_compact(x, dtype, n, keep_bits, sc, codes, capacity, offset, ws, st);
    ExWS w;
    ex_carve(ws, n, &w);
    const uint64_t ntiles = (n + EX_TILE - 1) / EX_TILE;
    if (ntiles > 0x7fffffffull) return cudaErrorInvalidValue;
    uint64_t cg = (uint64_t)num_sms() * 8, need = (ntiles + 15) / 16;
    k_extract_count<<<(unsigned)(need < cg ? (need ? need : 1) : cg), EX_THREADS, 0, st>>>(keep_bits, n, ntiles, w, sc);
    cudaError_t e = scan_u32_u64(w.tcount, w.toff, ntiles, w.scan_tmp, st);
    if (e != cudaSuccess) return e;
    k_extract_seg<float, int32_t><<<(unsigned)ntiles, EX_THREADS, 0, st>>>((const float *)x, n, ntiles, keep_bits, w, sc,
                                                                         (int32_t *)codes, capacity, offset);
    k_extract_total<<<1, 1, 0, st>>>(scan_total_ptr(w.scan_tmp, ntiles), w, sc);
    return cudaGetLastError();
}
