// k_decode.cu -- NEXT-4: reconstruction ("each row is precisely restored using the preserved
// metadata") and the confusion counts behind the ROI quality metrics.
//
// Decoded value of a code (the inverse of a1, reading G-37), s = fl32(2 eb) from roix_scalars:
//   uint16 input  x^ = min(65535, RNE(code * s)) -- an integer product when s is an integer, else the
//                 binary64 product (exact: 16-bit code x 24-bit s) rounded half to even
//   fp32 input    x^ = fl32(fl32(code) * s) -- one correctly rounded fp32 multiply (fl32(code) = code
//                 for every code the quantiser produces, |code| <= 2^23)
//
//   k_dec_count     kept voxels per 8192-voxel tile of K (one warp per tile)            \  mask form:
//   scan            tile offsets into the dense code stream                               > roix_decode
//   k_dec_mask      per tile: word ranks by a block scan, the tile's codes staged in      /
//                   shared memory with 16-byte loads, every voxel written once (16-byte stores)
//   k_span_map      span records -> per-row (x_start, length), checking the format         \  span form:
//   scan            per-row section offsets                                                 > roix_decode_spans
//   k_span_decode   one warp per row: the whole row, zero outside [x_start, x_end)         /
//   k_conf          tp / fp / fn by popcount of the packed masks, tn = n - the rest         roix_confusion
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace roix {

constexpr int DC_T = 256;                // threads per CTA
constexpr int DC_WORDS = 256;            // mask words per tile
constexpr int DC_TILE = DC_WORDS * 32;   // voxels per tile

__device__ __forceinline__ uint16_t dec_u16(uint32_t c, uint32_t s_int, double s) {
    if (s_int) {
        const uint64_t v = (uint64_t)c * s_int;
        return (uint16_t)(v > 65535u ? 65535u : v);
    }
    const double v = rint((double)c * s);
    return (uint16_t)(v > 65535.0 ? 65535.0 : v);
}
__device__ __forceinline__ float dec_f32(int32_t c, float s) { return __fmul_rn(__int2float_rn(c), s); }

template <typename T, typename C>
struct Decoder;
template <>
struct Decoder<uint16_t, uint16_t> {
    uint32_t s_int;
    double s;
    __device__ explicit Decoder(const roix_scalars *sc) : s_int(sc->s_int), s((double)sc->s) {}
    __device__ __forceinline__ uint16_t operator()(uint16_t c) const { return dec_u16(c, s_int, s); }
};
template <>
struct Decoder<float, int32_t> {
    float s;
    __device__ explicit Decoder(const roix_scalars *sc) : s(sc->s) {}
    __device__ __forceinline__ float operator()(int32_t c) const { return dec_f32(c, s); }
};

// V consecutive outputs as one 16-byte store (streaming: the volume is not re-read)
template <typename T, int V>
__device__ __forceinline__ void store16(T *p, const T (&v)[V]) {
    static_assert(sizeof(T) * V == 16, "16-byte groups");
    uint4 u;
    memcpy(&u, v, 16);
    __stcs(reinterpret_cast<uint4 *>(p), u);
}

// ------------------------------------------------------------------------------------ mask form
struct DcWS {
    uint32_t *tcount;    // [ntiles]
    uint64_t *toff;      // [ntiles + 1]
    uint64_t *scan_tmp;
};

static size_t dc_carve(void *base, uint64_t n, DcWS *w) {
    const uint64_t ntiles = (n + DC_TILE - 1) / DC_TILE;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_c = take((ntiles + 1) * 4), o_o = take((ntiles + 1) * 8), o_t = take(scan_tmp_elems(ntiles) * 8);
    if (w) {
        char *b = (char *)base;
        w->tcount = (uint32_t *)(b + o_c);
        w->toff = (uint64_t *)(b + o_o);
        w->scan_tmp = (uint64_t *)(b + o_t);
    }
    return off;
}

// word wi of K with the pad bits past n cleared (G-16 says they are 0; a decoder does not rely on it)
__device__ __forceinline__ uint32_t kword(uint32_t v, uint64_t wi, uint64_t n) {
    const uint64_t rem = n - 32 * wi;
    return rem < 32 ? v & low_mask((uint32_t)rem) : v;
}

__global__ void __launch_bounds__(DC_T) k_dec_count(const uint32_t *__restrict__ K, uint64_t n, uint64_t ntiles,
                                                    uint32_t *tcount, const roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t nwords = (n + 31) / 32;
    const uint32_t lane = lane_id();
    const uint64_t wpg = (uint64_t)gridDim.x * (DC_T / 32);
    for (uint64_t t = (uint64_t)blockIdx.x * (DC_T / 32) + (threadIdx.x >> 5); t < ntiles; t += wpg) {
        uint32_t c = 0;
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const uint64_t wi = t * DC_WORDS + (h * 32 + lane) * 4;   // first word of this lane's 16 bytes
            if (wi + 4 <= nwords) {
                const uint4 v = __ldcs(reinterpret_cast<const uint4 *>(K + wi));
                c += __popc(kword(v.x, wi, n)) + __popc(kword(v.y, wi + 1, n)) + __popc(kword(v.z, wi + 2, n)) +
                     __popc(kword(v.w, wi + 3, n));
            } else {
                for (uint64_t j = wi; j < nwords && j < wi + 4; j++) c += __popc(kword(K[j], j, n));
            }
        }
        c = __reduce_add_sync(FULL, c);
        if (lane == 0) tcount[t] = c;
    }
}

// One tile per CTA iteration.  Thread t owns word t of the tile (its rank among the tile's kept
// voxels from a block scan); the tile's codes [toff[t], toff[t+1]) are staged in shared memory with
// aligned 16-byte loads; then every 16-byte group of outputs is assembled from its mask bits and the
// staged codes and stored once.
template <typename T, typename C>
__global__ void __launch_bounds__(DC_T) k_dec_mask(const uint32_t *__restrict__ K, uint64_t n, uint64_t ntiles,
                                                   const C *__restrict__ codes, uint64_t ncodes,
                                                   const uint64_t *__restrict__ toff, roix_scalars *sc,
                                                   T *__restrict__ xhat) {
    constexpr int V = 16 / sizeof(T);    // outputs per 16-byte store: u16 8, f32 4
    constexpr int CV = 16 / sizeof(C);   // codes per 16-byte load
    __shared__ uint32_t s_word[DC_WORDS], s_woff[DC_WORDS], s_wsum[DC_T / 32];
    __shared__ __align__(16) C s_code[DC_TILE + 2 * CV];
    if (get_err(sc)) return;
    if (toff[ntiles] > ncodes) {   // every CTA takes the same decision: nothing is written
        if (blockIdx.x == 0 && threadIdx.x == 0) set_err(sc, ROIX_ERR_CAPACITY);
        return;
    }
    const Decoder<T, C> dec(sc);
    const uint64_t nwords = (n + 31) / 32;
    const uint32_t tid = threadIdx.x, lane = lane_id(), warp = tid >> 5;
    for (uint64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const uint64_t wi = t * DC_WORDS + tid;
        const uint32_t word = wi < nwords ? kword(__ldcs(K + wi), wi, n) : 0u;
        const uint32_t inc = warp_incl_scan(__popc(word));
        if (lane == 31) s_wsum[warp] = inc;
        const uint64_t base = toff[t];
        const uint32_t cnt = (uint32_t)(toff[t + 1] - base);
        __syncthreads();
        uint32_t wbase = 0;
#pragma unroll
        for (int k = 0; k < DC_T / 32; k++) wbase += k < (int)warp ? s_wsum[k] : 0u;
        const uint32_t sh = (uint32_t)(base % CV);   // staged code j of the tile sits at s_code[sh + j]
        s_word[tid] = word;
        s_woff[tid] = wbase + inc - __popc(word) + sh;
        {
            const uint64_t a0 = base - sh;
            const uint32_t nch = (sh + cnt + CV - 1) / CV;
            for (uint32_t k = tid; k < nch; k += DC_T) {
                const uint64_t g = a0 + (uint64_t)k * CV;
                if (g + CV <= ncodes) {
                    *reinterpret_cast<uint4 *>(&s_code[k * CV]) = __ldcs(reinterpret_cast<const uint4 *>(codes + g));
                } else {
                    for (int j = 0; j < CV; j++)
                        if (g + j < ncodes) s_code[k * CV + j] = codes[g + j];
                }
            }
        }
        __syncthreads();
        const uint64_t t0 = t * DC_TILE;
        for (uint32_t gi = tid; gi < DC_TILE / V; gi += DC_T) {
            const uint64_t i0 = t0 + (uint64_t)gi * V;
            if (i0 >= n) break;
            const uint32_t w = gi * V / 32, sub = gi * V % 32;
            const uint32_t wd = s_word[w];
            const uint32_t bits = (wd >> sub) & low_mask(V);
            uint32_t r = s_woff[w] + __popc(wd & low_mask(sub));
            T v[V];
#pragma unroll
            for (int j = 0; j < V; j++) v[j] = (bits >> j) & 1u ? dec(s_code[r++]) : (T)0;
            if (i0 + V <= n) {
                store16<T, V>(xhat + i0, v);
            } else {
                for (int j = 0; j < V && i0 + j < n; j++) xhat[i0 + j] = v[j];
            }
        }
        __syncthreads();   // the next tile reuses the shared buffers
    }
}

// ------------------------------------------------------------------------------------ span form
struct SdWS {
    uint32_t *rlen, *rstart;   // [rows]
    uint64_t *roff;            // [rows + 1]
    uint64_t *scan_tmp;
};

static size_t sd_carve(void *base, uint64_t rows, SdWS *w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_l = take(rows * 4), o_s = take(rows * 4), o_o = take((rows + 1) * 8),
                 o_t = take(scan_tmp_elems(rows) * 8);
    if (w) {
        char *b = (char *)base;
        w->rlen = (uint32_t *)(b + o_l);
        w->rstart = (uint32_t *)(b + o_s);
        w->roff = (uint64_t *)(b + o_o);
        w->scan_tmp = (uint64_t *)(b + o_t);
    }
    return off;
}

// Record k -> its row: the format of roix_row_spans (rows strictly increasing, inside the slab,
// 0 <= x_start < x_end <= X) is checked here; a violation sets ROIX_ERR_FORMAT and nothing is decoded.
__global__ void __launch_bounds__(256) k_span_map(const roix_span *__restrict__ spans, const uint64_t *counts,
                                                  uint64_t span_cap, uint64_t rows, uint64_t X, uint64_t row0,
                                                  SdWS w, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t m = counts[0];
    if (m > span_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_err(sc, ROIX_ERR_CAPACITY);
        return;
    }
    bool bad = false;
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (uint64_t)gridDim.x * blockDim.x) {
        const roix_span sp = spans[k];
        const bool ok = sp.row >= row0 && sp.row - row0 < rows && sp.x_start < sp.x_end && sp.x_end <= X &&
                        (k == 0 || spans[k - 1].row < sp.row);
        if (!ok) {
            bad = true;
            continue;
        }
        w.rlen[sp.row - row0] = sp.x_end - sp.x_start;
        w.rstart[sp.row - row0] = sp.x_start;
    }
    if (bad) set_err(sc, ROIX_ERR_FORMAT);
}

template <typename T, typename C>
__global__ void __launch_bounds__(256) k_span_decode(const C *__restrict__ codes, const uint64_t *counts,
                                                     uint64_t code_cap, uint64_t rows, uint64_t X, SdWS w,
                                                     roix_scalars *sc, T *__restrict__ xhat) {
    constexpr int V = 16 / sizeof(T);
    if (get_err(sc)) return;
    const uint64_t total = w.roff[rows];
    if (total > code_cap || total != counts[1]) {   // same decision in every CTA
        if (blockIdx.x == 0 && threadIdx.x == 0) set_err(sc, total > code_cap ? ROIX_ERR_CAPACITY : ROIX_ERR_FORMAT);
        return;
    }
    const Decoder<T, C> dec(sc);
    const uint32_t lane = lane_id();
    const uint64_t wpg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += wpg) {
        const uint32_t len = w.rlen[r];
        const uint32_t xs = len ? w.rstart[r] : 0u, xe = xs + len;
        const C *src = codes + w.roff[r] - xs;   // code of column x (xs <= x < xe): src[x]
        T *row = xhat + r * X;
        auto val = [&](uint64_t x) -> T { return x >= xs && x < xe ? dec(src[x]) : (T)0; };
        // head up to 16-byte alignment, 16-byte body, tail
        const uint64_t mis = (uint64_t)(reinterpret_cast<uintptr_t>(row) / sizeof(T)) % V;
        const uint64_t head = min(X, mis ? (uint64_t)V - mis : (uint64_t)0);
        if (lane < head) row[lane] = val(lane);
        const uint64_t nb = (X - head) / V;
        for (uint64_t b = lane; b < nb; b += 32) {
            const uint64_t x0 = head + b * V;
            T v[V];
            if (x0 >= xe || x0 + V <= xs) {
#pragma unroll
                for (int j = 0; j < V; j++) v[j] = (T)0;
            } else {
#pragma unroll
                for (int j = 0; j < V; j++) v[j] = val(x0 + j);
            }
            store16<T, V>(row + x0, v);
        }
        const uint64_t x1 = head + nb * V;
        if (x1 + lane < X) row[x1 + lane] = val(x1 + lane);
    }
}

// ------------------------------------------------------------------------------------ confusion
__global__ void k_conf_init(uint64_t *c, uint64_t n) {
    c[0] = c[1] = c[2] = 0;
    c[3] = n;
}

__global__ void __launch_bounds__(256) k_conf(const uint32_t *__restrict__ P, const uint32_t *__restrict__ G, uint64_t n,
                                              uint64_t *c) {
    __shared__ unsigned long long s[3][8];
    const uint64_t nfull = n / 32;          // words with no pad bits
    const uint64_t nvec = nfull / 4;        // 16-byte chunks of them
    uint64_t tp = 0, fp = 0, fn = 0;
    const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
    for (uint64_t k = tid; k < nvec; k += nt) {
        const uint4 p = __ldcs(reinterpret_cast<const uint4 *>(P) + k);
        const uint4 g = __ldcs(reinterpret_cast<const uint4 *>(G) + k);
        tp += __popc(p.x & g.x) + __popc(p.y & g.y) + __popc(p.z & g.z) + __popc(p.w & g.w);
        fp += __popc(p.x & ~g.x) + __popc(p.y & ~g.y) + __popc(p.z & ~g.z) + __popc(p.w & ~g.w);
        fn += __popc(~p.x & g.x) + __popc(~p.y & g.y) + __popc(~p.z & g.z) + __popc(~p.w & g.w);
    }
    // the remaining full words and the partial last word (pad bits masked off)
    for (uint64_t wi = 4 * nvec + tid; wi < (n + 31) / 32; wi += nt) {
        const uint32_t m = wi < nfull ? FULL : low_mask((uint32_t)(n - 32 * wi));
        const uint32_t p = P[wi] & m, g = G[wi] & m;
        tp += __popc(p & g);
        fp += __popc(p & ~g);
        fn += __popc(~p & g & m);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        tp += __shfl_xor_sync(FULL, tp, d);
        fp += __shfl_xor_sync(FULL, fp, d);
        fn += __shfl_xor_sync(FULL, fn, d);
    }
    const uint32_t warp = threadIdx.x >> 5;
    if (lane_id() == 0) {
        s[0][warp] = tp;
        s[1][warp] = fp;
        s[2][warp] = fn;
    }
    __syncthreads();
    if (threadIdx.x < 3) {
        unsigned long long v = 0;
        for (uint32_t k = 0; k < blockDim.x / 32; k++) v += s[threadIdx.x][k];
        if (v) {
            atomicAdd((unsigned long long *)&c[threadIdx.x], v);
            atomicAdd((unsigned long long *)&c[3], 0ull - v);   // tn = n - tp - fp - fn
        }
    }
}

}  // namespace roix

using namespace roix;

size_t decode_workspace_bytes(uint64_t n) { return dc_carve(nullptr, n, nullptr); }

cudaError_t launch_decode(const uint32_t *K, const void *codes, uint64_t ncodes, int dtype, uint64_t n,
                          roix_scalars *sc, void *xhat, void *ws, cudaStream_t st) {
    if (n == 0) return cudaSuccess;
    DcWS w;
    dc_carve(ws, n, &w);
    const uint64_t ntiles = (n + DC_TILE - 1) / DC_TILE;
    const unsigned cg = (unsigned)min((ntiles + 7) / 8, (uint64_t)num_sms() * 8);
    k_dec_count<<<cg, DC_T, 0, st>>>(K, n, ntiles, w.tcount, sc);
    cudaError_t e = scan_u32_u64(w.tcount, w.toff, ntiles, w.scan_tmp, st);
    if (e != cudaSuccess) return e;
    const unsigned grid = (unsigned)min(ntiles, (uint64_t)num_sms() * 6);
    if (dtype == ROIX_U16)
        k_dec_mask<uint16_t, uint16_t><<<grid, DC_T, 0, st>>>(K, n, ntiles, (const uint16_t *)codes, ncodes, w.toff, sc,
                                                             (uint16_t *)xhat);
    else
        k_dec_mask<float, int32_t><<<grid, DC_T, 0, st>>>(K, n, ntiles, (const int32_t *)codes, ncodes, w.toff, sc,
                                                         (float *)xhat);
    return cudaGetLastError();
}

size_t decode_spans_workspace_bytes(const roix_geom &g) { return sd_carve(nullptr, g.nz * g.ny, nullptr); }

cudaError_t launch_decode_spans(const roix_span *spans, uint64_t span_cap, const void *codes, uint64_t code_cap,
                                const uint64_t *counts, int dtype, const roix_geom &g, roix_scalars *sc, void *xhat,
                                void *ws, cudaStream_t st) {
    const uint64_t rows = g.nz * g.ny;
    if (rows == 0 || g.nx == 0) return cudaSuccess;
    SdWS w;
    sd_carve(ws, rows, &w);
    cudaError_t e = cudaMemsetAsync(w.rlen, 0, rows * 4, st);
    if (e != cudaSuccess) return e;
    const unsigned mg = (unsigned)min((max(span_cap, (uint64_t)1) + 255) / 256, (uint64_t)num_sms() * 8);
    k_span_map<<<mg, 256, 0, st>>>(spans, counts, span_cap, rows, g.nx, g.z0 * g.ny, w, sc);
    if ((e = scan_u32_u64(w.rlen, w.roff, rows, w.scan_tmp, st)) != cudaSuccess) return e;
    const unsigned grid = (unsigned)min((rows + 7) / 8, (uint64_t)num_sms() * 8);
    if (dtype == ROIX_U16)
        k_span_decode<uint16_t, uint16_t><<<grid, 256, 0, st>>>((const uint16_t *)codes, counts, code_cap, rows, g.nx,
                                                                w, sc, (uint16_t *)xhat);
    else
        k_span_decode<float, int32_t><<<grid, 256, 0, st>>>((const int32_t *)codes, counts, code_cap, rows, g.nx, w,
                                                            sc, (float *)xhat);
    return cudaGetLastError();
}

cudaError_t launch_confusion(const uint32_t *pred, const uint32_t *truth, uint64_t n, uint64_t *counts,
                             cudaStream_t st) {
    k_conf_init<<<1, 1, 0, st>>>(counts, n);
    if (n == 0) return cudaGetLastError();
    const uint64_t nvec = n / 128 + 1;
    const unsigned grid = (unsigned)min((nvec + 255) / 256, (uint64_t)num_sms() * 4);
    k_conf<<<grid, 256, 0, st>>>(pred, truth, n, counts);
    return cudaGetLastError();
}
