// k_extract.cu -- a1+a8 EXTRACT: uniform error-bounded quantisation (BJ north_star, G-2..G-4) of the
// kept voxels, compacted into a dense code stream in increasing linear index (G-17).
//
// Single pass with a decoupled look-back scan (Merrill & Garland 2016): a CTA takes the next tile of
// 8192 voxels (256 mask words), publishes its count, looks back over its predecessors' published
// aggregates / inclusive prefixes (32 at a time, one warp), then quantises its kept voxels into a
// shared-memory staging buffer and stores the tile's codes contiguously.  x is loaded only for the
// 16-byte groups of voxels whose mask byte (u16) / nibble (fp32) is non-zero, so DRAM reads x only
// under kept 32-byte sectors.
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

constexpr int EX_THREADS = 256;
constexpr int EX_WORDS = 256;            // mask words per tile
constexpr int EX_TILE = EX_WORDS * 32;   // voxels per tile
constexpr uint64_t ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_MASK = 3ull << 62, VAL_MASK = ST_AGG - 1;

struct ExWS {
    unsigned long long *flags;  // [ntiles]
    uint32_t *ticket;
    uint32_t *err_snap;
};

static size_t ex_carve(void *base, uint64_t n, ExWS *w) {
    uint64_t ntiles = (n + EX_TILE - 1) / EX_TILE;
    size_t fbytes = ((ntiles * 8) + 255) & ~(size_t)255;
    if (w) {
        w->flags = (unsigned long long *)base;
        w->ticket = (uint32_t *)((char *)base + fbytes);
        w->err_snap = w->ticket + 1;
    }
    return fbytes + 256;
}

__global__ void k_extract_prep(ExWS w, const roix_scalars *sc) {
    *w.ticket = 0;
    *w.err_snap = sc->err;
}

template <typename T, typename C>
__global__ void __launch_bounds__(EX_THREADS) k_extract(const T *__restrict__ x, uint64_t n, uint64_t ntiles,
                                                        const uint32_t *__restrict__ K, ExWS w, roix_scalars *sc,
                                                        C *__restrict__ out, uint64_t capacity, const uint64_t *offset) {
    constexpr int VPL = 16 / sizeof(T);   // voxels per 16-byte group
    constexpr int GPW = 32 / VPL;         // groups per mask word
    constexpr int CHUNKS = 32 / VPL;      // 32-group chunks per warp (a warp covers 32 words = 1024 voxels)
    __shared__ C stage[EX_TILE];
    __shared__ uint32_t warp_tot[EX_THREADS / 32];
    __shared__ uint64_t s_excl;
    __shared__ uint32_t s_tile;
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tile = atomicAdd(w.ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const bool skip = *w.err_snap != 0;
    const uint64_t nwords = (n + 31) / 32;
    const uint64_t wbase = tile * EX_WORDS + warp * 32;
    uint32_t word = 0;
    if (!skip && wbase + lane < nwords) word = K[wbase + lane];
    const uint32_t cnt = __popc(word);
    const uint32_t incl = warp_incl_scan(cnt);
    if (lane == 31) warp_tot[warp] = incl;
    __syncthreads();
    uint32_t wpre = 0, total = 0;
    for (int k = 0; k < EX_THREADS / 32; k++) {
        uint32_t t = warp_tot[k];
        if (k < (int)warp) wpre += t;
        total += t;
    }
    // publish the aggregate, look back, publish the inclusive prefix
    if (warp == 0) {
        uint64_t excl = 0;
        if (tile == 0) {
            if (lane == 0) atomicExch(&w.flags[0], ST_INC | total);
        } else {
            if (lane == 0) atomicExch(&w.flags[tile], ST_AGG | total);
            int64_t p = (int64_t)tile - 1;
            while (true) {
                int64_t idx = p - lane;
                uint64_t f = idx >= 0 ? *((volatile unsigned long long *)&w.flags[idx]) : ST_INC;
                uint32_t inc = __ballot_sync(FULL, (f & ST_MASK) == ST_INC);
                uint32_t zero = __ballot_sync(FULL, (f & ST_MASK) == 0);
                int L = inc ? __ffs(inc) - 1 : 31;
                uint32_t upto = L == 31 ? FULL : ((2u << L) - 1u);
                if (zero & upto) continue;  // a predecessor has not published yet
                uint64_t v = (lane <= (uint32_t)L) ? (f & VAL_MASK) : 0;
#pragma unroll
                for (int d = 16; d > 0; d >>= 1) v += __shfl_xor_sync(FULL, v, d);
                excl += v;
                if (inc) break;
                p -= 32;
            }
            __threadfence();
            if (lane == 0) atomicExch(&w.flags[tile], ST_INC | (excl + total));
        }
        if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    if (skip) return;
    const uint64_t excl = s_excl;
    const uint64_t base = (offset ? *offset : 0) + excl;
    const QP q = load_qp(sc);
    uint32_t err = 0;
    // quantise the kept voxels of this warp's 32 words into stage[wpre ...]
    uint32_t run = wpre;
    const uint64_t gbase = wbase * 32;  // first voxel of the warp
    for (int c = 0; c < CHUNKS; c++) {
        const uint32_t g = c * 32 + lane;                       // group within the warp
        const uint32_t wsrc = g / GPW, sh = (g % GPW) * VPL;
        const uint32_t wv = __shfl_sync(FULL, word, wsrc);
        const uint32_t m = (wv >> sh) & ((1u << VPL) - 1u);
        const uint32_t pc = __popc(m);
        const uint32_t pos = warp_incl_scan(pc) - pc + run;
        run += __shfl_sync(FULL, pos + pc, 31) - run;
        if (m) {
            const uint64_t v0 = gbase + (uint64_t)g * VPL;
            uint32_t p = pos;
            if (v0 + VPL <= n) {
                uint4 d = __ldcs(reinterpret_cast<const uint4 *>(x + v0));
                if constexpr (sizeof(T) == 2) {
                    uint32_t ww[4] = {d.x, d.y, d.z, d.w};
#pragma unroll
                    for (int k = 0; k < 8; k++)
                        if (m >> k & 1) stage[p++] = (C)code_u16((ww[k >> 1] >> ((k & 1) * 16)) & 0xffffu, q, err);
                } else {
                    float ff[4] = {__uint_as_float(d.x), __uint_as_float(d.y), __uint_as_float(d.z), __uint_as_float(d.w)};
#pragma unroll
                    for (int k = 0; k < 4; k++)
                        if (m >> k & 1) stage[p++] = (C)code_f32(ff[k], q, err);
                }
            } else {
                for (int k = 0; k < VPL; k++)
                    if (m >> k & 1) {
                        if constexpr (sizeof(T) == 2) stage[p++] = (C)code_u16(x[v0 + k], q, err);
                        else stage[p++] = (C)code_f32(x[v0 + k], q, err);
                    }
            }
        }
    }
    if (base + total > capacity) err |= ROIX_ERR_CAPACITY;
    if (err) set_err(sc, err);
    __syncthreads();
    const uint64_t lim = base < capacity ? min((uint64_t)total, capacity - base) : 0;
    for (uint64_t j = threadIdx.x; j < lim; j += EX_THREADS) out[base + j] = stage[j];
    if (tile == ntiles - 1 && threadIdx.x == 0) atomicAdd((unsigned long long *)&sc->count, excl + total);
}

}  // namespace roix

using namespace roix;

size_t extract_workspace_bytes(uint64_t n) { return ex_carve(nullptr, n, nullptr); }

cudaError_t launch_extract(const void *x, int dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                           void *codes, uint64_t capacity, const uint64_t *offset, void *ws, cudaStream_t st) {
    ExWS w;
    ex_carve(ws, n, &w);
    const uint64_t ntiles = (n + EX_TILE - 1) / EX_TILE;
    cudaError_t e = cudaMemsetAsync(w.flags, 0, ntiles * 8, st);
    if (e != cudaSuccess) return e;
    k_extract_prep<<<1, 1, 0, st>>>(w, sc);
    if (ntiles > 0x7fffffffull) return cudaErrorInvalidValue;
    if (dtype == ROIX_U16)
        k_extract<uint16_t, uint16_t><<<(unsigned)ntiles, EX_THREADS, 0, st>>>(
            (const uint16_t *)x, n, ntiles, keep_bits, w, sc, (uint16_t *)codes, capacity, offset);
    else
        k_extract<float, int32_t><<<(unsigned)ntiles, EX_THREADS, 0, st>>>((const float *)x, n, ntiles, keep_bits, w, sc,
                                                                          (int32_t *)codes, capacity, offset);
    return cudaGetLastError();
}
