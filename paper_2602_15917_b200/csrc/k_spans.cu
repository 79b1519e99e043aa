// k_spans.cu -- NEXT-1: the paper's ROI representation.  For every row
// i = z*Y + y of the kept mask K with a set bit: the geometry record G(i) = [i, x_start, x_end)
// (leftmost set column, rightmost + 1) and the pixel section P(i) = codes of x[i][x_start:x_end],
// interior gaps included, quantised with the a1 quantiser (RNE(x / s), G-2..G-4).
//
//   k_row_extent  one warp per row: the first and last set bit from a min / max reduction over the
//                 row's words (ffs / clz); len[i] = x_end - x_start (0 for an empty row)
//   scans         span index = prefix count of non-empty rows, code offset = prefix of len (uint64)
//   k_span_write  one warp per non-empty row: its record, then its section (warp_segment: 16-byte
//                 loads of x, codes quantised in registers, 16-byte stores)
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"
#include "segment.cuh"

namespace roix {

struct SpanWS {
    uint32_t *start, *len, *nonempty, *sidx;   // [rows], [rows], [rows], [rows + 1]
    uint64_t *coff;                            // [rows + 1]
    uint64_t *tmp_a, *tmp_b;                   // scan workspaces
    uint32_t *err_snap;                        // error bits before k_span_write
};

static size_t span_carve(void *base, uint64_t rows, SpanWS *w) {
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += (bytes + 255) & ~(size_t)255;
        return o;
    };
    const size_t o_st = take(rows * 4), o_ln = take(rows * 4), o_ne = take(rows * 4), o_si = take((rows + 1) * 4);
    const size_t o_co = take((rows + 1) * 8), o_ta = take(scan_tmp_elems(rows) * 8), o_tb = take(scan_tmp_elems(rows) * 8);
    const size_t o_es = take(4);
    if (w) {
        char *b = (char *)base;
        w->start = (uint32_t *)(b + o_st);
        w->len = (uint32_t *)(b + o_ln);
        w->nonempty = (uint32_t *)(b + o_ne);
        w->sidx = (uint32_t *)(b + o_si);
        w->coff = (uint64_t *)(b + o_co);
        w->tmp_a = (uint64_t *)(b + o_ta);
        w->tmp_b = (uint64_t *)(b + o_tb);
        w->err_snap = (uint32_t *)(b + o_es);
    }
    return off;
}

// word k of row r of a linear bit array (pad bits beyond X cleared); never reads past word nwords-1
__device__ __forceinline__ uint32_t span_row_word(const uint32_t *bits, uint64_t X, uint64_t r, uint32_t k,
                                                  uint64_t nwords) {
    const uint64_t b = r * X + 32ull * k;
    const uint32_t sh = (uint32_t)(b & 31);
    const uint64_t wi = b >> 5;
    uint32_t v = bits[wi];
    if (sh) v = __funnelshift_r(v, wi + 1 < nwords ? bits[wi + 1] : 0u, sh);
    const uint64_t rem = X - 32ull * k;
    if (rem < 32) v &= low_mask((uint32_t)rem);
    return v;
}

__global__ void __launch_bounds__(256) k_row_extent(const uint32_t *__restrict__ K, uint64_t rows, uint64_t X,
                                                    SpanWS w, roix_scalars *sc) {
    if (blockIdx.x == 0 && threadIdx.x == 0) *w.err_snap = get_err(sc);
    if (get_err(sc)) return;
    const uint32_t lane = lane_id();
    const uint32_t W = (uint32_t)((X + 31) / 32);
    const uint64_t nwords = (rows * X + 31) / 32;
    const uint64_t wpg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += wpg) {
        uint32_t lo = 0xffffffffu, hi = 0;   // first set column, last set column + 1
        for (uint32_t k0 = 0; k0 < W; k0 += 32) {
            const uint32_t k = k0 + lane;
            const uint32_t v = k < W ? span_row_word(K, X, r, k, nwords) : 0u;
            if (v) {
                lo = min(lo, 32 * k + (uint32_t)(__ffs(v) - 1));
                hi = max(hi, 32 * k + 32 - (uint32_t)__clz(v));
            }
        }
        lo = __reduce_min_sync(FULL, lo);
        hi = __reduce_max_sync(FULL, hi);
        if (lane == 0) {
            const bool ne = hi > 0;
            w.start[r] = ne ? lo : 0;
            w.len[r] = ne ? hi - lo : 0;
            w.nonempty[r] = ne;
        }
    }
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void span_rows(const T *__restrict__ x, uint64_t rows, uint64_t X, uint64_t row0,
                                          const SpanWS &w, roix_scalars *sc, roix_span *spans, uint64_t span_cap,
                                          C *__restrict__ codes, uint64_t code_cap, uint64_t *counts) {
    const uint32_t lane = lane_id();
    const QP q = load_qp(sc);
    uint32_t err = 0;
    const uint64_t wpg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        const uint64_t ns = w.sidx[rows], nc = w.coff[rows];
        counts[0] = ns;
        counts[1] = nc;
        if (ns > span_cap || nc > code_cap) err |= ROIX_ERR_CAPACITY;
    }
    for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += wpg) {
        const uint32_t len = w.len[r];
        if (!len) continue;
        const uint32_t x0 = w.start[r];
        const uint64_t si = w.sidx[r], co = w.coff[r];
        if (lane == 0 && si < span_cap) {
            roix_span sp;
            sp.row = row0 + r;
            sp.x_start = x0;
            sp.x_end = x0 + len;
            spans[si] = sp;
        }
        warp_segment<T, C, QM, 2>(x, r * X + x0, codes, co, len, code_cap, q, err);
    }
    if (err) set_err(sc, err);
}

template <typename T, typename C>
__global__ void __launch_bounds__(256) k_span_write(const T *__restrict__ x, uint64_t rows, uint64_t X, uint64_t row0,
                                                    SpanWS w, roix_scalars *sc, roix_span *spans, uint64_t span_cap,
                                                    C *__restrict__ codes, uint64_t code_cap, uint64_t *counts) {
    if (*w.err_snap) return;   // (not get_err: this kernel's own capacity bit must not stop its other CTAs)
    if constexpr (sizeof(T) == 4) {
        span_rows<T, C, QM_FLOAT>(x, rows, X, row0, w, sc, spans, span_cap, codes, code_cap, counts);
    } else {
        switch (qmode(load_qp(sc))) {
        case QM_POW2: span_rows<T, C, QM_POW2>(x, rows, X, row0, w, sc, spans, span_cap, codes, code_cap, counts); break;
        case QM_INT: span_rows<T, C, QM_INT>(x, rows, X, row0, w, sc, spans, span_cap, codes, code_cap, counts); break;
        case QM_ONE: span_rows<T, C, QM_ONE>(x, rows, X, row0, w, sc, spans, span_cap, codes, code_cap, counts); break;
        default: span_rows<T, C, QM_FLOAT>(x, rows, X, row0, w, sc, spans, span_cap, codes, code_cap, counts); break;
        }
    }
}

}  // namespace roix

using namespace roix;

size_t row_spans_workspace_bytes(const roix_geom &g) { return span_carve(nullptr, g.nz * g.ny, nullptr); }

cudaError_t launch_row_spans(const uint32_t *K, const void *x, int dtype, const roix_geom &g, roix_scalars *sc,
                             roix_span *spans, uint64_t span_cap, void *codes, uint64_t code_cap, uint64_t *counts,
                             void *ws, cudaStream_t st) {
    SpanWS w;
    const uint64_t rows = g.nz * g.ny;
    span_carve(ws, rows, &w);
    const unsigned grid = (unsigned)min((rows + 7) / 8, (uint64_t)num_sms() * 8);
    k_row_extent<<<grid, 256, 0, st>>>(K, rows, g.nx, w, sc);
    cudaError_t e = scan_u32(w.nonempty, w.sidx, rows, w.tmp_a, st);
    if (e != cudaSuccess) return e;
    if ((e = scan_u32_u64(w.len, w.coff, rows, w.tmp_b, st)) != cudaSuccess) return e;
    const uint64_t row0 = g.z0 * g.ny;
    if (dtype == ROIX_U16)
        k_span_write<uint16_t, uint16_t><<<grid, 256, 0, st>>>((const uint16_t *)x, rows, g.nx, row0, w, sc, spans,
                                                               span_cap, (uint16_t *)codes, code_cap, counts);
    else
        k_span_write<float, int32_t><<<grid, 256, 0, st>>>((const float *)x, rows, g.nx, row0, w, sc, spans, span_cap,
                                                           (int32_t *)codes, code_cap, counts);
    return cudaGetLastError();
}
