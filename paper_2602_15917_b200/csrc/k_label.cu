// k_label.cu -- a6 CONNECTED COMPONENTS + a7 FILTER on x-runs of the opened mask o.
//
// A run is a maximal stretch of set bits of o in one row (z, y).  Runs are stored in raster order
// (row, then x), so run index order equals the order of their first voxel's linear index, and a
// union-find that always links the larger index under the smaller one ends with every component's
// root = its first run = the run holding the component's minimum linear index (the canonical label,
// reading G-14).  Steps (one launch each, all on the caller's stream):
//   count   runs per row (skipped when roix_morph already produced them)
//   scan    row_start = exclusive prefix of the counts; n_runs; capacity check
//   runs    (x0, x1, row) of every run: copied from the opening's run records for rows with at most
//           rs runs (roix_morph_slots), extracted from o for the others
//   union   each run links with the overlapping runs of its "previous" neighbour rows, in shared
//           memory per block of 4-16 K runs, the pairs that cross blocks globally (lock-free
//           union-by-min with atomicMin on uint32 parents)
//   flatten parent[i] = root(i)
//   sizes   size[root] += run length (warp-aggregated)
//   table   roots in index order -> (min_index, size, kept = size >= min_size)  (G-13)
//   clear   K = o with the bits of dropped components cleared (in place when K aliases o)
//   labels  optional per-voxel uint64 labels
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"

namespace roix {

struct LabelWS {
    uint32_t *row_runs;   // [rows]
    uint32_t *row_start;  // [rows + 1]
    uint64_t *scan_tmp;   // [scan_tmp_len]
    uint32_t *x0, *x1, *rrow, *parent, *cidx;  // [cap]
    uint64_t *size;       // [cap]
    uint8_t *kept;        // [cap]
    uint64_t *ctr;        // [8]: 0 n_runs, 1 n_cross_pairs, 2 n_kept, 3 gather error snapshot, 4 n_block_roots,
                          //      5, 6 keep-largest (size, label)
    uint32_t *broots;     // [cap]: the block-local roots left by k_union_local
    uint2 *pairs;         // [pair_cap]: run pairs that cross union blocks
    uint64_t pair_cap;
    uint32_t *klen;       // [cap]: kept length of every run (roix_extract_runs)
    uint64_t *koff;       // [cap + 1]: their exclusive prefix
};

constexpr int UB_MAX = 16384;     // max runs per union block (their parents live in shared memory: 64 KB)
constexpr int UB_THREADS = 1024;   // 4 runs per thread: short dependent chains

static size_t align256(size_t v) { return (v + 255) & ~(size_t)255; }

static size_t carve(void *base, const roix_geom &g, uint64_t cap, LabelWS *ws) {
    const uint64_t rows = g.nz * g.ny;
    size_t off = 0;
    auto take = [&](size_t bytes) {
        size_t o = off;
        off += align256(bytes);
        return o;
    };
    size_t o_rr = take(rows * 4), o_rs = take((rows + 1) * 4);
    size_t o_st = take(scan_tmp_elems(rows + 1 > cap ? rows + 1 : cap) * 8);
    size_t o_x0 = take(cap * 4), o_x1 = take(cap * 4), o_rw = take(cap * 4), o_pa = take(cap * 4),
           o_ci = take((cap + 1) * 4);
    size_t o_sz = take(cap * 8), o_kp = take(cap), o_ct = take(8 * 8), o_br = take(cap * 4);
    const uint64_t pair_cap = 2 * cap + 1024;
    size_t o_pr = take(pair_cap * 8);
    size_t o_kl = take(cap * 4), o_ko = take((cap + 1) * 8);
    if (ws) {
        char *b = (char *)base;
        ws->row_runs = (uint32_t *)(b + o_rr);
        ws->row_start = (uint32_t *)(b + o_rs);
        ws->scan_tmp = (uint64_t *)(b + o_st);
        ws->x0 = (uint32_t *)(b + o_x0);
        ws->x1 = (uint32_t *)(b + o_x1);
        ws->rrow = (uint32_t *)(b + o_rw);
        ws->parent = (uint32_t *)(b + o_pa);
        ws->cidx = (uint32_t *)(b + o_ci);
        ws->size = (uint64_t *)(b + o_sz);
        ws->kept = (uint8_t *)(b + o_kp);
        ws->ctr = (uint64_t *)(b + o_ct);
        ws->broots = (uint32_t *)(b + o_br);
        ws->pairs = (uint2 *)(b + o_pr);
        ws->pair_cap = pair_cap;
        ws->klen = (uint32_t *)(b + o_kl);
        ws->koff = (uint64_t *)(b + o_ko);
    }
    return off;
}

struct LGeo {
    uint64_t nz, ny, nx, z0;
    uint32_t W;
};

// word k (row-local) of row r of a linear bit array, pad bits beyond X cleared; never reads past
// word nwords - 1.
__device__ __forceinline__ uint32_t row_word_safe(const uint32_t *bits, const LGeo &G, uint64_t r, uint32_t k,
                                                  uint64_t nwords) {
    uint64_t b = r * G.nx + 32ull * k;
    uint32_t sh = (uint32_t)(b & 31);
    uint64_t wi = b >> 5;
    uint32_t lo = bits[wi];
    uint32_t hi = (sh && wi + 1 < nwords) ? bits[wi + 1] : 0u;
    uint32_t v = sh ? __funnelshift_r(lo, hi, sh) : lo;
    uint64_t rem = G.nx - 32ull * k;
    if (rem < 32) v &= low_mask((uint32_t)rem);
    return v;
}

__global__ void k_count_runs(const uint32_t *__restrict__ o, LGeo G, uint64_t nwords, uint32_t *row_runs,
                             roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t rows = G.nz * G.ny;
    const uint64_t wpg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t r = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += wpg) {
        uint32_t carry = 0, cnt = 0;
        for (uint32_t k0 = 0; k0 < G.W; k0 += 32) {
            uint32_t k = k0 + lane_id();
            uint32_t w = k < G.W ? row_word_safe(o, G, r, k, nwords) : 0u;
            uint32_t prev = __shfl_up_sync(FULL, w, 1);
            if (lane_id() == 0) prev = carry;
            carry = __shfl_sync(FULL, w, 31);
            cnt += __popc(w & ~((w << 1) | (prev >> 31)));
        }
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) cnt += __shfl_xor_sync(FULL, cnt, d);
        if (lane_id() == 0) row_runs[r] = cnt;
    }
}


// Warp per group of RIF consecutive rows: the offsets and (for rows of <= 128 words) all words of
// the RIF rows are loaded before any of them is processed, so each warp keeps RIF rows of loads in
// flight.  Longer rows are streamed 32 words at a time.
constexpr int RIF = 4, RW = 4;   // rows in flight per warp; words per lane kept in registers per row
__device__ __forceinline__ void runs_of_chunk(uint32_t cw, uint32_t next_lane31, uint32_t &carry, uint32_t k,
                                              uint32_t b0, uint32_t &sbase, uint32_t &ebase, uint32_t r,
                                              uint32_t *__restrict__ x0, uint32_t *__restrict__ x1,
                                              uint32_t *__restrict__ rrow) {
    const uint32_t lane = lane_id();
    uint32_t prev = __shfl_up_sync(FULL, cw, 1);
    if (lane == 0) prev = carry;
    uint32_t next = __shfl_down_sync(FULL, cw, 1);
    if (lane == 31) next = next_lane31;
    carry = __shfl_sync(FULL, cw, 31);
    uint32_t starts = cw & ~((cw << 1) | (prev >> 31));
    uint32_t ends = cw & ~((cw >> 1) | (next << 31));
    if (!__any_sync(FULL, (starts | ends) != 0)) return;   // no run boundary in these 32 words
    const uint32_t ns = __popc(starts), ne = __popc(ends);
    const uint32_t both = warp_incl_scan(ns | (ne << 16));  // both counts <= 32 * 16: one scan
    const uint32_t is = (both & 0xffffu) - ns, ie = (both >> 16) - ne;
    uint32_t ps = b0 + sbase + is, pe = b0 + ebase + ie;
    while (starts) {
        const uint32_t bb = __ffs(starts) - 1;
        starts &= starts - 1;
        x0[ps] = 32 * k + bb;
        rrow[ps] = r;
        ps++;
    }
    while (ends) {
        const uint32_t bb = __ffs(ends) - 1;
        ends &= ends - 1;
        x1[pe++] = 32 * k + bb + 1;
    }
    const uint32_t tot = __shfl_sync(FULL, both, 31);
    sbase += tot & 0xffffu;
    ebase += tot >> 16;
}

// after the row scan: total runs -> ctr[0], sc->n_runs, capacity check (block 0); over capacity no
// run is written and every later step sees none
__device__ __forceinline__ bool runs_total(const uint64_t *total, uint64_t cap, const LabelWS &W, roix_scalars *sc) {
    const uint64_t t = *total;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        W.ctr[0] = t > cap ? 0 : t;
        W.ctr[1] = 0;   // cross-block pairs
        W.ctr[2] = 0;
        W.ctr[4] = 0;   // block roots
        sc->n_runs = t;
        if (t > cap) set_err(sc, ROIX_ERR_CAPACITY);
    }
    return t <= cap;
}

__global__ void __launch_bounds__(256) k_extract_runs(const uint32_t *__restrict__ o, LGeo G, uint64_t nwords,
                                                      LabelWS W, const uint64_t *total, uint64_t cap,
                                                      roix_scalars *sc, uint32_t nslots) {
    if (get_err(sc)) return;
    if (!runs_total(total, cap, W, sc)) return;
    const uint32_t skip = (nslots && sc->run_slots == nslots) ? nslots : 0u;   // rows with <= skip runs came from the slots
    const uint64_t rows = G.nz * G.ny;
    const uint64_t ngroups = (rows + RIF - 1) / RIF;
    const uint64_t wpg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    const uint32_t lane = lane_id();
    uint32_t *__restrict__ x0 = W.x0;
    uint32_t *__restrict__ x1 = W.x1;
    uint32_t *__restrict__ rrow = W.rrow;
    const uint32_t *__restrict__ rs = W.row_start;
    const bool regs = G.W <= 32 * RW;
    for (uint64_t gi = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gi < ngroups; gi += wpg) {
        const uint64_t r0 = gi * RIF;
        // offsets of the group's rows: lanes 0..RIF load row_start[r0 .. r0+RIF]
        uint32_t off = 0;
        if (lane <= RIF && r0 + lane <= rows) off = rs[r0 + lane];
        if (!regs) {
            // long rows: the group's RIF rows advance chunk by chunk together, so their loads and
            // their (dependent) chunk steps interleave
            uint32_t carry[RIF], sb[RIF], eb[RIF], b0[RIF];
            bool live[RIF];
#pragma unroll
            bool any = false;
            for (int q = 0; q < RIF; q++) {
                b0[q] = __shfl_sync(FULL, off, q);
                live[q] = r0 + q < rows && __shfl_sync(FULL, off, q + 1) - b0[q] > skip;
                carry[q] = sb[q] = eb[q] = 0;
                any |= live[q];
            }
            if (!any) continue;   // every row of the group empty or taken from the run records
            for (uint32_t k0 = 0; k0 < G.W; k0 += 32) {
                uint32_t cw[RIF], nx[RIF];
#pragma unroll
                for (int q = 0; q < RIF; q++) {
                    cw[q] = (live[q] && k0 + lane < G.W) ? row_word_safe(o, G, r0 + q, k0 + lane, nwords) : 0u;
                    nx[q] = (live[q] && k0 + 32 < G.W) ? row_word_safe(o, G, r0 + q, k0 + 32, nwords) : 0u;
                }
#pragma unroll
                for (int q = 0; q < RIF; q++)
                    if (live[q])
                        runs_of_chunk(cw[q], nx[q], carry[q], k0 + lane, b0[q], sb[q], eb[q], (uint32_t)(r0 + q), x0, x1,
                                      rrow);
            }
            continue;
        }
        uint32_t wv[RIF][RW];
#pragma unroll
        for (int q = 0; q < RIF; q++) {
            const uint32_t a = __shfl_sync(FULL, off, q), b = __shfl_sync(FULL, off, q + 1);
            const bool live = r0 + q < rows && b - a > skip;
#pragma unroll
            for (int h = 0; h < RW; h++) {
                const uint32_t k = h * 32 + lane;
                wv[q][h] = (live && k < G.W) ? row_word_safe(o, G, r0 + q, k, nwords) : 0u;
            }
        }
#pragma unroll
        for (int q = 0; q < RIF; q++) {
            const uint64_t r = r0 + q;
            const uint32_t b0 = __shfl_sync(FULL, off, q), b1 = __shfl_sync(FULL, off, q + 1);
            if (r >= rows || b1 - b0 <= skip) continue;
            uint32_t carry = 0, sbase = 0, ebase = 0;
#pragma unroll
            for (int h = 0; h < RW; h++) {
                if (h * 32 >= (int)G.W) break;
                const uint32_t nxt = h + 1 < RW ? __shfl_sync(FULL, wv[q][h + 1], 0) : 0u;
                runs_of_chunk(wv[q][h], nxt, carry, h * 32 + lane, b0, sbase, ebase, (uint32_t)r, x0, x1, rrow);
            }
        }
    }
}

// Rows with at most rs runs: their run records, written by roix_morph_slots with o (the opening
// already had every row in registers), are copied to their scanned place -- those rows of o are not
// read again.  A warp per 32 rows: the rows with records are taken two at a time (both rows' record
// loads in flight before either is stored), lanes over the records (coalesced loads and stores).
__global__ void __launch_bounds__(256) k_runs_slots(LGeo G, LabelWS W, const uint2 *__restrict__ slots, uint32_t rs,
                                                    const uint64_t *total, uint64_t cap, roix_scalars *sc) {
    if (get_err(sc)) return;
    if (!runs_total(total, cap, W, sc)) return;
    if (sc->run_slots != rs) return;   // the opening did not write run records of this width
    const uint64_t rows = G.nz * G.ny;
    const uint32_t lane = lane_id();
    const uint64_t ng = (rows + 31) / 32, wstride = (uint64_t)gridDim.x * (blockDim.x >> 5);
    for (uint64_t gi = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); gi < ng; gi += wstride) {
        const uint64_t r = gi * 32 + lane;
        uint32_t a = 0, c = 0;
        if (r < rows) {
            a = W.row_start[r];
            c = W.row_start[r + 1] - a;
        }
        uint32_t use = __ballot_sync(FULL, c > 0 && c <= rs);
        while (use) {
            const uint32_t q0 = __ffs(use) - 1;
            use &= use - 1;
            const uint32_t q1 = use ? __ffs(use) - 1 : 32u;
            if (use) use &= use - 1;
            const uint32_t a0 = __shfl_sync(FULL, a, q0), c0 = __shfl_sync(FULL, c, q0);
            const uint32_t a1 = __shfl_sync(FULL, a, q1 & 31), c1 = q1 < 32 ? __shfl_sync(FULL, c, q1 & 31) : 0u;
            for (uint32_t i = lane; i < max(c0, c1); i += 32) {
                uint2 v0 = make_uint2(0, 0), v1 = make_uint2(0, 0);
                if (i < c0) v0 = slots[(gi * 32 + q0) * rs + i];
                if (i < c1) v1 = slots[(gi * 32 + q1) * rs + i];
                if (i < c0) {
                    W.x0[a0 + i] = v0.x;
                    W.x1[a0 + i] = v0.y;
                    W.rrow[a0 + i] = (uint32_t)(gi * 32 + q0);
                }
                if (i < c1) {
                    W.x0[a1 + i] = v1.x;
                    W.x1[a1 + i] = v1.y;
                    W.rrow[a1 + i] = (uint32_t)(gi * 32 + q1);
                }
            }
        }
    }
}

// Whole-row form (X % 32 == 0, W = L KW words, L a power of two <= 32): a warp holds S = 32 / L row
// segments, lane sl of a segment the KW consecutive words [KW sl, KW sl + KW) of a row; each segment
// takes RR consecutive rows per iteration, all their loads issued before any row is processed.  Run
// starts / ends of every word come from one shfl each way; one packed segment scan gives every
// lane's first start / end slot.
template <int L, int KW, int RR>
__global__ void __launch_bounds__(256) k_extract_runs_rows(const uint32_t *__restrict__ o, LGeo G, LabelWS W,
                                                           const uint64_t *total, uint64_t cap, roix_scalars *sc,
                                                           uint32_t nslots) {
    if (get_err(sc)) return;
    if (!runs_total(total, cap, W, sc)) return;
    const uint32_t skip = (nslots && sc->run_slots == nslots) ? nslots : 0u;   // rows with <= skip runs came from the slots
    constexpr int S = 32 / L;
    const uint32_t lane = lane_id(), sl = lane & (L - 1), seg = lane / L;
    const uint64_t rows = G.nz * G.ny;
    const uint64_t ngroups = (rows + S * RR - 1) / (S * RR);
    const uint64_t wpg = (uint64_t)gridDim.x * (blockDim.x >> 5);
    uint32_t *__restrict__ x0 = W.x0;
    uint32_t *__restrict__ x1 = W.x1;
    uint32_t *__restrict__ rrow = W.rrow;
    const uint32_t *__restrict__ rs = W.row_start;
    // row offsets of a group, one per lane when the segment is wide enough (loaded an iteration ahead)
    auto load_off = [&](uint64_t g) -> uint32_t {
        const uint64_t r = (g * S + seg) * RR + sl;
        return (g < ngroups && sl <= (uint32_t)RR && r <= rows) ? __ldg(rs + r) : 0u;
    };
    // the words of a group's live rows (rows with runs left to extract); offv: the group's offsets
    auto load_words = [&](uint64_t g, uint32_t offv, const uint32_t *offa, uint32_t (&dst)[RR][KW]) {
        const uint64_t rg = (g * S + seg) * RR;
#pragma unroll
        for (int q = 0; q < RR; q++) {
            uint32_t a, b;
            if constexpr (L > RR) {
                a = __shfl_sync(FULL, offv, q, L);
                b = __shfl_sync(FULL, offv, q + 1, L);
            } else {
                a = offa[q];
                b = offa[q + 1];
            }
            const bool live = g < ngroups && rg + q < rows && b - a > skip;
            const uint32_t *src = o + (rg + q) * (uint64_t)(L * KW) + KW * sl;
#pragma unroll
            for (int i = 0; i < KW; i++) dst[q][i] = 0u;
            if (live) {
                if constexpr (KW == 1) {
                    dst[q][0] = __ldg(src);
                } else if constexpr (KW == 2) {
                    const uint2 v = __ldg(reinterpret_cast<const uint2 *>(src));
                    dst[q][0] = v.x;
                    dst[q][1] = v.y;
                } else {
                    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(src));
                    dst[q][0] = v.x;
                    dst[q][1] = v.y;
                    dst[q][2] = v.z;
                    dst[q][3] = v.w;
                }
            }
        }
    };
    // whole-warp segments (L > RR): offsets two groups ahead, words one group ahead
    uint64_t gi = (uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    uint32_t off_cur = 0, off_nxt = 0, wv_nxt[RR][KW];
    if constexpr (L > RR) {
        off_cur = load_off(gi);
        off_nxt = load_off(gi + wpg);
        load_words(gi, off_cur, nullptr, wv_nxt);
    }
    for (; gi < ngroups; gi += wpg) {
        const uint64_t r0 = (gi * S + seg) * RR;   // this segment's first row
        // row offsets rs[r0 .. r0 + RR]: one per lane when the segment is wide enough, else all per lane
        uint32_t off = 0, offs[RR + 1];
        uint32_t wv[RR][KW];
        if constexpr (L > RR) {
            off = off_cur;
#pragma unroll
            for (int q = 0; q < RR; q++)
#pragma unroll
                for (int i = 0; i < KW; i++) wv[q][i] = wv_nxt[q][i];
            off_cur = off_nxt;
            off_nxt = load_off(gi + 2 * wpg);
            load_words(gi + wpg, off_cur, nullptr, wv_nxt);
        } else {
#pragma unroll
            for (int q = 0; q <= RR; q++) offs[q] = r0 + q <= rows ? __ldg(rs + r0 + q) : 0u;
            load_words(gi, 0u, offs, wv);
        }
        auto row_off = [&](int q) {
            if constexpr (L > RR) return __shfl_sync(FULL, off, q, L);
            else return offs[q];
        };
#pragma unroll
        for (int q = 0; q < RR; q++) {
            const uint64_t r = r0 + q;
            const uint32_t b0 = row_off(q);
            // a whole-warp segment skips rows without a run to extract (most rows of a sparse volume)
            if constexpr (L == 32) {
                if (r >= rows || row_off(q + 1) - b0 <= skip) continue;
            }
            uint32_t left = __shfl_up_sync(FULL, wv[q][KW - 1], 1, L);
            uint32_t right = __shfl_down_sync(FULL, wv[q][0], 1, L);
            if (sl == 0) left = 0u;
            if (sl == L - 1) right = 0u;
            uint32_t st[KW], en[KW], ns = 0, ne = 0;
#pragma unroll
            for (int i = 0; i < KW; i++) {
                const uint32_t c = wv[q][i];
                st[i] = c & ~__funnelshift_l(i ? wv[q][i - 1] : left, c, 1);
                en[i] = c & ~__funnelshift_r(c, i < KW - 1 ? wv[q][i + 1] : right, 1);
                ns += __popc(st[i]);
                ne += __popc(en[i]);
            }
            if constexpr (L == 32) {
                // common case: no lane holds two starts or two ends -- ranks by ballot, one store each
                if (!__any_sync(FULL, (ns | ne) > 1)) {
                    const uint32_t lt = (1u << sl) - 1u;
                    const uint32_t bS = __ballot_sync(FULL, ns != 0), bE = __ballot_sync(FULL, ne != 0);
                    uint32_t xs = 0, xe = 0;
#pragma unroll
                    for (int i = KW - 1; i >= 0; i--) {
                        if (st[i]) xs = 32 * i + __ffs(st[i]) - 1;
                        if (en[i]) xe = 32 * i + __ffs(en[i]);
                    }
                    const uint32_t xb = 32 * KW * sl;
                    if (ns) {
                        const uint32_t ps = b0 + __popc(bS & lt);
                        x0[ps] = xb + xs;
                        rrow[ps] = (uint32_t)r;
                    }
                    if (ne) x1[b0 + __popc(bE & lt)] = xb + xe;
                    continue;
                }
            }
            // inclusive segment scan of (starts | ends << 16); both <= 16 KW per lane
            uint32_t both = ns | (ne << 16);
#pragma unroll
            for (int d = 1; d < L; d <<= 1) {
                const uint32_t t = __shfl_up_sync(FULL, both, d, L);
                if (sl >= (uint32_t)d) both += t;
            }
            uint32_t ps = b0 + (both & 0xffffu) - ns, pe = b0 + (both >> 16) - ne;
#pragma unroll
            for (int i = 0; i < KW; i++) {
                const uint32_t xb = 32 * (KW * sl + i);
                uint32_t m = st[i];
                while (m) {
                    const uint32_t bb = __ffs(m) - 1;
                    m &= m - 1;
                    x0[ps] = xb + bb;
                    rrow[ps] = (uint32_t)r;
                    ps++;
                }
                m = en[i];
                while (m) {
                    const uint32_t bb = __ffs(m) - 1;
                    m &= m - 1;
                    x1[pe++] = xb + bb + 1;
                }
            }
        }
    }
}

__device__ __forceinline__ uint32_t find_root(const uint32_t *parent, uint32_t x) {
    uint32_t p = parent[x];
    while (p != x) {
        x = p;
        p = parent[x];
    }
    return x;
}

__device__ __forceinline__ uint32_t find_compress(uint32_t *parent, uint32_t x) {
    // path halving: parent pointers only ever move to ancestors, so racing writes stay valid
    uint32_t p = parent[x];
    while (p != x) {
        uint32_t gp = parent[p];
        if (gp != p) parent[x] = gp;
        x = p;
        p = gp;
    }
    return x;
}

__device__ void unite(uint32_t *parent, uint32_t a, uint32_t b) {
    while (true) {
        a = find_compress(parent, a);
        b = find_compress(parent, b);
        if (a == b) return;
        if (a < b) {
            uint32_t t = a;
            a = b;
            b = t;
        }
        uint32_t old = atomicMin(&parent[a], b);  // link the larger root under the smaller
        if (old == a) return;
        a = old;
    }
}

struct Nb {
    int dz, dy, ext;
};

// previous-row neighbourhoods per connectivity (rows (z, y-1) and (z-1, *))
__constant__ Nb c_nb[5][4] = {
    /* 4  */ {{0, -1, 0}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    /* 8  */ {{0, -1, 1}, {0, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    /* 6  */ {{0, -1, 0}, {-1, 0, 0}, {0, 0, 0}, {0, 0, 0}},
    /* 18 */ {{0, -1, 1}, {-1, 0, 1}, {-1, -1, 0}, {-1, 1, 0}},
    /* 26 */ {{0, -1, 1}, {-1, -1, 1}, {-1, 0, 1}, {-1, 1, 1}},
};
__constant__ int c_nnb[5] = {1, 1, 2, 4, 4};

__device__ __forceinline__ uint32_t sfind(uint32_t *lp, uint32_t x) {
    uint32_t p = lp[x];
    while (p != x) {
        uint32_t gp = lp[p];
        if (gp != p) lp[x] = gp;
        x = p;
        p = gp;
    }
    return x;
}

__device__ __forceinline__ void sunite(uint32_t *lp, uint32_t a, uint32_t b) {
    while (true) {
        a = sfind(lp, a);
        b = sfind(lp, b);
        if (a == b) return;
        if (a < b) {
            uint32_t t = a;
            a = b;
            b = t;
        }
        uint32_t old = atomicMin(&lp[a], b);
        if (old == a) return;
        a = old;
    }
}

// Union, phase 1: a CTA owns the runs [base, base + UB_RUNS) and their parent pointers in shared
// memory.  Neighbour pairs inside the block are united there; pairs reaching an earlier block are
// queued.  The block's runs then point (globally) at their block-local root.
__global__ void __launch_bounds__(UB_THREADS) k_union_local(LGeo G, int ci, LabelWS W, uint32_t UB_RUNS,
                                                           roix_scalars *sc) {
    extern __shared__ uint32_t lp[];
    if (get_err(sc)) return;
    const uint64_t n = W.ctr[0];
    for (uint64_t base = (uint64_t)blockIdx.x * UB_RUNS; base < n; base += (uint64_t)gridDim.x * UB_RUNS) {
    const uint32_t cnt = (uint32_t)min((uint64_t)UB_RUNS, n - base);
    __syncthreads();   // the previous block of runs is finished with lp[]
    for (uint32_t k = threadIdx.x; k < cnt; k += blockDim.x) lp[k] = k;
    __syncthreads();
    const int nnb = c_nnb[ci];
    for (uint32_t k0 = 0; k0 < cnt; k0 += blockDim.x) {
        const uint32_t k = k0 + threadIdx.x;
        const bool act = k < cnt;
        uint2 pend[8];
        int np = 0;
        if (act) {
            const uint64_t i = base + k;
            const uint32_t r = W.rrow[i];
            const int64_t z = r / G.ny, y = r % G.ny;
            const uint32_t a0 = W.x0[i], a1 = W.x1[i];
            for (int q = 0; q < nnb; q++) {
                const Nb nb = c_nb[ci][q];
                const int64_t zz = z + nb.dz, yy = y + nb.dy;
                if (zz < 0 || yy < 0 || yy >= (int64_t)G.ny) continue;
                const uint64_t nr = (uint64_t)zz * G.ny + yy;
                uint32_t lo = W.row_start[nr], hi = W.row_start[nr + 1];
                const uint32_t end = hi;
                while (lo < hi) {
                    uint32_t mid = (lo + hi) >> 1;
                    if (W.x1[mid] + nb.ext > a0) hi = mid;
                    else lo = mid + 1;
                }
                for (uint32_t j = lo; j < end && W.x0[j] < a1 + nb.ext; j++) {
                    if (j >= base) sunite(lp, k, (uint32_t)(j - base));
                    else if (np < 8) pend[np++] = make_uint2((uint32_t)i, j);
                    else {  // flush (rare: more than 8 cross-block overlaps of one run)
                        unsigned long long at = atomicAdd((unsigned long long *)&W.ctr[1], 8ull);
                        for (int t = 0; t < 8; t++)
                            if (at + t < W.pair_cap) W.pairs[at + t] = pend[t];
                        np = 0;
                        pend[np++] = make_uint2((uint32_t)i, j);
                    }
                }
            }
        }
        // warp-aggregated append of the queued cross-block pairs
        const uint32_t tot = warp_incl_scan((uint32_t)np);
        unsigned long long at = 0;
        const uint32_t wsum = __shfl_sync(FULL, tot, 31);
        if (lane_id() == 31 && wsum) at = atomicAdd((unsigned long long *)&W.ctr[1], (unsigned long long)wsum);
        at = __shfl_sync(FULL, at, 31) + (tot - np);
        for (int t = 0; t < np; t++)
            if (at + t < W.pair_cap) W.pairs[at + t] = pend[t];
    }
    __syncthreads();
    for (uint32_t k0 = 0; k0 < cnt; k0 += blockDim.x) {   // whole warps (the root list append below)
        const uint32_t k = k0 + threadIdx.x;
        bool root = false;
        if (k < cnt) {
            uint32_t r = k, p = lp[r];
            while (p != r) {
                r = p;
                p = lp[r];
            }
            W.parent[base + k] = (uint32_t)(base + r);
            W.size[base + k] = 0;
            root = r == k;
        }
        // block-local roots -> W.broots: only they can be linked further by k_union_cross
        const uint32_t bal = __ballot_sync(FULL, root);
        unsigned long long at = 0;
        if (lane_id() == 0 && bal) at = atomicAdd((unsigned long long *)&W.ctr[4], (unsigned long long)__popc(bal));
        at = __shfl_sync(FULL, at, 0);
        if (root) W.broots[at + __popc(bal & low_mask(lane_id()))] = (uint32_t)(base + k);
    }
    }
}

// Union, phase 2: the queued cross-block pairs, lock-free union-by-min on the global parents.
__global__ void k_union_cross(LabelWS W, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t np = W.ctr[1];
    if (np > W.pair_cap) {
        if (blockIdx.x == 0 && threadIdx.x == 0) set_err(sc, ROIX_ERR_CAPACITY);
        return;
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < np; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint2 pr = W.pairs[i];
        unite(W.parent, pr.x, pr.y);
    }
}

// After k_union_cross: every block-local root points at its final root (compressing on the way).
// Every other run's parent is then one of those block roots (unions only ever link roots, and path
// halving only moves a pointer to an ancestor), so two hops reach the final root.
// Union by min index makes parent values strictly decrease towards a root, so every pointer update
// here is an atomicMin: a thread's halving step can never overwrite another's final root pointer
// with an intermediate ancestor.
__global__ void k_resolve_broots(LabelWS W, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t nb = W.ctr[4];
    uint32_t *par = W.parent;
    for (uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; t < nb; t += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t b = W.broots[t];
        uint32_t x = b, p = par[x];
        while (p != x) {   // find with path halving
            const uint32_t gp = par[p];
            if (gp != p) atomicMin(&par[x], gp);
            x = p;
            p = gp;
        }
        atomicMin(&par[b], x);
    }
}

// Final roots (two hops) and component sizes.  A warp owns FL_J x 32 consecutive runs (lane l: runs
// l, l + 32, ...); each lane sums run lengths while the root stays the same and flushes on a change,
// then the lanes holding the same root merge their sums (match.any) -- one atomic per root per warp,
// so a component spanning the whole volume (C4's matrix) is not one hot address hit per run.
constexpr int FL_J = 16;
__global__ void k_flatten_sizes(LabelWS W, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = W.ctr[0];
    const uint32_t lane = lane_id();
    const uint64_t nw = (uint64_t)gridDim.x * (blockDim.x >> 5);
    // runs per lane: up to FL_J, fewer when there are not enough runs to keep every warp busy
    const int J = (int)min((uint64_t)FL_J, max((uint64_t)1, n / (nw * 32)));
    for (uint64_t b0 = ((uint64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * (32 * J); b0 < n;
         b0 += nw * 32 * J) {
        uint32_t cur = 0xffffffffu;
        uint64_t sum = 0;
        // four runs at a time: their parent loads, then the second hops, issued before any is used
        for (int j0 = 0; j0 < J; j0 += 4) {
            uint32_t pp[4], rt[4], ln[4];
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint64_t i = b0 + (uint64_t)(j0 + u) * 32 + lane;
                const bool ok = j0 + u < J && i < n;
                pp[u] = ok ? W.parent[i] : 0u;
                ln[u] = ok ? W.x1[i] - W.x0[i] : 0u;
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint64_t i = b0 + (uint64_t)(j0 + u) * 32 + lane;
                rt[u] = (j0 + u < J && i < n) ? W.parent[pp[u]] : 0u;   // two hops after k_resolve_broots
            }
#pragma unroll
            for (int u = 0; u < 4; u++) {
                const uint64_t i = b0 + (uint64_t)(j0 + u) * 32 + lane;
                if (j0 + u >= J || i >= n) break;
                W.parent[i] = rt[u];
                if (rt[u] != cur) {
                    if (sum) atomicAdd((unsigned long long *)&W.size[cur], (unsigned long long)sum);
                    cur = rt[u];
                    sum = 0;
                }
                sum += ln[u];
            }
        }
        const uint32_t grp = __match_any_sync(FULL, cur);
        const uint64_t tot = __reduce_add_sync(grp, (uint32_t)sum);   // per-warp sums fit 32 bits
        if (cur != 0xffffffffu && (__ffs(grp) - 1) == (int)lane && tot)
            atomicAdd((unsigned long long *)&W.size[cur], (unsigned long long)tot);
    }
}

// ------------------------------------------------------------------ finish: table, filter, K
// Merge map (sharded volumes): sorted global labels of this slab's boundary components with their
// merged label (the global minimum index of the merged component) and total size.  nmap = 0 on a
// single GPU.
struct MapView {
    const uint64_t *label, *final_label, *total;
    const uint64_t *n;   // device: map length (null: no map)
};

__device__ __forceinline__ uint64_t gidx(const LGeo &G, const LabelWS &W, uint32_t i) {
    return ((G.z0 * G.ny) + W.rrow[i]) * G.nx + W.x0[i];
}

// (final label, total size) of local root i
__device__ __forceinline__ void resolve_root(const LGeo &G, const LabelWS &W, const MapView &M, uint32_t i,
                                             uint64_t &fin, uint64_t &tot) {
    const uint64_t L = gidx(G, W, i);
    fin = L;
    tot = W.size[i];
    const uint64_t mn = M.n ? *M.n : 0;
    uint64_t lo = 0, hi = mn;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (M.label[mid] < L) lo = mid + 1;
        else hi = mid;
    }
    if (lo < mn && M.label[lo] == L) {
        fin = M.final_label[lo];
        tot = M.total[lo];
    }
}

// NEXT-3 keep-largest: over the components this slab owns (local roots whose
// final label is their own first voxel), phase 0 takes the largest size into best[0], phase 1 the
// smallest label among the components of that size into best[1] (the raster-order anchor tie-break).
// best[] is pre-set to (0, 2^63 - 1 = none); sharded callers reduce it over ranks between the phases
// (labels are < 2^63, so signed and unsigned minima agree).
__global__ void k_largest(LGeo G, LabelWS W, MapView M, uint64_t *best, int phase, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = W.ctr[0];
    const uint64_t want = phase ? best[0] : 0;
    uint64_t v = phase ? ~0ull : 0ull;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (W.parent[i] != (uint32_t)i) continue;
        uint64_t fin, tot;
        resolve_root(G, W, M, (uint32_t)i, fin, tot);
        if (fin != gidx(G, W, (uint32_t)i)) continue;   // another slab owns it
        if (phase == 0) v = max(v, tot);
        else if (tot == want) v = min(v, fin);
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) {
        const uint64_t o = __shfl_xor_sync(FULL, v, d);
        v = phase ? min(v, o) : max(v, o);
    }
    if (lane_id() == 0) {
        if (phase == 0 && v) atomicMax((unsigned long long *)&best[0], (unsigned long long)v);
        if (phase == 1 && v != ~0ull) atomicMin((unsigned long long *)&best[1], (unsigned long long)v);
    }
}

__global__ void k_largest_init(uint64_t *best) {
    best[0] = 0;
    best[1] = 0x7fffffffffffffffull;
}

// cidx flags: 1 for local roots that own a table entry (their label is the merged component's label).
// kept: size >= min_size, or (keep != NULL) the component labelled keep[1]
__global__ void k_root_flags(LGeo G, LabelWS W, MapView M, uint64_t min_size, const uint64_t *keep,
                             roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = W.ctr[0];
    const uint64_t keep_label = keep ? keep[1] : 0;
    uint32_t nk = 0;
    constexpr int TC = 4;   // runs per thread per step, their parent loads issued together
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * TC;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * TC + threadIdx.x; i0 < n; i0 += stride) {
        uint32_t p[TC];
#pragma unroll
        for (int t = 0; t < TC; t++) {
            const uint64_t i = i0 + (uint64_t)t * blockDim.x;
            p[t] = i < n ? W.parent[i] : 0u;
        }
#pragma unroll
        for (int t = 0; t < TC; t++) {
            const uint64_t i = i0 + (uint64_t)t * blockDim.x;
            if (i >= n) break;
            uint32_t f = 0;
            if (p[t] == (uint32_t)i) {
                uint64_t fin, tot;
                resolve_root(G, W, M, (uint32_t)i, fin, tot);
                const uint8_t kp = keep ? fin == keep_label : tot >= min_size;
                W.kept[i] = kp;
                f = fin == gidx(G, W, (uint32_t)i);
                nk += f & kp;
            }
            W.cidx[i] = f;
        }
    }
#pragma unroll
    for (int d = 16; d > 0; d >>= 1) nk += __shfl_xor_sync(FULL, nk, d);
    if (lane_id() == 0 && nk) atomicAdd((unsigned long long *)&W.ctr[2], (unsigned long long)nk);
}

// a7 outputs, one pass over the runs: the component table (entries owned by roots whose final label
// is their own first voxel, at their scanned index: increasing min index), and K = o with the bits of
// every run of a dropped component cleared (in place when K aliases o)
__global__ void k_table_clear(LGeo G, LabelWS W, MapView M, const uint32_t *cscan, const uint64_t *nroots,
                              roix_label_out out, roix_scalars *sc) {
    if (get_err(sc)) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        sc->n_components = *nroots;
        sc->n_kept = W.ctr[2];
        if (out.comp_min && *nroots > out.comp_cap) set_err(sc, ROIX_ERR_CAPACITY);
    }
    const uint64_t n = W.ctr[0];
    uint32_t *K = out.keep_bits;
    // TC runs per thread per step (a block's runs are consecutive: coalesced run loads), every load of
    // the step issued before any is used: the random kept[parent] reads overlap each other
    constexpr int TC = 4;
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * TC;
    for (uint64_t i0 = (uint64_t)blockIdx.x * blockDim.x * TC + threadIdx.x; i0 < n; i0 += stride) {
        uint32_t p[TC], r[TC], a[TC], z[TC];
        uint8_t kp[TC];
#pragma unroll
        for (int t = 0; t < TC; t++) {
            const uint64_t i = i0 + (uint64_t)t * blockDim.x;
            p[t] = i < n ? W.parent[i] : 0u;
            r[t] = i < n ? W.rrow[i] : 0u;
            a[t] = i < n ? W.x0[i] : 0u;
            z[t] = i < n ? W.x1[i] : 0u;
        }
#pragma unroll
        for (int t = 0; t < TC; t++) kp[t] = i0 + (uint64_t)t * blockDim.x < n ? W.kept[p[t]] : 1;
#pragma unroll
        for (int t = 0; t < TC; t++) {
            const uint64_t i = i0 + (uint64_t)t * blockDim.x;
            if (i >= n) break;
            if (out.comp_min && p[t] == (uint32_t)i) {
                uint64_t fin, tot;
                resolve_root(G, W, M, (uint32_t)i, fin, tot);
                if (fin == gidx(G, W, (uint32_t)i)) {
                    const uint64_t c = cscan[i];
                    if (c < out.comp_cap) {
                        out.comp_min[c] = fin;
                        out.comp_size[c] = tot;
                        if (out.comp_kept) out.comp_kept[c] = kp[t];
                    }
                }
            }
            if (K && !kp[t]) {
                uint64_t b = (uint64_t)r[t] * G.nx + a[t], e = (uint64_t)r[t] * G.nx + z[t];
                while (b < e) {
                    const uint64_t wi = b >> 5;
                    const uint32_t sh = (uint32_t)(b & 31);
                    const uint32_t take = (uint32_t)min((uint64_t)(32 - sh), e - b);
                    atomicAnd(&K[wi], ~(low_mask(take) << sh));
                    b += take;
                }
            }
        }
    }
}

__global__ void k_labels(LGeo G, LabelWS W, MapView M, uint64_t *labels, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = W.ctr[0];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint64_t lab, tot;
        resolve_root(G, W, M, W.parent[i], lab, tot);
        const uint64_t base = (uint64_t)W.rrow[i] * G.nx;
        for (uint32_t x = W.x0[i]; x < W.x1[i]; x++) labels[base + x] = lab;
    }
}

// ------------------------------------------------------------------ sharded volumes: slab faces
// runs of the slab's first (side 0) or last (side 1) plane, with their local root's global label
__global__ void k_boundary_runs(LGeo G, LabelWS W, int side, roix_brun *out, uint64_t cap, uint64_t *count,
                                roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t r0 = side ? (G.nz - 1) * G.ny : 0, r1 = r0 + G.ny;
    const uint32_t a = W.row_start[r0], b = W.row_start[r1];
    const uint64_t nb = W.ctr[0] ? (uint64_t)(b - a) : 0;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *count = nb;
        if (nb > cap) set_err(sc, ROIX_ERR_CAPACITY);
    }
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nb && k < cap; k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = a + (uint32_t)k;
        roix_brun rr;
        rr.y = (uint32_t)(W.rrow[i] - r0);
        rr.x0 = W.x0[i];
        rr.x1 = W.x1[i];
        rr.pad = 0;
        rr.label = gidx(G, W, W.parent[i]);
        out[k] = rr;
    }
}

// pairs (label of this slab's first-plane component, label of the previous slab's last-plane one)
__global__ void k_link(LGeo G, LabelWS W, int ci, const roix_brun *prev, const uint64_t *n_prev, uint64_t *pairs,
                       uint64_t pair_cap, uint64_t *n_pairs, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint32_t a = W.row_start[0], b = W.row_start[G.ny];
    const uint64_t np = *n_prev;
    if (!W.ctr[0]) return;
    // cross-plane neighbourhood rows (dz = -1) per connectivity: dy range and x extension
    const int dymax = (ci == 4 || ci == 3) ? 1 : 0;   // 26: all dy; 18: dy != 0 only without x extension
    for (uint64_t k = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; k < (uint64_t)(b - a); k += (uint64_t)gridDim.x * blockDim.x) {
        const uint32_t i = a + (uint32_t)k;
        const int64_t y = W.rrow[i];
        const uint32_t x0 = W.x0[i], x1 = W.x1[i];
        const uint64_t mylab = gidx(G, W, W.parent[i]);
        for (int dy = -dymax; dy <= dymax; dy++) {
            const int64_t yy = y + dy;
            if (yy < 0 || yy >= (int64_t)G.ny) continue;
            const uint32_t ext = (ci == 4 || (ci == 3 && dy == 0)) ? 1u : 0u;
            // first prev run with (y, x1 + ext) > (yy, x0)
            uint64_t lo = 0, hi = np;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) >> 1;
                const roix_brun r = prev[mid];
                if ((int64_t)r.y < yy || ((int64_t)r.y == yy && r.x1 + ext <= x0)) lo = mid + 1;
                else hi = mid;
            }
            for (uint64_t j = lo; j < np; j++) {
                const roix_brun r = prev[j];
                if ((int64_t)r.y != yy || r.x0 >= x1 + ext) break;
                const unsigned long long at = atomicAdd((unsigned long long *)n_pairs, 1ull);
                if (at < pair_cap) {
                    pairs[2 * at] = mylab;
                    pairs[2 * at + 1] = r.label;
                } else {
                    set_err(sc, ROIX_ERR_CAPACITY);
                }
            }
        }
    }
}

// (label, size) of the local components touching the slab's first or last plane
__global__ void k_mark_boundary(LGeo G, LabelWS W, roix_scalars *sc) {
    if (get_err(sc)) return;
    if (!W.ctr[0]) return;
    const uint32_t ranges[4] = {W.row_start[0], W.row_start[G.ny], W.row_start[(G.nz - 1) * G.ny],
                                W.row_start[G.nz * G.ny]};
    for (int s = 0; s < 2; s++)
        for (uint64_t i = ranges[2 * s] + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ranges[2 * s + 1];
             i += (uint64_t)gridDim.x * blockDim.x)
            W.kept[W.parent[i]] = 2;   // scratch mark (kept[] is rewritten by the finish phase)
}

// boundary roots in increasing run index (= increasing label): flag, scan, write
__device__ __forceinline__ bool broot(const LabelWS &W, uint64_t i) { return W.parent[i] == (uint32_t)i && W.kept[i] == 2; }

__global__ void k_broot_flags(LabelWS W) {
    const uint64_t n = W.ctr[0];   // the scan reads [0, n) only
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        W.cidx[i] = broot(W, i);
}

__global__ void k_boundary_roots(LGeo G, LabelWS W, const uint64_t *total, uint64_t *labels, uint64_t *sizes,
                                 uint64_t cap, uint64_t *count, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = W.ctr[0], m = *total;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        *count = m;
        if (m > cap) set_err(sc, ROIX_ERR_CAPACITY);
    }
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        if (!broot(W, i)) continue;
        const uint64_t at = W.cidx[i];
        if (at < cap) {
            labels[at] = gidx(G, W, (uint32_t)i);
            sizes[at] = W.size[i];
        }
    }
}

__global__ void k_clear_marks(LabelWS W) {
    const uint64_t n = W.ctr[0];
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) W.kept[i] = 0;
}

}  // namespace roix

using namespace roix;

size_t label_workspace_bytes(const roix_geom &g, uint64_t cap) { return carve(nullptr, g, cap, nullptr); }

static int ctas(uint64_t work, int threads) {
    uint64_t need = (work + threads - 1) / threads;
    uint64_t cap = (uint64_t)num_sms() * 8;
    if (need < 1) need = 1;
    return (int)(need < cap ? need : cap);
}

static LGeo make_geo(const roix_geom &g) {
    LGeo G;
    G.nz = g.nz;
    G.ny = g.ny;
    G.nx = g.nx;
    G.z0 = g.z0;
    G.W = (uint32_t)((g.nx + 31) / 32);
    return G;
}

static int conn_index(uint32_t conn) { return conn == 4 ? 0 : conn == 8 ? 1 : conn == 6 ? 2 : conn == 18 ? 3 : 4; }

// a6 on the slab: runs, union (block-local then cross-block), flatten, sizes
cudaError_t launch_label_local(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom &g, uint32_t conn,
                               uint64_t cap, void *ws, roix_scalars *sc, cudaStream_t st, const uint2 *run_slots,
                               uint32_t rs) {
    LabelWS W;
    carve(ws, g, cap, &W);
    const LGeo G = make_geo(g);
    const uint64_t rows = g.nz * g.ny, n = rows * g.nx, nwords = (n + 31) / 32;
    const int ci = conn_index(conn);
    cudaError_t e;
    const uint32_t *rr = row_runs;
    if (!rr) {
        k_count_runs<<<ctas(rows * 32, 256), 256, 0, st>>>(o_bits, G, nwords, W.row_runs, sc);
        rr = W.row_runs;
    }
    if ((e = scan_u32(rr, W.row_start, rows, W.scan_tmp, st)) != cudaSuccess) return e;
    const uint64_t *rtot = scan_total_ptr(W.scan_tmp, rows);
    const int runs_grid = num_sms() * 8;
    if (!row_runs || !run_slots) rs = 0;   // run records exist only next to the opening's run counts
    if (rs) k_runs_slots<<<ctas(rows, 256), 256, 0, st>>>(G, W, run_slots, rs, rtot, cap, sc);
    const uint32_t Wd = G.W;
    if (g.nx % 32 == 0 && ((Wd <= 32 && (Wd & (Wd - 1)) == 0) || Wd == 64 || Wd == 128)) {
        const uint32_t L = Wd < 32 ? Wd : 32;
        const int grid = ctas(rows * L / 4, 256);   // ~4 rows per warp iteration
#define ROIX_RUNS_ROWS(LL, KK, RR) \
    k_extract_runs_rows<LL, KK, RR><<<grid, 256, 0, st>>>(o_bits, G, W, rtot, cap, sc, rs)
        switch (Wd) {
        case 1: ROIX_RUNS_ROWS(1, 1, 4); break;
        case 2: ROIX_RUNS_ROWS(2, 1, 4); break;
        case 4: ROIX_RUNS_ROWS(4, 1, 4); break;
        case 8: ROIX_RUNS_ROWS(8, 1, 4); break;
        case 16: ROIX_RUNS_ROWS(16, 1, 4); break;
        case 32: ROIX_RUNS_ROWS(32, 1, 4); break;
        case 64: ROIX_RUNS_ROWS(32, 2, 4); break;
        default: ROIX_RUNS_ROWS(32, 4, 2); break;
        }
#undef ROIX_RUNS_ROWS
    } else {
        k_extract_runs<<<ctas(rows * 32, 256), 256, 0, st>>>(o_bits, G, nwords, W, rtot, cap, sc, rs);
    }
    static std::atomic<unsigned long long> attr{0};
    if ((e = dyn_smem_once(k_union_local, UB_MAX * 4, attr)) != cudaSuccess) return e;
    // Union blocks: 16 K runs for large slabs -- several planes' runs, so most z-links stay inside one
    // block and the cross-block queue is 3x shorter (C4: union_cross 490 -> 142 us) -- 4 K runs for
    // small ones, where more, smaller blocks keep the SMs busy (C2: union_local 81 -> 29 us).
    const uint32_t ub = cap >= (1ull << 23) ? UB_MAX : UB_MAX / 4;
    uint64_t nub = (cap + ub - 1) / ub;
    if (nub > (uint64_t)num_sms() * 2) nub = (uint64_t)num_sms() * 2;   // persistent over blocks of runs
    k_union_local<<<(unsigned)nub, UB_THREADS, ub * 4, st>>>(G, ci, W, ub, sc);
    k_union_cross<<<runs_grid, 256, 0, st>>>(W, sc);
    k_resolve_broots<<<runs_grid, 256, 0, st>>>(W, sc);
    k_flatten_sizes<<<runs_grid, 256, 0, st>>>(W, sc);
    return cudaGetLastError();
}

// a7: resolve every local root through the merge map, component table, kept flags, K, labels
cudaError_t launch_label_largest(const roix_geom &g, uint64_t cap, void *ws, const uint64_t *map_label,
                                 const uint64_t *map_final, const uint64_t *map_total, const uint64_t *nmap, uint64_t *best,
                                 int phase, roix_scalars *sc, cudaStream_t st) {
    LabelWS W;
    carve(ws, g, cap, &W);
    const MapView M = {map_label, map_final, map_total, nmap};
    if (phase == 0) k_largest_init<<<1, 1, 0, st>>>(best);
    k_largest<<<num_sms() * 8, 256, 0, st>>>(make_geo(g), W, M, best, phase, sc);
    return cudaGetLastError();
}

cudaError_t launch_label_finish(const uint32_t *o_bits, const roix_geom &g, uint64_t min_size, uint64_t cap, void *ws,
                                const uint64_t *map_label, const uint64_t *map_final, const uint64_t *map_total,
                                const uint64_t *nmap, const roix_label_out &out, roix_scalars *sc, cudaStream_t st,
                                const uint64_t *keep) {
    LabelWS W;
    carve(ws, g, cap, &W);
    const LGeo G = make_geo(g);
    const uint64_t n = g.nz * g.ny * g.nx, nwords = (n + 31) / 32;
    const MapView M = {map_label, map_final, map_total, nmap};
    const int runs_grid = num_sms() * 8;
    cudaError_t e;
    k_root_flags<<<runs_grid, 256, 0, st>>>(G, W, M, min_size, keep, sc);
    if ((e = scan_u32_dev(W.cidx, W.cidx, W.ctr, cap, W.scan_tmp, st)) != cudaSuccess) return e;
    if (out.keep_bits && out.keep_bits != o_bits &&
        (e = cudaMemcpyAsync(out.keep_bits, o_bits, nwords * 4, cudaMemcpyDeviceToDevice, st)) != cudaSuccess)
        return e;
    k_table_clear<<<runs_grid, 256, 0, st>>>(G, W, M, W.cidx, scan_total_ptr(W.scan_tmp, cap), out, sc);
    if (out.labels) {
        if ((e = cudaMemsetAsync(out.labels, 0xff, n * 8, st)) != cudaSuccess) return e;
        k_labels<<<runs_grid, 256, 0, st>>>(G, W, M, out.labels, sc);
    }
    return cudaGetLastError();
}

cudaError_t launch_label(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom &g, uint32_t conn,
                         uint64_t min_size, uint64_t cap, void *ws, const roix_label_out &out, roix_scalars *sc,
                         cudaStream_t st, const uint2 *run_slots, uint32_t rs) {
    cudaError_t e = launch_label_local(o_bits, row_runs, g, conn, cap, ws, sc, st, run_slots, rs);
    if (e != cudaSuccess) return e;
    if (min_size == ROIX_KEEP_LARGEST) {   // both phases on this GPU; (size, label) in ctr[5], ctr[6]
        LabelWS W;
        carve(ws, g, cap, &W);
        uint64_t *best = W.ctr + 5;
        if ((e = launch_label_largest(g, cap, ws, nullptr, nullptr, nullptr, 0, best, 0, sc, st)) != cudaSuccess ||
            (e = launch_label_largest(g, cap, ws, nullptr, nullptr, nullptr, 0, best, 1, sc, st)) != cudaSuccess)
            return e;
        return launch_label_finish(o_bits, g, 0, cap, ws, nullptr, nullptr, nullptr, 0, out, sc, st, best);
    }
    return launch_label_finish(o_bits, g, min_size, cap, ws, nullptr, nullptr, nullptr, 0, out, sc, st);
}

cudaError_t launch_extract_runs(const void *x, int dtype, const roix_geom &g, uint64_t cap, void *ws, roix_scalars *sc,
                                void *codes, uint64_t capacity, const uint64_t *offset, cudaStream_t st) {
    LabelWS W;
    carve(ws, g, cap, &W);
    RunsView R;
    R.n_runs = W.ctr;
    R.x0 = W.x0;
    R.x1 = W.x1;
    R.rrow = W.rrow;
    R.parent = W.parent;
    R.kept = W.kept;
    R.err_snap = reinterpret_cast<uint32_t *>(W.ctr + 3);
    return launch_runx(x, dtype, g.nz * g.ny * g.nx, g.nx, R, cap, W.klen, W.koff, W.scan_tmp, sc, codes, capacity,
                       offset, st);
}

cudaError_t launch_label_boundary(const void *ws, const roix_geom &g, uint64_t cap, int side, roix_brun *out,
                                  uint64_t out_cap, uint64_t *count, roix_scalars *sc, cudaStream_t st) {
    LabelWS W;
    carve((void *)ws, g, cap, &W);
    k_boundary_runs<<<num_sms() * 2, 256, 0, st>>>(make_geo(g), W, side, out, out_cap, count, sc);
    return cudaGetLastError();
}

cudaError_t launch_label_link(const void *ws, const roix_geom &g, uint64_t cap, uint32_t conn, const roix_brun *prev,
                              const uint64_t *n_prev, uint64_t *pairs, uint64_t pair_cap, uint64_t *n_pairs,
                              roix_scalars *sc, cudaStream_t st) {
    LabelWS W;
    carve((void *)ws, g, cap, &W);
    cudaError_t e = cudaMemsetAsync(n_pairs, 0, 8, st);
    if (e != cudaSuccess) return e;
    k_link<<<num_sms() * 2, 256, 0, st>>>(make_geo(g), W, conn_index(conn), prev, n_prev, pairs, pair_cap, n_pairs, sc);
    return cudaGetLastError();
}

cudaError_t launch_label_boundary_roots(const void *ws, const roix_geom &g, uint64_t cap, uint64_t *labels,
                                        uint64_t *sizes, uint64_t out_cap, uint64_t *count, roix_scalars *sc,
                                        cudaStream_t st) {
    LabelWS W;
    carve((void *)ws, g, cap, &W);
    const LGeo G = make_geo(g);
    const int grid = num_sms() * 8;
    k_clear_marks<<<grid, 256, 0, st>>>(W);
    k_mark_boundary<<<grid, 256, 0, st>>>(G, W, sc);
    k_broot_flags<<<grid, 256, 0, st>>>(W);
    cudaError_t e = scan_u32_dev(W.cidx, W.cidx, W.ctr, cap, W.scan_tmp, st);
    if (e != cudaSuccess) return e;
    k_boundary_roots<<<grid, 256, 0, st>>>(G, W, scan_total_ptr(W.scan_tmp, cap), labels, sizes, out_cap, count, sc);
    return cudaGetLastError();
}
