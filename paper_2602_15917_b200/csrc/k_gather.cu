// k_gather.cu -- a1+a8 EXTRACT from the kept x-runs of a6/a7 (roix_extract_runs).
//
// The code stream is the concatenation, in run order (= increasing linear index, G-17), of the
// quantised voxels of every run whose component was kept.  So instead of scanning the kept mask K
// (N/8 bytes) and gathering x under its set bits, this path reads exactly the kept voxels of x,
// contiguously run by run, and never reads K:
//   1. k_kept_len     klen[r] = x1 - x0 if run r's component is kept, else 0
//   2. scan           koff = exclusive prefix of klen (uint64): run r's codes are [koff[r], koff[r+1])
//   3. k_chunk_first  cfirst[c] = the run holding the first code of output chunk c
//   4. k_gather       persistent CTAs over output chunks of 16 KB of x.  Producer warps (one per
//                     stage of a 4-stage shared-memory ring) read a chunk's runs and stage the kept
//                     x of each with one bulk copy (cp.async.bulk on the TMA engine, completion on
//                     the stage's mbarrier); consumer warps take groups of V = 16 / sizeof(x)
//                     consecutive codes: a group inside one run is two 16-byte shared loads, V codes
//                     quantised in registers and one 16-byte streaming store; groups across a run
//                     boundary (and the stream's ragged ends) go element by element.  Chunks
//                     touching more than GT_RBS non-empty runs take a direct element-wise path.
// Output positions are handled in the global stream space p = offset + j so that every group is
// 16-byte aligned in codes_out whatever the rank's offset.
#include "common.cuh"
#include "kernels.cuh"
#include "scan.cuh"
#include "async.cuh"

namespace roix {

template <typename T>
__host__ __device__ constexpr int gr_v() { return 16 / (int)sizeof(T); }   // elements per 16-byte group

__global__ void k_kept_len(const RunsView R, uint32_t *klen, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
        klen[i] = R.kept[R.parent[i]] ? R.x1[i] - R.x0[i] : 0u;
}

// chunk c starts at j = max(0, c * CH - a), a = offset mod V; it belongs to the run r with
// koff[r] <= j < koff[r + 1]
__global__ void k_chunk_first(const RunsView R, const uint64_t *koff, const uint64_t *offset, uint64_t ch,
                              uint32_t V, uint32_t *cfirst, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    const uint64_t a = (offset ? *offset : 0) % V;
    for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t b = koff[r], e = koff[r + 1];
        if (b == e) continue;
        if (b == 0) cfirst[0] = (uint32_t)r;
        for (uint64_t c = (b + a + ch - 1) / ch; c * ch < e + a; c++)
            if (c > 0) cfirst[c] = (uint32_t)r;
    }
}

// V consecutive elements starting at element k (0 <= k < V) of the 32 bytes {b0, b1}
template <typename T>
__device__ __forceinline__ uint4 window16(uint4 b0, uint4 b1, uint32_t k) {
    const uint32_t w[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
    const uint32_t q = sizeof(T) == 2 ? k >> 1 : k;   // whole-word shift
    uint32_t t[6], u[5];
#pragma unroll
    for (int i = 0; i < 6; i++) t[i] = (q & 2) ? w[i + 2] : w[i];
#pragma unroll
    for (int i = 0; i < 5; i++) u[i] = (q & 1) ? t[i + 1] : t[i];
    if constexpr (sizeof(T) == 2) {
        const uint32_t sh = (k & 1) * 16;
        return make_uint4(__funnelshift_r(u[0], u[1], sh), __funnelshift_r(u[1], u[2], sh),
                          __funnelshift_r(u[2], u[3], sh), __funnelshift_r(u[3], u[4], sh));
    } else {
        return make_uint4(u[0], u[1], u[2], u[3]);
    }
}

template <typename T, int QM>
__device__ __forceinline__ uint32_t code1(T v, const QP &q, uint32_t &err) {
    if constexpr (sizeof(T) == 2) return code_u16_m<QM>(v, q, err);
    else return (uint32_t)code_f32(v, q, err);
}

template <typename T, int QM>
__device__ __forceinline__ uint4 code_group(uint4 v, const QP &q, uint32_t &err) {
    if constexpr (sizeof(T) == 2) {
        return make_uint4(code_pair_u16_m<QM>(v.x, q, err), code_pair_u16_m<QM>(v.y, q, err),
                          code_pair_u16_m<QM>(v.z, q, err), code_pair_u16_m<QM>(v.w, q, err));
    } else {
        return make_uint4((uint32_t)code_f32(__uint_as_float(v.x), q, err), (uint32_t)code_f32(__uint_as_float(v.y), q, err),
                          (uint32_t)code_f32(__uint_as_float(v.z), q, err), (uint32_t)code_f32(__uint_as_float(v.w), q, err));
    }
}

constexpr int GT_CW = 8;                       // consumer warps
constexpr int GT_S = 4;                        // ring stages = producer warps (warp GT_CW + s fills stage s)
constexpr int GT_THREADS = 32 * (GT_CW + GT_S);
constexpr int GT_GPT = 4;                      // groups per consumer thread per chunk
constexpr int GT_RBS = 96;                     // non-empty runs per chunk on the bulk path
constexpr uint32_t GT_XB = 16384 + 32 * GT_RBS;   // staged x bytes per stage (alignment slack per run)

template <typename T>
__host__ __device__ constexpr uint64_t gt_ch() { return (uint64_t)32 * GT_CW * GT_GPT * gr_v<T>(); }   // 16 KB of x

struct GtStage {
    uint64_t jc, je, rb, re;   // chunk outputs [jc, je); runs rb..re touch it
    uint32_t n, slow;          // table entries; 1: direct path
};

struct GtSmem {
    uint4 x[GT_S][GT_XB / 16];
    uint32_t rlo[GT_S][GT_RBS + 1];   // entry k: outputs [jc + rlo[k], jc + rlo[k+1]) of one run
    uint32_t sidx[GT_S][GT_RBS];      // shared-memory element index of output jc + rlo[k]
    GtStage hdr[GT_S];
    uint64_t full[GT_S], empty[GT_S];
};

// largest k in [lo, hi) with a[k] <= v (a[lo] <= v < a[hi])
__device__ __forceinline__ int ufind(const uint32_t *a, int lo, int hi, uint32_t v) {
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (a[mid] <= v) lo = mid;
        else hi = mid;
    }
    return lo;
}

template <typename T, typename C, int QM>
__device__ __forceinline__ void gather_tma(const T *__restrict__ x, const RunsView &R, uint64_t nx,
                                           const uint64_t *__restrict__ koff, const uint32_t *__restrict__ cfirst,
                                           roix_scalars *sc, C *__restrict__ out, uint64_t capacity,
                                           uint64_t base_off, const QP &q, GtSmem &sm) {
    constexpr int V = gr_v<T>();
    constexpr uint64_t CH = gt_ch<T>();
    const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
    const uint64_t nruns = *R.n_runs;
    const uint64_t total = nruns ? koff[nruns] : 0;
    const uint64_t a = base_off % V;
    const uint64_t nchunks = total ? (total + a + CH - 1) / CH : 0;
    if (warp >= GT_CW) {
        // ------------------------------------------------------------------ producer of stage s
        // Chunk k+S's first 32 runs are loaded while chunk k's copies fly, and chunk k+2S's run range
        // (cfirst) one round earlier still, so issuing a chunk's copies never waits on a global load.
        const int s = (int)warp - GT_CW;
        char *xs = reinterpret_cast<char *>(sm.x[s]);
        auto chunk_of = [&](uint64_t k) { return (uint64_t)blockIdx.x + k * gridDim.x; };
        auto range = [&](uint64_t k, uint64_t &rb, uint64_t &re) {
            const uint64_t c = chunk_of(k);
            rb = re = 0;
            if (c < nchunks) {
                rb = cfirst[c];
                re = c + 1 < nchunks ? cfirst[c + 1] : nruns - 1;
            }
        };
        // per lane: run rb + lane of the prefetched chunk (koff, koff + 1, row, x0)
        struct RunPF {
            uint64_t rb, re, k0, k1;
            uint32_t row, x0;
        };
        auto runs = [&](uint64_t rb, uint64_t re, uint64_t w) {
            RunPF p;
            p.rb = rb;
            p.re = re;
            p.k0 = p.k1 = 0;
            p.row = p.x0 = 0;
            const uint64_t r = w + lane;
            if (r <= re) {
                p.k0 = koff[r];
                p.k1 = koff[r + 1];
                p.row = R.rrow[r];
                p.x0 = R.x0[r];
            }
            return p;
        };
        uint64_t rb1, re1, rb2, re2;
        range(s, rb1, re1);
        RunPF P = runs(rb1, re1, rb1);
        range(s + GT_S, rb2, re2);
        for (uint64_t k = s, i = 0;; k += GT_S, i++) {
            const uint64_t c = chunk_of(k);
            if (c >= nchunks) break;
            if (i > 0) mbar_wait(&sm.empty[s], (uint32_t)((i - 1) & 1));
            const uint64_t jc = c * CH > a ? c * CH - a : 0, je = min(total, (c + 1) * CH - a);
            const uint64_t rb = P.rb, re = P.re;
            uint32_t n = 0, cursor = 0, slow = 0;
            for (uint64_t w = rb; w <= re; w += 32) {
                const RunPF q = w == rb ? P : runs(rb, re, w);   // windows past the first: rare
                uint64_t lo = 0, hi = 0, xb = 0;
                if (w + lane <= re) {
                    lo = max(q.k0, jc);
                    hi = min(q.k1, je);
                    if (hi > lo) xb = (uint64_t)q.row * nx + q.x0 + (lo - q.k0);   // x element of output lo
                }
                const bool ne = hi > lo;
                const uint32_t bal = __ballot_sync(FULL, ne);
                if (n + __popc(bal) > (uint32_t)GT_RBS) {
                    slow = 1;
                    break;
                }
                uint32_t len = 0, b_lo = 0;
                uint64_t src = 0;
                if (ne) {
                    const uint64_t e0 = xb * sizeof(T), e1 = (xb + (hi - lo)) * sizeof(T);
                    src = e0 & ~15ull;
                    len = (uint32_t)(((e1 + 15) & ~15ull) - src);
                    b_lo = (uint32_t)(e0 - src);
                }
                const uint32_t incl = warp_incl_scan(len);
                const uint32_t tot = __shfl_sync(FULL, incl, 31);
                const uint32_t my = cursor + incl - len;
                if (ne) {
                    const uint32_t idx = n + __popc(bal & low_mask(lane));
                    sm.rlo[s][idx] = (uint32_t)(lo - jc);
                    sm.sidx[s][idx] = (my + b_lo) / (uint32_t)sizeof(T);
                }
                if (lane == 0 && tot) mbar_expect_tx(&sm.full[s], tot);
                __syncwarp();
                if (ne) bulk_g2s(xs + my, reinterpret_cast<const char *>(x) + src, len, &sm.full[s]);
                cursor += tot;
                n += __popc(bal);
            }
            if (lane == 0) {
                sm.rlo[s][slow ? 0 : n] = (uint32_t)(je - jc);
                GtStage h;
                h.jc = jc;
                h.je = je;
                h.rb = rb;
                h.re = re;
                h.n = n;
                h.slow = slow;
                sm.hdr[s] = h;
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&sm.full[s]);
            // prefetch: runs of chunk k + S (range known), range of chunk k + 2S
            P = runs(rb2, re2, rb2);
            range(k + 2 * GT_S, rb2, re2);
        }
        return;
    }
    // ---------------------------------------------------------------------- consumers
    const uint32_t t = threadIdx.x;
    uint32_t err = 0;
    if (blockIdx.x == 0 && t == 0 && base_off + total > capacity) err |= ROIX_ERR_CAPACITY;
    for (uint64_t k = 0;; k++) {
        const uint64_t c = blockIdx.x + k * gridDim.x;
        if (c >= nchunks) break;
        const int s = (int)(k % GT_S);
        mbar_wait(&sm.full[s], (uint32_t)((k / GT_S) & 1));
        const GtStage h = sm.hdr[s];
        const int64_t jc0 = (int64_t)(c * CH) - (int64_t)a;   // stream-aligned chunk origin (<= h.jc)
        if (!h.slow) {
            const uint32_t *rlo = sm.rlo[s], *sidx = sm.sidx[s];
            const T *xs = reinterpret_cast<const T *>(sm.x[s]);
            const int n = (int)h.n;
            int hint = 0;
#pragma unroll
            for (int u = 0; u < GT_GPT; u++) {
                const int64_t jg = jc0 + (int64_t)(t + u * 32 * GT_CW) * V;   // group start (16-byte aligned in out)
                const uint64_t j = jg < (int64_t)h.jc ? h.jc : (uint64_t)jg;
                if (j >= h.je) break;
                const uint32_t rj = (uint32_t)(j - h.jc);
                if (rlo[hint + 1] <= rj) hint = ufind(rlo, hint + 1, n, rj);
                const uint64_t p = base_off + (uint64_t)jg;
                const bool whole = jg >= (int64_t)h.jc && (uint64_t)jg + V <= h.je && rlo[hint + 1] >= rj + V;
                if (whole) {
                    const uint32_t si = sidx[hint] + (rj - rlo[hint]);
                    const uint32_t kk = si % V;
                    const uint4 *b = reinterpret_cast<const uint4 *>(xs + (si - kk));
                    const uint4 b0 = b[0];
                    const uint4 b1 = kk ? b[1] : b0;
                    const uint4 cv = code_group<T, QM>(window16<T>(b0, b1, kk), q, err);
                    if (p + V <= capacity) {
                        __stcs(reinterpret_cast<uint4 *>(out + p), cv);
                    } else {
                        const uint32_t cw[4] = {cv.x, cv.y, cv.z, cv.w};
#pragma unroll
                        for (int e = 0; e < V; e++) {
                            const uint32_t cd = sizeof(C) == 2 ? (cw[e >> 1] >> ((e & 1) * 16)) & 0xffffu : cw[e];
                            if (p + e < capacity) out[p + e] = (C)cd;
                        }
                    }
                } else {
                    int hh = hint;
                    for (uint64_t jj = j; jj < (uint64_t)(jg + V) && jj < h.je; jj++) {
                        const uint32_t r2 = (uint32_t)(jj - h.jc);
                        if (rlo[hh + 1] <= r2) hh = ufind(rlo, hh + 1, n, r2);
                        const uint32_t cd = code1<T, QM>(xs[sidx[hh] + (r2 - rlo[hh])], q, err);
                        if (base_off + jj < capacity) out[base_off + jj] = (C)cd;
                    }
                }
            }
        } else {
            // many short runs: element by element, binary search over the chunk's runs in koff
            for (uint64_t jj = h.jc + t; jj < h.je; jj += 32 * GT_CW) {
                uint64_t lo = h.rb, hi = h.re + 1;
                while (hi - lo > 1) {
                    const uint64_t mid = (lo + hi) >> 1;
                    if (koff[mid] <= jj) lo = mid;
                    else hi = mid;
                }
                const uint64_t v = (uint64_t)R.rrow[lo] * nx + R.x0[lo] + (jj - koff[lo]);
                const uint32_t cd = code1<T, QM>(x[v], q, err);
                if (base_off + jj < capacity) out[base_off + jj] = (C)cd;
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&sm.empty[s]);
    }
    if (err) set_err(sc, err);
}

template <typename T, typename C>
__global__ void __launch_bounds__(GT_THREADS) k_gather(const T *__restrict__ x, const RunsView R, uint64_t nx,
                                                       const uint64_t *__restrict__ koff,
                                                       const uint32_t *__restrict__ cfirst, roix_scalars *sc,
                                                       C *__restrict__ out, uint64_t capacity, const uint64_t *offset) {
    extern __shared__ uint4 gt_dyn[];
    GtSmem &sm = *reinterpret_cast<GtSmem *>(gt_dyn);
    __shared__ uint32_t skip;
    if (threadIdx.x == 0) {
        skip = get_err(sc);   // read once: other CTAs may set error bits while this one starts
        for (int s = 0; s < GT_S; s++) {
            mbar_init(&sm.full[s], 1);
            mbar_init(&sm.empty[s], GT_CW);
        }
    }
    __syncthreads();
    if (skip) return;
    const QP q = load_qp(sc);
    const uint64_t base_off = offset ? *offset : 0;
    if constexpr (sizeof(T) == 4) {
        gather_tma<T, C, QM_FLOAT>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, sm);
    } else {
        switch (qmode(q)) {
        case QM_POW2: gather_tma<T, C, QM_POW2>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, sm); break;
        case QM_INT: gather_tma<T, C, QM_INT>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, sm); break;
        case QM_ONE: gather_tma<T, C, QM_ONE>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, sm); break;
        default: gather_tma<T, C, QM_FLOAT>(x, R, nx, koff, cfirst, sc, out, capacity, base_off, q, sm); break;
        }
    }
}

__global__ void k_gather_total(const RunsView R, const uint64_t *koff, roix_scalars *sc) {
    if (get_err(sc)) return;
    const uint64_t n = *R.n_runs;
    sc->count += n ? koff[n] : 0;
}

}  // namespace roix

using namespace roix;

uint64_t gather_chunks_max(uint64_t n) { return (n + 16) / gt_ch<float>() + 2; }

template <typename T, typename C>
static cudaError_t gather_grid(int *grid) {
    const size_t smem = sizeof(GtSmem);
    cudaError_t e = cudaFuncSetAttribute(k_gather<T, C>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int occ = 0;
    if ((e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_gather<T, C>, GT_THREADS, smem)) != cudaSuccess)
        return e;
    *grid = num_sms() * (occ > 0 ? occ : 1);
    return cudaSuccess;
}

cudaError_t launch_gather(const void *x, int dtype, uint64_t nx, const RunsView &R, uint64_t cap, uint32_t *klen,
                          uint64_t *koff, uint32_t *cfirst, uint64_t *scan_tmp, roix_scalars *sc, void *codes,
                          uint64_t capacity, const uint64_t *offset, cudaStream_t st) {
    const int grid = num_sms() * 8;
    k_kept_len<<<grid, 256, 0, st>>>(R, klen, sc);
    cudaError_t e = scan_u64_dev(klen, koff, R.n_runs, cap, scan_tmp, st);
    if (e != cudaSuccess) return e;
    static int g16 = 0, g32 = 0;
    if (dtype == ROIX_U16) {
        if (!g16 && (e = gather_grid<uint16_t, uint16_t>(&g16)) != cudaSuccess) return e;
        k_chunk_first<<<grid, 256, 0, st>>>(R, koff, offset, gt_ch<uint16_t>(), gr_v<uint16_t>(), cfirst, sc);
        k_gather<uint16_t, uint16_t><<<g16, GT_THREADS, sizeof(GtSmem), st>>>(
            (const uint16_t *)x, R, nx, koff, cfirst, sc, (uint16_t *)codes, capacity, offset);
    } else {
        if (!g32 && (e = gather_grid<float, int32_t>(&g32)) != cudaSuccess) return e;
        k_chunk_first<<<grid, 256, 0, st>>>(R, koff, offset, gt_ch<float>(), gr_v<float>(), cfirst, sc);
        k_gather<float, int32_t><<<g32, GT_THREADS, sizeof(GtSmem), st>>>(
            (const float *)x, R, nx, koff, cfirst, sc, (int32_t *)codes, capacity, offset);
    }
    k_gather_total<<<1, 1, 0, st>>>(R, koff, sc);
    return cudaGetLastError();
}
