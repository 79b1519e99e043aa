// k_threshold.cu -- a3 THRESHOLD: Eq. 1 normalisation (round-half-up S:82) folded into
// a 256-bin histogram, then 2-class Otsu (k = 2 reading G-9) with exact integer scores.
//
// Otsu's criterion sigma_B^2(t) = w0 w1 (mu0 - mu1)^2 equals D(t)^2 / (N^2 n0 n1) with
// D = N s0 - n0 S (n0, s0: count and intensity sum of bins <= t; N, S: totals).  Candidates are
// compared as D_a^2 n0_b n1_b  vs  D_b^2 n0_a n1_a  in 384-bit integers, the smallest t winning ties
// (S:170), so the result is exact for any histogram with N < 2^39.
//
// NEXT-3 multi-Otsu, k = 3: thresholds t1 < t2 maximise
// sum_k w_k (mu_k - mu_T)^2 = (sum_k s_k^2 / n_k - S^2 / N) / N over the 32 385 tuples with non-empty
// classes; ties go to the lexicographically smallest (t1, t2).  Every thread scores its tuples in
// binary32 (relative error < 1e-6: three positive terms), the block keeps those within 1e-5 of the
// best approximate score, and compares them exactly: V = num / den with num = s1^2 n2 n3 + s2^2 n1 n3 +
// s3^2 n1 n2 (< 2^176) and den = n1 n2 n3 (< 2^117), cross-multiplied in 448-bit integers.
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

struct U384 {
    uint64_t w[6];
};

__device__ __forceinline__ void mul_add(uint64_t a, uint64_t b, uint64_t *acc, int pos, int len) {
    // acc[pos..] += a*b (128-bit product), carry propagated within len limbs
    uint64_t lo = a * b, hi = __umul64hi(a, b);
    uint64_t s = acc[pos] + lo;
    uint64_t c = s < lo;
    acc[pos] = s;
    if (pos + 1 >= len) return;
    uint64_t h = hi + c;  // hi <= 2^64 - 2: no overflow
    s = acc[pos + 1] + h;
    c = s < h;
    acc[pos + 1] = s;
    for (int k = pos + 2; k < len && c; k++) {
        acc[k] += 1;
        c = acc[k] == 0;
    }
}

// (a1:a0)^2 * (b1:b0), all operands 128-bit, result 384-bit
__device__ U384 sq_times(uint64_t a0, uint64_t a1, uint64_t b0, uint64_t b1) {
    uint64_t sq[4] = {0, 0, 0, 0};
    mul_add(a0, a0, sq, 0, 4);
    mul_add(a0, a1, sq, 1, 4);
    mul_add(a1, a0, sq, 1, 4);
    mul_add(a1, a1, sq, 2, 4);
    U384 r = {{0, 0, 0, 0, 0, 0}};
    for (int i = 0; i < 4; i++) {
        mul_add(sq[i], b0, r.w, i, 6);
        mul_add(sq[i], b1, r.w, i + 1, 6);
    }
    return r;
}

__device__ __forceinline__ int cmp384(const U384 &a, const U384 &b) {
    for (int i = 5; i >= 0; i--) {
        if (a.w[i] != b.w[i]) return a.w[i] > b.w[i] ? 1 : -1;
    }
    return 0;
}

struct Cand {
    uint64_t d0, d1;   // |D|
    uint64_t n0, n1;   // class counts
    int t;             // threshold, -1 = invalid
};

// is a strictly preferable to b?
__device__ bool better(const Cand &a, const Cand &b) {
    if (a.t < 0) return false;
    if (b.t < 0) return true;
    // den = n0 * n1 (< 2^78)
    uint64_t ad0 = a.n0 * a.n1, ad1 = __umul64hi(a.n0, a.n1);
    uint64_t bd0 = b.n0 * b.n1, bd1 = __umul64hi(b.n0, b.n1);
    U384 lhs = sq_times(a.d0, a.d1, bd0, bd1);
    U384 rhs = sq_times(b.d0, b.d1, ad0, ad1);
    int c = cmp384(lhs, rhs);
    return c > 0 || (c == 0 && a.t < b.t);
}

// r[0 .. na+nb) = a[0 .. na) * b[0 .. nb)
__device__ void mulw(const uint64_t *a, int na, const uint64_t *b, int nb, uint64_t *r) {
    for (int k = 0; k < na + nb; k++) r[k] = 0;
    for (int i = 0; i < na; i++)
        for (int j = 0; j < nb; j++) mul_add(a[i], b[j], r, i + j, na + nb);
}

__device__ void addw(uint64_t *acc, const uint64_t *b, int n) {
    uint64_t c = 0;
    for (int k = 0; k < n; k++) {
        const uint64_t t = acc[k] + c;
        const uint64_t c1 = t < c;
        acc[k] = t + b[k];
        c = c1 | (acc[k] < b[k]);
    }
}

struct Cand3 {
    uint64_t num[4], den[3];   // V = num / den (see frac3)
    int key;                   // t1 * 256 + t2 (lexicographic order), -1 = invalid
};

// num = s1^2 n2 n3 + s2^2 n1 n3 + s3^2 n1 n2 (< 2^176: 4 limbs), den = n1 n2 n3 (< 2^117: 3 limbs)
__device__ void frac3(const uint64_t s[3], const uint64_t n[3], Cand3 &c) {
    for (int k = 0; k < 4; k++) c.num[k] = 0;
    for (int a = 0; a < 3; a++) {
        const int b = (a + 1) % 3, d = (a + 2) % 3;
        uint64_t sq[2], nn[2], t[4];
        mulw(&s[a], 1, &s[a], 1, sq);
        mulw(&n[b], 1, &n[d], 1, nn);
        mulw(sq, 2, nn, 2, t);
        addw(c.num, t, 4);
    }
    uint64_t n12[2];
    mulw(&n[0], 1, &n[1], 1, n12);
    mulw(n12, 2, &n[2], 1, c.den);
}

__device__ bool better3(const Cand3 &a, const Cand3 &b) {
    if (a.key < 0) return false;
    if (b.key < 0) return true;
    uint64_t l[7], r[7];
    mulw(a.num, 4, b.den, 3, l);
    mulw(b.num, 4, a.den, 3, r);
    for (int k = 6; k >= 0; k--)
        if (l[k] != r[k]) return l[k] > r[k];
    return a.key < b.key;
}

__device__ __forceinline__ Cand3 shfl_cand3(const Cand3 &c, int src) {
    Cand3 o;
    for (int k = 0; k < 4; k++) o.num[k] = __shfl_sync(FULL, c.num[k], src);
    for (int k = 0; k < 3; k++) o.den[k] = __shfl_sync(FULL, c.den[k], src);
    o.key = __shfl_sync(FULL, c.key, src);
    return o;
}

// 3-class search over the inclusive prefix sums sn / ss of the norm8 histogram (totals N, S); every
// thread of the 1024-thread block calls it.  Returns (t1, t2) or (-1, -1) if fewer than three bins
// are populated.  Approximate score V(t1, t2) = A1[t1] + (ss[t2] - ss[t1])^2 / (sn[t2] - sn[t1]) +
// A3[t2] with the outer classes' terms tabulated once; the exact comparison sees only the tuples
// within the margin of the best approximate score.
__device__ void otsu3_search(const unsigned long long *h8, const uint64_t *sn, const uint64_t *ss, uint64_t N,
                             uint64_t S, int *t1_out, int *t2_out) {
    __shared__ float s_v[32], s_a1[256], s_a3[256];
    __shared__ Cand3 s_c[32];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid < 256) {
        const float n1 = (float)sn[tid], s1 = (float)ss[tid];
        const float n3 = (float)(N - sn[tid]), s3 = (float)(S - ss[tid]);
        s_a1[tid] = n1 > 0 ? s1 * s1 / n1 : 0.0f;
        s_a3[tid] = n3 > 0 ? s3 * s3 / n3 : 0.0f;
    }
    __syncthreads();
    // tuple p = t1 * 256 + t2 with non-empty classes: its approximate score, or -1.  A threshold on an
    // empty bin gives the same classes as the one below it, a lexicographically smaller tuple: only
    // populated bins are candidates (exact, and it removes the exact ties of sparse histograms).
    // binary32 scores: every term within ~5 ulps (< 1e-6 relative, all terms positive), so every tuple
    // whose exact score reaches the maximum scores within the 1e-5 margin below.
    auto score = [&](int p) -> float {
        const int t1 = p >> 8, t2 = p & 255;
        if (t1 >= t2 || t2 > 254 || h8[t1] == 0 || h8[t2] == 0) return -1.0f;
        const uint64_t n1 = sn[t1], n12 = sn[t2];
        if (n1 == 0 || n12 == n1 || n12 == N) return -1.0f;
        const float m = (float)(ss[t2] - ss[t1]);
        return s_a1[t1] + __fdividef(m * m, (float)(n12 - n1)) + s_a3[t2];
    };
    float vmax = -1.0f;
    for (int p = tid; p < 65536; p += 1024) vmax = fmaxf(vmax, score(p));
    for (int d = 16; d > 0; d >>= 1) vmax = fmaxf(vmax, __shfl_xor_sync(FULL, vmax, d));
    if (lane == 0) s_v[warp] = vmax;
    __syncthreads();
    vmax = s_v[0];
    for (int k = 1; k < 32; k++) vmax = fmaxf(vmax, s_v[k]);
    const float thr = vmax - vmax * 1e-5f;
    Cand3 best;
    best.key = -1;
    for (int k = 0; k < 4; k++) best.num[k] = 0;
    for (int k = 0; k < 3; k++) best.den[k] = 0;
    if (vmax >= 0) {
        for (int p = tid; p < 65536; p += 1024) {   // increasing p = lexicographic: strict `better` keeps the first
            if (score(p) < thr) continue;
            const int t1 = p >> 8, t2 = p & 255;
            const uint64_t n[3] = {sn[t1], sn[t2] - sn[t1], N - sn[t2]};
            const uint64_t sm[3] = {ss[t1], ss[t2] - ss[t1], S - ss[t2]};
            Cand3 c;
            frac3(sm, n, c);
            c.key = p;
            if (better3(c, best)) best = c;
        }
    }
    for (int d = 16; d > 0; d >>= 1) {
        const Cand3 o = shfl_cand3(best, lane ^ d);
        if (better3(o, best)) best = o;
    }
    if (lane == 0) s_c[warp] = best;
    __syncthreads();
    if (warp == 0) {
        best = s_c[lane];
        for (int d = 16; d > 0; d >>= 1) {
            const Cand3 o = shfl_cand3(best, lane ^ d);
            if (better3(o, best)) best = o;
        }
    }
    if (tid == 0) s_c[0] = best;
    __syncthreads();
    *t1_out = s_c[0].key < 0 ? -1 : s_c[0].key >> 8;
    *t2_out = s_c[0].key < 0 ? -1 : s_c[0].key & 255;
    __syncthreads();
}

// Exact 2-class Otsu over a 1024-thread block.  u16: hist has 65536 raw bins (I_max and the norm8
// fold are derived here); fp32: hist is the 256-bin norm8 histogram.  Returns t8 (-1 if fewer than
// two populated bins) and I_max (u16).  Every thread of the block must call it.
__device__ void otsu_block(const uint64_t *__restrict__ hist, int dtype, uint32_t *imax_out, int *t8_out,
                           int classes = 2, int *t8_hi_out = nullptr) {
    __shared__ unsigned long long h8[256];
    __shared__ uint64_t scan_n[256], scan_s[256];
    __shared__ Cand cand[256];
    __shared__ uint32_t s_imax;
    const int t = threadIdx.x;
    if (t < 256) h8[t] = 0;
    if (t == 0) s_imax = 0;
    __syncthreads();
    uint32_t imax = 1;
    if (dtype == ROIX_U16) {
        // I_max = the largest populated value (Eq. 1); 1 if none above 0
        uint32_t mymax = 0;
#pragma unroll 8
        for (int v = t; v < 65536; v += 1024)
            if (hist[v]) mymax = (uint32_t)v;
#pragma unroll
        for (int d = 16; d > 0; d >>= 1) mymax = max(mymax, __shfl_xor_sync(FULL, mymax, d));
        if (lane_id() == 0 && mymax) atomicMax(&s_imax, mymax);
        __syncthreads();
        imax = s_imax ? s_imax : 1;
        // fold: h8[norm8(v)] += hist[v], norm8(v) = round_half_up(255 v / I_max) = floor((510 v + I) / 2I)
        const uint32_t two_i = 2 * imax;
#pragma unroll 8
        for (int v = t; v <= (int)imax; v += 1024) {
            uint64_t c = hist[v];
            if (c) atomicAdd(&h8[(510u * (uint32_t)v + imax) / two_i], (unsigned long long)c);
        }
    } else if (t < 256) {
        h8[t] = hist[t];
    }
    __syncthreads();
    // threads >= 256 stay for the barriers only
    const bool act = t < 256;
    const int ti = act ? t : 255;
    // inclusive prefix sums of counts and intensity sums over bins 0..t
    if (act) {
        scan_n[t] = h8[t];
        scan_s[t] = (uint64_t)t * h8[t];
    }
    __syncthreads();
    for (int d = 1; d < 256; d <<= 1) {
        uint64_t an = (act && t >= d) ? scan_n[t - d] : 0, as = (act && t >= d) ? scan_s[t - d] : 0;
        __syncthreads();
        if (act) {
            scan_n[t] += an;
            scan_s[t] += as;
        }
        __syncthreads();
    }
    const uint64_t N = scan_n[255], S = scan_s[255];
    if (classes == 3) {
        int t1, t2;
        otsu3_search(h8, scan_n, scan_s, N, S, &t1, &t2);
        *imax_out = imax;
        *t8_out = t1;
        *t8_hi_out = t2;
        return;
    }
    Cand c;
    c.t = -1;
    c.d0 = c.d1 = c.n0 = c.n1 = 0;
    if (ti < 255 && act) {
        uint64_t n0 = scan_n[ti], s0 = scan_s[ti];
        if (n0 > 0 && n0 < N) {
            unsigned __int128 a = (unsigned __int128)N * s0, b = (unsigned __int128)n0 * S;
            unsigned __int128 d = a >= b ? a - b : b - a;
            c.d0 = (uint64_t)d;
            c.d1 = (uint64_t)(d >> 64);
            c.n0 = n0;
            c.n1 = N - n0;
            c.t = ti;
        }
    }
    if (act) cand[t] = c;
    __syncthreads();
    for (int stride = 128; stride > 0; stride >>= 1) {
        if (t < stride && better(cand[t + stride], cand[t])) cand[t] = cand[t + stride];
        __syncthreads();
    }
    *imax_out = imax;
    *t8_out = cand[0].t;
    __syncthreads();
}

__device__ __forceinline__ uint32_t thr_u16_of(uint32_t imax, int t8) {
    return (uint32_t)(((uint64_t)imax * (2 * t8 + 1) + 509) / 510);   // first v with norm8(v) > t8
}

__global__ void __launch_bounds__(1024) k_threshold(const uint64_t *__restrict__ hist, int dtype, int polarity,
                                                     int classes, roix_scalars *sc) {
    if (get_err(sc)) return;
    uint32_t imax;
    int t8, t8_hi = -1;
    otsu_block(hist, dtype, &imax, &t8, classes, &t8_hi);
    if (threadIdx.x == 0) {
        sc->polarity = (uint32_t)polarity;
        if (dtype == ROIX_U16) sc->i_max = (float)imax;
        if (t8 < 0) {
            set_err(sc, ROIX_ERR_DEGENERATE);
            sc->t8 = 0;
            sc->t8_all = 0;
            return;
        }
        // the ROI threshold: the only one (k = 2); k = 3: the lowest for HIGH, the highest for
        // LOW (G-39)
        sc->t8_all = classes == 3 ? (uint32_t)t8 | ((uint32_t)t8_hi << 8) : (uint32_t)t8;
        if (classes == 3 && polarity == ROIX_POL_LOW) t8 = t8_hi;
        sc->t8 = (uint32_t)t8;
        if (dtype == ROIX_U16) sc->thr_u16 = thr_u16_of(imax, t8);
        else sc->thr_f32 = sc->edges[t8 + 1];
    }
}

// NEXT-3 per-frame thresholds: one CTA per frame of a uint16 stack, each the whole k_threshold on its
// own 65536-bin histogram (its I_max, norm8 fold, (multi-)Otsu); results in frames[z].
__global__ void __launch_bounds__(1024) k_threshold_frames(const uint64_t *__restrict__ hist, int polarity,
                                                            int classes, roix_scalars *sc, roix_frame *frames) {
    if (get_err(sc)) return;
    const uint64_t z = blockIdx.x;
    uint32_t imax;
    int t8, t8_hi = -1;
    otsu_block(hist + z * 65536, ROIX_U16, &imax, &t8, classes, &t8_hi);
    if (threadIdx.x == 0) {
        if (z == 0) sc->polarity = (uint32_t)polarity;
        roix_frame f;
        f.i_max = imax;
        if (t8 < 0) {
            set_err(sc, ROIX_ERR_DEGENERATE);
            f.t8 = f.t8_all = 0;
            f.thr_u16 = 65536;
        } else {
            f.t8_all = classes == 3 ? (uint32_t)t8 | ((uint32_t)t8_hi << 8) : (uint32_t)t8;
            if (classes == 3 && polarity == ROIX_POL_LOW) t8 = t8_hi;
            f.t8 = (uint32_t)t8;
            f.thr_u16 = thr_u16_of(imax, t8);
        }
        frames[z] = f;
    }
}

// Speculative threshold window from a sample histogram (roix_histogram_binarize): the exact raw
// threshold is expected within [spec_lo, spec_hi] -- Otsu on the sample +- SPEC_D norm8 bins, and for
// u16 an I_max up to 1/8 above the sample maximum.  spec_state = 1 (window set) or 3 (no window).
constexpr int SPEC_D = 3;
__global__ void __launch_bounds__(1024) k_spec(const uint64_t *__restrict__ shist, int dtype, int polarity,
                                                roix_scalars *sc) {
    if (get_err(sc)) return;
    uint32_t imax;
    int t8;
    otsu_block(shist, dtype, &imax, &t8);
    if (threadIdx.x == 0) {
        sc->polarity = (uint32_t)polarity;
        sc->n_uncertain = 0;
        if (t8 < 0) {
            sc->spec_state = 3;
            return;
        }
        const int tlo = max(t8 - SPEC_D, 0), thi = min(t8 + SPEC_D, 254);
        if (dtype == ROIX_U16) {
            const uint32_t ihi = min(65535u, imax + imax / 8 + 64);
            sc->spec_lo = thr_u16_of(imax, tlo);
            sc->spec_hi = thr_u16_of(ihi, thi);
        } else {
            sc->spec_lo = __float_as_uint(sc->edges[tlo + 1]);
            sc->spec_hi = __float_as_uint(sc->edges[thi + 1]);
        }
        sc->spec_state = 1;
    }
}

}  // namespace roix

cudaError_t launch_threshold(const uint64_t *hist, int dtype, int polarity, roix_scalars *sc, cudaStream_t st,
                             int classes) {
    roix::k_threshold<<<1, 1024, 0, st>>>(hist, dtype, polarity, classes, sc);
    return cudaGetLastError();
}

cudaError_t launch_threshold_frames(const uint64_t *hist, uint64_t nframes, int polarity, int classes,
                                    roix_scalars *sc, roix_frame *frames, cudaStream_t st) {
    for (uint64_t z0 = 0; z0 < nframes; z0 += 65535) {
        const unsigned nz = (unsigned)min(nframes - z0, (uint64_t)65535);
        roix::k_threshold_frames<<<nz, 1024, 0, st>>>(hist + z0 * 65536, polarity, classes, sc, frames + z0);
    }
    return cudaGetLastError();
}

cudaError_t launch_spec(const uint64_t *shist, int dtype, int polarity, roix_scalars *sc, cudaStream_t st) {
    roix::k_spec<<<1, 1024, 0, st>>>(shist, dtype, polarity, sc);
    return cudaGetLastError();
}
