/*
 * roix_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * A plain, slow, single-threaded CPU statement of what the ROIX hot path computes.  It exists to
 * prove the CUDA path right: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * `--impl reference` legs may load it.  It shares no code, header, table or constant with the
 * product library (paper_2602_15917_b200/csrc); neither side includes the other.
 *
 * Citations: P:n = /root/reference/PAPER.md line n, S:n = SPEC.md line n, G-n = a reading
 * recorded in DESIGN.md §3 (and SURVEY.md §8c).  Build: gcc -O2 -ffp-contract=off (no fast-math)
 * so every floating-point expression below is evaluated exactly as written, in IEEE binary64.
 *
 * Every function is the plain definition written out: one loop over the voxels in linear-index
 * order i = (z*Y + y)*X + x, no blocking, no fusion.  Volumes are Z x Y x X, x fastest.
 * Masks are one byte per voxel (0/1); bit-packing is done by the Python side with numpy.
 *
 * Status codes returned: 0 = ok, 1 = value/quotient outside the quantiser's range (G-4, G-7),
 * 2 = non-finite input (G-32), 3 = capacity exceeded.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define OR_OK 0
#define OR_RANGE 1
#define OR_NONFINITE 2
#define OR_CAPACITY 3

/* ---------------------------------------------------------------------------------------------
 * a1 QUANTISE (BJ.north_star "code = round(x / 2eb), round-half-even"; G-1..G-4, G-7).
 * Definition: code = the integer nearest to the exact real quotient x / s, s = fl32(2*eb), ties to
 * the even integer.  Written out with exact binary64 arithmetic: x and s are binary32 values, so
 * k*s (|k| < 2^24) and (2k+1)*s are exact products in binary64, and 2x is exact.
 * Validity range (G-4): |x| >= 2^23 * s is rejected (status OR_RANGE) -- the same predicate the
 * paper-independent reading fixes for both sides.
 * ------------------------------------------------------------------------------------------- */
static int rne_exact(double x, double s, double *code)
{
    if (!(fabs(x) < 8388608.0 * s)) return OR_RANGE; /* also catches NaN */
    double k = floor(x / s);                          /* a first guess, then made exact: */
    while (k * s > x) k -= 1.0;                       /*   k*s <= x            */
    while ((k + 1.0) * s <= x) k += 1.0;              /*   x < (k+1)*s         */
    double twice = 2.0 * x, mid = (2.0 * k + 1.0) * s;
    if (twice > mid) *code = k + 1.0;                 /* above the half-way point */
    else if (twice < mid) *code = k;                  /* below it */
    else *code = (fmod(k, 2.0) == 0.0) ? k : k + 1.0; /* exactly half-way: the even one */
    return OR_OK;
}

/* s = fl32(2 * eb): doubling a binary32 is exact unless it overflows. */
static int step_of(float eb, double *s)
{
    float s32 = 2.0f * eb;
    if (!(eb > 0.0f) || !isfinite(s32)) return OR_RANGE;
    *s = (double)s32;
    return OR_OK;
}

int oracle_quantize_u16(const uint16_t *x, uint64_t n, float eb, uint16_t *codes)
{
    double s, c;
    if (step_of(eb, &s)) return OR_RANGE;
    for (uint64_t i = 0; i < n; i++) {
        if (rne_exact((double)x[i], s, &c)) return OR_RANGE;
        if (c > 65535.0) return OR_RANGE; /* u16 codes (G-7) */
        codes[i] = (uint16_t)c;
    }
    return OR_OK;
}

int oracle_quantize_f32(const float *x, uint64_t n, float eb, int32_t *codes)
{
    double s, c;
    if (step_of(eb, &s)) return OR_RANGE;
    for (uint64_t i = 0; i < n; i++) {
        if (!isfinite(x[i])) return OR_NONFINITE;
        if (rne_exact((double)x[i], s, &c)) return OR_RANGE;
        codes[i] = (int32_t)c;
    }
    return OR_OK;
}

/* ---------------------------------------------------------------------------------------------
 * a0 RANGE (fp32 only; G-6): min and max over all voxels, non-finite rejected (G-32).
 * Relative eb (G-6, SZ value-range convention): eb_abs = fl32(rel * (fl64(max) - fl64(min))).
 * ------------------------------------------------------------------------------------------- */
int oracle_range_f32(const float *x, uint64_t n, float *mn, float *mx)
{
    float lo = INFINITY, hi = -INFINITY;
    for (uint64_t i = 0; i < n; i++) {
        if (!isfinite(x[i])) return OR_NONFINITE;
        if (x[i] < lo) lo = x[i];
        if (x[i] > hi) hi = x[i];
    }
    *mn = lo;
    *mx = hi;
    return OR_OK;
}

float oracle_resolve_eb(float mn, float mx, double rel)
{
    return (float)(rel * ((double)mx - (double)mn));
}

/* ---------------------------------------------------------------------------------------------
 * a2 HISTOGRAM ("based on intensity distribution"; bin[v] = count of v).
 * uint16: 65 536 raw bins, accumulated (+=) so slabs can be summed.
 * ------------------------------------------------------------------------------------------- */
void oracle_hist_u16(const uint16_t *x, uint64_t n, uint64_t *h)
{
    for (uint64_t i = 0; i < n; i++) h[x[i]] += 1;
}

/* I_max (Eq. 1, "the maximum pixel intensity"; 1 if the image is all-zero). */
uint32_t oracle_imax_u16(const uint64_t *h)
{
    for (int v = 65535; v > 0; v--)
        if (h[v]) return (uint32_t)v;
    return 1;
}

/* Eq. 1 with round-half-up: norm8(v) = round_half_up(255 v / I_max).
 * For integers, round_half_up(a/b) = floor((2a + b) / 2b) with a = 255 v, b = I_max. */
uint32_t oracle_norm8_u16(uint32_t v, uint32_t imax)
{
    uint64_t a = 255ull * v, b = imax;
    uint64_t r = (2 * a + b) / (2 * b);
    return r > 255 ? 255 : (uint32_t)r;
}

/* fp32 input, G-30: norm8(x) = clamp(floor(fl64(fl64(x) * 255 / fl64(I_max)) + 0.5), 0, 255). */
uint32_t oracle_norm8_f32(float x, float imax)
{
    double q = ((double)x * 255.0) / (double)imax;
    double r = floor(q + 0.5);
    if (!(r > 0.0)) return 0;
    if (r > 255.0) return 255;
    return (uint32_t)r;
}

/* The 256-bin histogram of norm8 values that Otsu runs on. */
void oracle_hist8_from_u16(const uint64_t *h, uint32_t imax, uint64_t *h8)
{
    memset(h8, 0, 256 * sizeof(uint64_t));
    for (uint32_t v = 0; v < 65536; v++) h8[oracle_norm8_u16(v, imax)] += h[v];
}

void oracle_hist8_f32(const float *x, uint64_t n, float imax, uint64_t *h8)
{
    for (uint64_t i = 0; i < n; i++) h8[oracle_norm8_f32(x[i], imax)] += 1;
}

/* ---------------------------------------------------------------------------------------------
 * a4 BINARISE (Eq. 2; "bit = 1 iff pixel > threshold"), evaluated per voxel on
 * the normalised intensity.  polarity 0 = HIGH (norm8 > t8), 1 = LOW (norm8 <= t8; G-10).
 * ------------------------------------------------------------------------------------------- */
void oracle_binarize_u16(const uint16_t *x, uint64_t n, uint32_t imax, uint32_t t8, int polarity, uint8_t *m)
{
    for (uint64_t i = 0; i < n; i++) {
        uint32_t k = oracle_norm8_u16(x[i], imax);
        m[i] = polarity ? (k <= t8) : (k > t8);
    }
}

void oracle_binarize_f32(const float *x, uint64_t n, float imax, uint32_t t8, int polarity, uint8_t *m)
{
    for (uint64_t i = 0; i < n; i++) {
        uint32_t k = oracle_norm8_f32(x[i], imax);
        m[i] = polarity ? (k <= t8) : (k > t8);
    }
}

/* ---------------------------------------------------------------------------------------------
 * a5 MORPHOLOGICAL CLEANUP (G-11): one opening, o = dilate(erode(m)), cross structuring element
 * of radius 1: se = 6 -> the 6 face neighbours in 3-D; se = 4 -> the 4 in-plane neighbours.
 * Out-of-volume neighbours are ignored (erosion: treated as 1; dilation: treated as 0).
 *   e_i = m_i AND (AND over j in SE(i) inside the volume of m_j)
 *   o_i = e_i OR  (OR  over j in SE(i) inside the volume of e_j)
 * ------------------------------------------------------------------------------------------- */
static const int SE6[6][3] = {{-1, 0, 0}, {1, 0, 0}, {0, -1, 0}, {0, 1, 0}, {0, 0, -1}, {0, 0, 1}};

static int se_count(int se) { return se == 6 ? 6 : 4; } /* se 4: the y/x entries of SE6 only */
static const int *se_off(int se, int k) { return se == 6 ? SE6[k] : SE6[k + 2]; }

int oracle_open(const uint8_t *m, int64_t Z, int64_t Y, int64_t X, int se, uint8_t *o)
{
    if (se != 6 && se != 4) return OR_RANGE;
    uint64_t n = (uint64_t)(Z * Y * X);
    uint8_t *e = (uint8_t *)malloc(n ? n : 1);
    if (!e) return OR_CAPACITY;
    for (int64_t z = 0; z < Z; z++)
        for (int64_t y = 0; y < Y; y++)
            for (int64_t x = 0; x < X; x++) {
                uint64_t i = (uint64_t)((z * Y + y) * X + x);
                uint8_t v = m[i];
                for (int k = 0; k < se_count(se); k++) {
                    const int *d = se_off(se, k);
                    int64_t zz = z + d[0], yy = y + d[1], xx = x + d[2];
                    if (zz < 0 || zz >= Z || yy < 0 || yy >= Y || xx < 0 || xx >= X) continue;
                    v &= m[(zz * Y + yy) * X + xx];
                }
                e[i] = v;
            }
    for (int64_t z = 0; z < Z; z++)
        for (int64_t y = 0; y < Y; y++)
            for (int64_t x = 0; x < X; x++) {
                uint64_t i = (uint64_t)((z * Y + y) * X + x);
                uint8_t v = e[i];
                for (int k = 0; k < se_count(se); k++) {
                    const int *d = se_off(se, k);
                    int64_t zz = z + d[0], yy = y + d[1], xx = x + d[2];
                    if (zz < 0 || zz >= Z || yy < 0 || yy >= Y || xx < 0 || xx >= X) continue;
                    v |= e[(zz * Y + yy) * X + xx];
                }
                o[i] = v;
            }
    free(e);
    return OR_OK;
}

/* ---------------------------------------------------------------------------------------------
 * a6 CONNECTED COMPONENTS (BJ "3-D connected-component labelling"; G-14): breadth-first flood
 * fill from seeds taken in raster (linear-index) order.  A seed is the first voxel of its
 * component met in that order, i.e. the component's minimum linear index -- the canonical label.
 * conn: 6 / 18 / 26 (3-D neighbourhoods), 4 / 8 (in-plane, per z-plane).
 * Outputs: comp[i] = ordinal of i's component in min-index order (UINT32_MAX for background),
 * comp_min[c], comp_size[c]; returns the component count, or -1 on bad conn / capacity.
 * ------------------------------------------------------------------------------------------- */
static int neighbour_ok(int conn, int dz, int dy, int dx)
{
    int k = abs(dz) + abs(dy) + abs(dx);
    if (k == 0) return 0;
    switch (conn) {
    case 6: return k == 1;
    case 18: return k <= 2;
    case 26: return 1;
    case 4: return dz == 0 && k == 1;
    case 8: return dz == 0;
    default: return 0;
    }
}

int64_t oracle_label(const uint8_t *o, int64_t Z, int64_t Y, int64_t X, int conn, uint32_t *comp,
                     uint64_t *comp_min, uint64_t *comp_size, uint64_t cap)
{
    if (conn != 4 && conn != 6 && conn != 8 && conn != 18 && conn != 26) return -1;
    uint64_t n = (uint64_t)(Z * Y * X);
    int offs[26][3], noff = 0;
    for (int dz = -1; dz <= 1; dz++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++)
                if (neighbour_ok(conn, dz, dy, dx)) {
                    offs[noff][0] = dz;
                    offs[noff][1] = dy;
                    offs[noff][2] = dx;
                    noff++;
                }
    for (uint64_t i = 0; i < n; i++) comp[i] = UINT32_MAX;
    uint64_t *queue = (uint64_t *)malloc((n ? n : 1) * sizeof(uint64_t));
    if (!queue) return -1;
    int64_t nc = 0;
    for (uint64_t seed = 0; seed < n; seed++) {
        if (!o[seed] || comp[seed] != UINT32_MAX) continue;
        if ((uint64_t)nc >= cap) { free(queue); return -1; }
        uint64_t head = 0, tail = 0, size = 0;
        comp[seed] = (uint32_t)nc;
        queue[tail++] = seed;
        while (head < tail) {
            uint64_t i = queue[head++];
            size++;
            int64_t x = (int64_t)(i % (uint64_t)X), y = (int64_t)((i / (uint64_t)X) % (uint64_t)Y),
                    z = (int64_t)(i / ((uint64_t)X * (uint64_t)Y));
            for (int k = 0; k < noff; k++) {
                int64_t zz = z + offs[k][0], yy = y + offs[k][1], xx = x + offs[k][2];
                if (zz < 0 || zz >= Z || yy < 0 || yy >= Y || xx < 0 || xx >= X) continue;
                uint64_t j = (uint64_t)((zz * Y + yy) * X + xx);
                if (o[j] && comp[j] == UINT32_MAX) {
                    comp[j] = (uint32_t)nc;
                    queue[tail++] = j;
                }
            }
        }
        comp_min[nc] = seed;
        comp_size[nc] = size;
        nc++;
    }
    free(queue);
    return nc;
}

/* ---------------------------------------------------------------------------------------------
 * a7 FILTER + a8 EXTRACT (BJ "small-object removal", "stream compaction of the retained ROI
 * voxels into a dense code stream"; G-13, G-17): kept(c) = size(c) >= min_size; K_i = 1 iff i is
 * in a kept component; stream = codes of the voxels with K_i = 1 in increasing i.
 * ------------------------------------------------------------------------------------------- */
void oracle_filter(const uint32_t *comp, uint64_t n, const uint64_t *comp_size, uint64_t ncomp,
                   uint64_t min_size, uint8_t *kept, uint8_t *K)
{
    for (uint64_t c = 0; c < ncomp; c++) kept[c] = comp_size[c] >= min_size;
    for (uint64_t i = 0; i < n; i++) K[i] = comp[i] != UINT32_MAX && kept[comp[i]];
}

int64_t oracle_extract_u16(const uint16_t *x, const uint8_t *K, uint64_t n, float eb, uint16_t *stream)
{
    double s, c;
    int64_t j = 0;
    if (step_of(eb, &s)) return -1;
    for (uint64_t i = 0; i < n; i++) {
        if (!K[i]) continue;
        if (rne_exact((double)x[i], s, &c) || c > 65535.0) return -1;
        stream[j++] = (uint16_t)c;
    }
    return j;
}

int64_t oracle_extract_f32(const float *x, const uint8_t *K, uint64_t n, float eb, int32_t *stream)
{
    double s, c;
    int64_t j = 0;
    if (step_of(eb, &s)) return -1;
    for (uint64_t i = 0; i < n; i++) {
        if (!K[i]) continue;
        if (!isfinite(x[i]) || rne_exact((double)x[i], s, &c)) return -1;
        stream[j++] = (int32_t)c;
    }
    return j;
}

/* ------------------------------------------------------------------ NEXT-1: row spans
 * The paper's ROI representation: for every row i = z*Y + y of K holding a set bit, the
 * geometry record G(i) = [i, x_start, x_end] with x_start the leftmost and x_end the rightmost set
 * column + 1 (exclusive: n_i = x_end - x_start, S DESIGN DECISIONS), and the pixel section
 * P(i) = [p_0 .. p_{n_i - 1}], p_j the value at column x_start + j -- interior gaps included --
 * here quantised with the a1 quantiser.  spans: 3 int64 per record, in increasing i; returns the
 * number of records and writes the total section length to *ncodes; -1 on a quantiser range error.
 */
int64_t oracle_row_spans(const uint8_t *K, const void *x, int is_f32, int64_t Z, int64_t Y, int64_t X, float eb,
                         int64_t *spans, void *codes, int64_t *ncodes)
{
    double s, c;
    int64_t m = 0, nc = 0;
    if (step_of(eb, &s)) return -1;
    for (int64_t i = 0; i < Z * Y; i++) {
        const uint8_t *row = K + i * X;
        int64_t x0 = -1, x1 = -1;
        for (int64_t xx = 0; xx < X; xx++)
            if (row[xx]) {
                if (x0 < 0) x0 = xx;
                x1 = xx + 1;
            }
        if (x0 < 0) continue;
        spans[3 * m] = i;
        spans[3 * m + 1] = x0;
        spans[3 * m + 2] = x1;
        m++;
        for (int64_t xx = x0; xx < x1; xx++) {
            if (is_f32) {
                const float v = ((const float *)x)[i * X + xx];
                if (!isfinite(v) || rne_exact((double)v, s, &c)) return -1;
                ((int32_t *)codes)[nc++] = (int32_t)c;
            } else {
                const uint16_t v = ((const uint16_t *)x)[i * X + xx];
                if (rne_exact((double)v, s, &c) || c > 65535.0) return -1;
                ((uint16_t *)codes)[nc++] = (uint16_t)c;
            }
        }
    }
    *ncodes = nc;
    return m;
}

/* ----------------------------------------------- NEXT-2: greedy absolute-error-bounded quantiser
 * PAPER.md §4.2.3 Steps 1-5, literally: l = -inf, u = +inf, head = 0; for each i the
 * intersection [max(l, D[i] - E), min(u, D[i] + E)]; when it is empty the group [head, i) gets
 * Q = floor((u + l) / 2) and a new group starts at i with [D[i] - E, D[i] + E]; the final group
 * likewise; Q clipped to [0, qmax] (Step 5: 255 for 8-bit data; 65535 here for 16-bit data).
 * E >= 0 (S:299 admits 0); group_start[i] = 1 where a group begins.  Returns the group count. */
int64_t oracle_greedy_quantize(const uint16_t *D, uint64_t m, double E, uint32_t qmax, uint16_t *Q, uint8_t *group_start)
{
    double l = -INFINITY, u = INFINITY;
    uint64_t head = 0;
    int64_t groups = 0;
    for (uint64_t i = 0; i < m; i++) {
        const double lo = (double)D[i] - E, hi = (double)D[i] + E;
        const double ln = l > lo ? l : lo, un = u < hi ? u : hi;
        group_start[i] = 0;
        if (un < ln) {
            double q = floor((u + l) / 2.0);
            if (q < 0) q = 0;
            if (q > qmax) q = qmax;
            for (uint64_t j = head; j < i; j++) Q[j] = (uint16_t)q;
            l = lo;
            u = hi;
            head = i;
            group_start[i] = 1;
            groups++;
        } else {
            l = ln;
            u = un;
        }
        if (i == 0) {
            group_start[0] = 1;
            groups++;
        }
    }
    if (m) {
        double q = floor((u + l) / 2.0);
        if (q < 0) q = 0;
        if (q > qmax) q = qmax;
        for (uint64_t j = head; j < m; j++) Q[j] = (uint16_t)q;
    }
    return groups;
}

/* =============================================================================================
 * STREAMING MODE -- the same definitions for volumes too large to hold: the
 * full-size C3 / C4 / C5 configs (17-34 G voxels, 34-69 GB of uint16).  The caller feeds the volume
 * plane by plane, in increasing z, once per pass; memory is O(plane) plus O(runs of o).
 *
 *   Pass A (os_hist):     oracle_hist_u16 over every plane -> h, then (caller) I_max, h8, Otsu.
 *   Pass B (os_feed):     per plane, m = oracle_binarize_u16 (Eq. 2 on norm8); the
 *                         opening by its definition (G-11, as oracle_open, written per plane with
 *                         rings of 3 planes of m and e); every finished plane of o labelled by the
 *                         classical two-pass raster scan (Rosenfeld & Pfaltz 1966): a foreground
 *                         voxel takes the provisional label of its already-visited neighbours
 *                         (left neighbour first) and the others are united with it; a voxel without
 *                         one opens a new label.  Labels are numbered in raster order and union
 *                         keeps the smaller, so every root is the label its component opened first,
 *                         at the component's minimum linear index (G-14).  The labels of a plane are
 *                         kept as x-runs (row, x0, x1, label): left-first labelling gives every
 *                         voxel of an x-run the same label.
 *   Resolve (os_resolve): roots, component sizes, the table in increasing minimum index, kept =
 *                         size >= min_size (G-13).
 *   Pass C (os_extract):  per plane, K (voxels of runs whose root is kept) and the stream of
 *                         codes = rne_exact(x / s) (a1) in increasing linear index (a8, G-17).
 * ------------------------------------------------------------------------------------------- */
typedef struct {
    uint32_t y, x0, x1, pad;
    uint64_t label;
} os_run;

typedef struct {
    int64_t Z, Y, X;
    int conn, se, polarity;
    uint32_t imax, t8;
    int64_t fed;           /* pass B: planes fed so far */
    uint8_t *m[3], *e[3];  /* rings: plane q lives in slot q % 3 */
    uint8_t *o, *o_prev;   /* the plane of o being labelled, and the plane before it */
    uint64_t *lab_prev, *lab_cur;
    uint64_t *parent, *first, *size;  /* per provisional label */
    uint64_t nlab, cap_lab;
    os_run *runs;
    uint64_t nruns, cap_runs;
    uint64_t *plane_run0;  /* [Z + 1]: first run of every plane */
    /* after os_resolve */
    uint64_t *root_size;   /* per label: the component size, at roots */
    uint64_t ncomp;
    uint64_t min_size;
    uint8_t *kept_root;    /* per label: kept flag, at roots */
} os_state;

void os_free(os_state *s)
{
    if (!s) return;
    for (int k = 0; k < 3; k++) {
        free(s->m[k]);
        free(s->e[k]);
    }
    free(s->o);
    free(s->o_prev);
    free(s->lab_prev);
    free(s->lab_cur);
    free(s->parent);
    free(s->first);
    free(s->size);
    free(s->runs);
    free(s->plane_run0);
    free(s->root_size);
    free(s->kept_root);
    free(s);
}

os_state *os_create(int64_t Z, int64_t Y, int64_t X, int conn, int se, int polarity, uint32_t imax, uint32_t t8)
{
    if (conn != 4 && conn != 6 && conn != 8 && conn != 18 && conn != 26) return NULL;
    if (se != 6 && se != 4) return NULL;
    os_state *s = (os_state *)calloc(1, sizeof(os_state));
    if (!s) return NULL;
    s->Z = Z;
    s->Y = Y;
    s->X = X;
    s->conn = conn;
    s->se = se;
    s->polarity = polarity;
    s->imax = imax;
    s->t8 = t8;
    size_t A = (size_t)(Y * X);
    int ok = 1;
    for (int k = 0; k < 3; k++) {
        s->m[k] = (uint8_t *)malloc(A);
        s->e[k] = (uint8_t *)malloc(A);
        ok &= s->m[k] && s->e[k];
    }
    s->o = (uint8_t *)malloc(A);
    s->o_prev = (uint8_t *)malloc(A);
    s->lab_prev = (uint64_t *)malloc(A * sizeof(uint64_t));
    s->lab_cur = (uint64_t *)malloc(A * sizeof(uint64_t));
    s->plane_run0 = (uint64_t *)calloc((size_t)Z + 1, sizeof(uint64_t));
    ok &= s->o && s->o_prev && s->lab_prev && s->lab_cur && s->plane_run0;
    if (!ok) {
        os_free(s);
        return NULL;
    }
    return s;
}

/* m, e of plane q (ring slot q % 3); only called for planes inside the volume */
static uint8_t os_m(const os_state *s, int64_t q, int64_t y, int64_t x) { return s->m[q % 3][y * s->X + x]; }
static uint8_t os_e(const os_state *s, int64_t q, int64_t y, int64_t x) { return s->e[q % 3][y * s->X + x]; }

/* erosion of plane q: e = m AND (AND of m over the SE neighbours inside the volume) -- oracle_open */
static void os_erode(os_state *s, int64_t q)
{
    uint8_t *e = s->e[q % 3];
    for (int64_t y = 0; y < s->Y; y++)
        for (int64_t x = 0; x < s->X; x++) {
            uint8_t v = os_m(s, q, y, x);
            for (int k = 0; k < se_count(s->se); k++) {
                const int *d = se_off(s->se, k);
                int64_t zz = q + d[0], yy = y + d[1], xx = x + d[2];
                if (zz < 0 || zz >= s->Z || yy < 0 || yy >= s->Y || xx < 0 || xx >= s->X) continue;
                v &= os_m(s, zz, yy, xx);
            }
            e[y * s->X + x] = v;
        }
}

/* dilation of plane q into s->o: o = e OR (OR of e over the SE neighbours inside the volume) */
static void os_dilate(os_state *s, int64_t q)
{
    for (int64_t y = 0; y < s->Y; y++)
        for (int64_t x = 0; x < s->X; x++) {
            uint8_t v = os_e(s, q, y, x);
            for (int k = 0; k < se_count(s->se); k++) {
                const int *d = se_off(s->se, k);
                int64_t zz = q + d[0], yy = y + d[1], xx = x + d[2];
                if (zz < 0 || zz >= s->Z || yy < 0 || yy >= s->Y || xx < 0 || xx >= s->X) continue;
                v |= os_e(s, zz, yy, xx);
            }
            s->o[y * s->X + x] = v;
        }
}

static uint64_t os_find(os_state *s, uint64_t a)
{
    while (s->parent[a] != a) {
        s->parent[a] = s->parent[s->parent[a]]; /* path halving */
        a = s->parent[a];
    }
    return a;
}

static void os_union(os_state *s, uint64_t a, uint64_t b)
{
    a = os_find(s, a);
    b = os_find(s, b);
    if (a < b) s->parent[b] = a;
    else if (b < a) s->parent[a] = b;
}

static int os_grow(void **p, uint64_t *cap, uint64_t need, size_t elem)
{
    if (need <= *cap) return 1;
    uint64_t c = *cap ? *cap : 1024;
    while (c < need) c *= 2;
    void *q = realloc(*p, c * elem);
    if (!q) return 0;
    *p = q;
    *cap = c;
    return 1;
}

/* label plane q of o (s->o); lab_prev holds the labels of plane q-1 (valid where o(q-1) = 1) */
static int os_label_plane(os_state *s, int64_t q)
{
    const int64_t Y = s->Y, X = s->X;
    /* the already-visited half of the neighbourhood, left neighbour first */
    int offs[13][3], noff = 0;
    offs[noff][0] = 0;
    offs[noff][1] = 0;
    offs[noff][2] = -1;
    noff++;
    for (int dz = -1; dz <= 0; dz++)
        for (int dy = -1; dy <= 1; dy++)
            for (int dx = -1; dx <= 1; dx++) {
                if (dz == 0 && dy >= 0) continue; /* (0, 0, -1) is first; (0, 0, >=0) and (0, 1, *) come later */
                if (neighbour_ok(s->conn, dz, dy, dx)) {
                    offs[noff][0] = dz;
                    offs[noff][1] = dy;
                    offs[noff][2] = dx;
                    noff++;
                }
            }
    if (!neighbour_ok(s->conn, 0, 0, -1)) return -1; /* every supported conn has the x-neighbour */
    s->plane_run0[q] = s->nruns;
    for (int64_t y = 0; y < Y; y++)
        for (int64_t x = 0; x < X; x++) {
            const int64_t a = y * X + x;
            if (!s->o[a]) continue;
            uint64_t L = UINT64_MAX;
            for (int k = 0; k < noff; k++) {
                int64_t zz = q + offs[k][0], yy = y + offs[k][1], xx = x + offs[k][2];
                if (zz < 0 || yy < 0 || yy >= Y || xx < 0 || xx >= X) continue;
                const int64_t b = yy * X + xx;
                uint64_t l2;
                if (zz == q) {
                    if (!s->o[b]) continue;
                    l2 = s->lab_cur[b];
                } else {
                    if (!s->o_prev[b]) continue;
                    l2 = s->lab_prev[b];
                }
                if (L == UINT64_MAX) L = l2;
                else os_union(s, L, l2);
            }
            if (L == UINT64_MAX) { /* a new provisional label */
                if (s->nlab == s->cap_lab) {
                    uint64_t c = s->cap_lab ? 2 * s->cap_lab : 1024, *a1, *a2, *a3;
                    a1 = (uint64_t *)realloc(s->parent, c * sizeof(uint64_t));
                    if (a1) s->parent = a1;
                    a2 = (uint64_t *)realloc(s->first, c * sizeof(uint64_t));
                    if (a2) s->first = a2;
                    a3 = (uint64_t *)realloc(s->size, c * sizeof(uint64_t));
                    if (a3) s->size = a3;
                    if (!a1 || !a2 || !a3) return -1;
                    s->cap_lab = c;
                }
                L = s->nlab++;
                s->parent[L] = L;
                s->first[L] = (uint64_t)((q * Y + y) * X + x);
                s->size[L] = 0;
            }
            s->lab_cur[a] = L;
            s->size[L] += 1;
            /* x-runs of equal label (left-first labelling: one label per x-run) */
            if (x > 0 && s->o[a - 1] && s->runs[s->nruns - 1].label == L && s->runs[s->nruns - 1].x1 == (uint32_t)x &&
                s->runs[s->nruns - 1].y == (uint32_t)y) {
                s->runs[s->nruns - 1].x1 = (uint32_t)x + 1;
            } else {
                if (!os_grow((void **)&s->runs, &s->cap_runs, s->nruns + 1, sizeof(os_run))) return -1;
                os_run r = {(uint32_t)y, (uint32_t)x, (uint32_t)x + 1, 0, L};
                s->runs[s->nruns++] = r;
            }
        }
    s->plane_run0[q + 1] = s->nruns;
    return 0;
}

/* after labelling plane q: it becomes the previous plane */
static void os_shift_planes(os_state *s)
{
    uint8_t *t = s->o_prev;
    s->o_prev = s->o;
    s->o = t;
    uint64_t *u = s->lab_prev;
    s->lab_prev = s->lab_cur;
    s->lab_cur = u;
}

/* o of plane q is ready in s->o: optionally copied out, then labelled */
static int os_emit(os_state *s, int64_t q, uint8_t *o_out, int64_t *n_out)
{
    if (o_out) memcpy(o_out + (size_t)(*n_out) * (size_t)(s->Y * s->X), s->o, (size_t)(s->Y * s->X));
    (*n_out)++;
    if (os_label_plane(s, q)) return -1;
    os_shift_planes(s);
    return 0;
}

/* Pass B: feed plane p = s->fed (x: Y*X uint16).  Every plane of o finished by this call is
 * written to o_out (room for 3 planes) and labelled; returns their number, -1 on failure.  With
 * x == NULL the call ends the volume (after all Z planes) and finishes the remaining planes. */
int64_t os_feed(os_state *s, const uint16_t *x, uint8_t *o_out)
{
    int64_t n_out = 0;
    const int64_t A = s->Y * s->X;
    if (x) {
        const int64_t p = s->fed;
        if (p >= s->Z) return -1;
        oracle_binarize_u16(x, (uint64_t)A, s->imax, s->t8, s->polarity, s->m[p % 3]);
        s->fed++;
        if (s->se == 4) { /* in-plane SE: every plane is opened on its own */
            os_erode(s, p);
            os_dilate(s, p);
            if (os_emit(s, p, o_out, &n_out)) return -1;
            return n_out;
        }
        if (p >= 1) os_erode(s, p - 1);            /* needs m(p-2 .. p) */
        if (p >= 2) {                               /* needs e(p-3 .. p-1) */
            os_dilate(s, p - 2);
            if (os_emit(s, p - 2, o_out, &n_out)) return -1;
        }
        return n_out;
    }
    if (s->fed != s->Z) return -1;
    if (s->se == 4) return 0;
    const int64_t Z = s->Z;
    os_erode(s, Z - 1);                             /* m(Z) is outside the volume */
    for (int64_t q = Z >= 2 ? Z - 2 : 0; q < Z; q++) {
        os_dilate(s, q);
        if (os_emit(s, q, o_out, &n_out)) return -1;
    }
    return n_out;
}

/* roots, sizes and the kept flags; returns the component count */
int64_t os_resolve(os_state *s, uint64_t min_size)
{
    free(s->root_size);
    free(s->kept_root);
    s->root_size = (uint64_t *)calloc(s->nlab ? s->nlab : 1, sizeof(uint64_t));
    s->kept_root = (uint8_t *)calloc(s->nlab ? s->nlab : 1, 1);
    if (!s->root_size || !s->kept_root) return -1;
    s->min_size = min_size;
    for (uint64_t l = 0; l < s->nlab; l++) s->root_size[os_find(s, l)] += s->size[l];
    int64_t nc = 0;
    for (uint64_t l = 0; l < s->nlab; l++)
        if (s->parent[l] == l) {
            s->kept_root[l] = s->root_size[l] >= min_size;
            nc++;
        }
    s->ncomp = (uint64_t)nc;
    return nc;
}

/* the component table in increasing minimum index (= increasing root label) */
int64_t os_table(os_state *s, uint64_t *cmin, uint64_t *csize, uint8_t *kept, uint64_t cap)
{
    int64_t c = 0;
    for (uint64_t l = 0; l < s->nlab; l++)
        if (s->parent[l] == l) {
            if ((uint64_t)c >= cap) return -1;
            cmin[c] = s->first[l];
            csize[c] = s->root_size[l];
            kept[c] = s->kept_root[l];
            c++;
        }
    return c;
}

/* Pass C for plane q (x: Y*X uint16): K (one byte per voxel) and the codes of its kept voxels in
 * increasing index; returns their number, -1 on a quantiser range error. */
int64_t os_extract(os_state *s, int64_t q, const uint16_t *x, float eb, uint8_t *K, uint16_t *codes)
{
    double st, c;
    if (step_of(eb, &st)) return -1;
    memset(K, 0, (size_t)(s->Y * s->X));
    int64_t j = 0;
    for (uint64_t r = s->plane_run0[q]; r < s->plane_run0[q + 1]; r++) {
        const os_run *R = &s->runs[r];
        if (!s->kept_root[os_find(s, R->label)]) continue;
        for (uint32_t xx = R->x0; xx < R->x1; xx++) {
            const int64_t a = (int64_t)R->y * s->X + xx;
            K[a] = 1;
            if (rne_exact((double)x[a], st, &c) || c > 65535.0) return -1;
            codes[j++] = (uint16_t)c;
        }
    }
    return j;
}

uint64_t os_nruns(const os_state *s) { return s->nruns; }
uint64_t os_nlabels(const os_state *s) { return s->nlab; }
