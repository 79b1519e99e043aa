/*
 * roix.h -- C ABI of libroix, the B200 (sm_100a) implementation of the ROIX-Comp hot path.
 *
 * ROIX-Comp (arXiv 2602.15917; /root/reference/PAPER.md, cited P:<line>) reduces X-CT data by
 * keeping only a region of interest (ROI) and storing it error-bounded.  The data-parallel hot path
 * built here (BASELINE.json north_star) is, per volume x[Z][Y][X]:
 *
 *   a0 RANGE      fp32 only: global min/max, relative eb                    roix_range, roix_resolve
 *   a2 HISTOGRAM  intensity histogram ("based on intensity distribution")  roix_histogram
 *   a3 THRESHOLD  Eq. 1 8-bit normalisation + Otsu       roix_threshold
 *   a4 BINARISE   Eq. 2 mask                                         \ roix_morph
 *   a5 MORPH      morphological cleanup: one opening, cross SE (reading G-11)    /
 *   a6 CCL        connected components, label = min linear index (G-14)        \ roix_label
 *   a7 FILTER     drop components smaller than min_size (G-13)                  /
 *   a1+a8 EXTRACT uniform error-bounded quantisation code = RNE(x / 2eb) of the kept voxels,
 *                 compacted in increasing linear index (paper analogue P:305-337)  roix_extract
 *   a1 alone      roix_quantize (every voxel)
 *
 * Conventions (all calls):
 *  - Linear index i = (z*Y + y)*X + x, uint64.  Volumes are dense, x fastest.
 *  - Bit-packed masks: bit (i mod 32) of uint32 word i/32, LSB first; pad bits are 0 (G-16).
 *  - Memory: every buffer is allocated by the caller (device memory unless stated).  The library
 *    never allocates, frees or synchronises; every call only enqueues work on `stream`, so a whole
 *    pipeline can be captured in a CUDA graph.  Pointers x, codes and bit arrays must be 16-byte
 *    aligned.  Workspaces are sized by the matching *_workspace() query (host-only, no GPU work).
 *  - Data-dependent scalars (eb, I_max, threshold, counts, error bits) live in a caller-allocated
 *    device struct roix_scalars so that no call needs a device->host read.
 *  - Host-detectable errors return a roix_status immediately and launch nothing:
 *      ROIX_E_INVALID      null pointer, misalignment, bad enum, bad size;
 *      ROIX_E_UNSUPPORTED  a parameter combination this library does not implement;
 *      ROIX_E_CUDA         a launch failed (text in roix_last_error()).
 *  - Data-dependent errors set sticky bits in roix_scalars.err (ROIX_ERR_*).  Every kernel reads
 *    err first and does nothing if it is non-zero, so no garbage propagates; check err after the
 *    final synchronisation.
 *  - Determinism: every output is a pure function of the inputs and parameters -- independent of
 *    launch configuration, atomic ordering and the number of GPUs a volume is sharded over.
 *  - n = 0 is valid everywhere and is a no-op.
 */
#ifndef ROIX_H
#define ROIX_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ROIX_VERSION 1

typedef struct CUstream_st *roix_stream_t; /* a cudaStream_t; NULL = the legacy default stream */

typedef enum { ROIX_OK = 0, ROIX_E_INVALID = 1, ROIX_E_UNSUPPORTED = 2, ROIX_E_CUDA = 3 } roix_status;

/* sticky device error bits (roix_scalars.err) */
#define ROIX_ERR_NONFINITE 1u  /* a NaN/Inf voxel in fp32 input (G-32)                              */
#define ROIX_ERR_RANGE 2u      /* |x| >= 2^23 * s, or a u16 code > 65535, or eb invalid (G-4, G-7)   */
#define ROIX_ERR_CAPACITY 4u   /* an output / workspace capacity was exceeded                        */
#define ROIX_ERR_DEGENERATE 8u /* fewer than two populated normalised-intensity bins      */
#define ROIX_ERR_FORMAT 16u    /* roix_decode_spans: records out of order / outside the slab / empty   */

typedef enum { ROIX_U16 = 1, ROIX_F32 = 2 } roix_dtype;
typedef enum { ROIX_POL_HIGH = 0, ROIX_POL_LOW = 1 } roix_polarity; /* ROI = norm8 > t8 / <= t8 (G-10) */

/*
 * Device-resident scalars of one volume.  Allocate sizeof(roix_scalars) bytes of device memory and
 * initialise with roix_scalars_init before the first call on a volume.
 */
typedef struct roix_scalars {
    uint32_t err;         /* sticky ROIX_ERR_* bits                                              */
    uint32_t min_ord;     /* a0: ordered-integer encoding of the fp32 minimum (atomicMin target)  */
    uint32_t max_ord;     /* a0: ordered-integer encoding of the fp32 maximum (atomicMax target)  */
    uint32_t polarity;    /* a3: roix_polarity used by roix_morph                                */
    float eb;             /* absolute error bound in input units (G-5, G-6)                      */
    float s;              /* quantisation step fl32(2*eb) (G-3)                                  */
    float s_inv;          /* fl32(1/s): fast-path reciprocal, always followed by an exact check   */
    uint32_t s_int;       /* s when s is an integer in [1, 65535], else 0 (u16 integer fast path) */
    uint32_t s_magic;     /* ceil(2^32 / s_int) for s_int >= 2: exact floor(v / s_int), v < 2^16 */
    uint32_t t8_all;      /* a3: every threshold, ascending, one per byte (k = 2: t8; k = 3: t1 | t2 << 8) */
    float i_max;          /* Eq. 1 I_max: global max, 1 when <= 0 (G-8)                  */
    uint32_t t8;          /* a3: Otsu threshold on the 8-bit normalised intensity                */
    uint32_t thr_u16;     /* a4 raw form: first u16 value v with norm8(v) > t8                   */
    float thr_f32;        /* a4 raw form: first fp32 value x with norm8(x) > t8                  */
    uint64_t count;       /* a8: number of kept voxels (global, after roix_extract)              */
    uint64_t n_components;/* a6: number of components (this slab's table)                        */
    uint64_t n_kept;      /* a7: number of kept components                                       */
    uint64_t n_runs;      /* a6: number of foreground x-runs found                               */
    uint32_t spec_lo;     /* fused a2+a4: speculative raw-threshold window (u16 value / fp32 bits)  */
    uint32_t spec_hi;
    uint32_t spec_state;  /* 0 none, 1 window set, 2 mask resolved, 3 fallback binarisation       */
    uint32_t run_slots;   /* a5 -> a6: run records per row roix_morph_slots wrote (0: none)       */
    uint64_t n_uncertain; /* fused a2+a4: voxels inside the window (resolved after the threshold)  */
    float edges[256];     /* fp32 only: edges[k] = smallest finite x with norm8(x) >= k (k>=1)   */
} roix_scalars;

/* Slab geometry: this buffer holds planes [z0, z0+nz) of a global volume of gz planes. */
typedef struct roix_geom {
    uint64_t nz, ny, nx;
    uint64_t z0, gz;
} roix_geom;

const char *roix_status_string(roix_status s);
const char *roix_last_error(void); /* thread-local text of the last failure */
int roix_version(void);
size_t roix_scalars_size(void);

/*
 * Initialise sc: clear err and counters, min/max to +inf/-inf, and set eb.  For absolute eb pass
 * eb_abs > 0 (it is validated on the host: ROIX_E_INVALID if not finite and > 0).  For a relative
 * eb (fp32 only) pass eb_abs = 0 and give rel_eb to roix_resolve.
 */
roix_status roix_scalars_init(roix_scalars *sc, float eb_abs, roix_stream_t stream);

/*
 * a0 RANGE (fp32; reading G-6/G-32).  Accumulates the min and max of x[0..n) into sc (call once
 * per buffer; several buffers may be accumulated).  Non-finite voxels set ROIX_ERR_NONFINITE.
 */
roix_status roix_range(const float *x, uint64_t n, roix_scalars *sc, roix_stream_t stream);

/*
 * Resolve data-dependent scalars once the range is known (G-6, G-8, G-30):
 *   - rel_eb > 0 (fp32): eb = fl32(rel_eb * (fl64(max) - fl64(min)));
 *   - s = fl32(2 eb), s_inv, s_int/s_magic;
 *   - fp32: I_max = max if max > 0 else 1, and edges[k] of norm8 (G-30) by bisection.
 * For u16 input call it with rel_eb = 0 after roix_scalars_init (I_max comes from the histogram).
 */
roix_status roix_resolve(roix_scalars *sc, roix_dtype dtype, double rel_eb, roix_stream_t stream);

/*
 * a1 QUANTISE every voxel: codes[i] = RNE(x[i] / s), the integer nearest the exact real quotient,
 * ties to even (BJ north_star; G-2..G-4).  u16 input -> uint16 codes, fp32 input -> int32 codes.
 * Requires roix_resolve.  Out-of-range voxels set ROIX_ERR_RANGE (their code is unspecified).
 */
roix_status roix_quantize(const void *x, roix_dtype dtype, uint64_t n, roix_scalars *sc, void *codes,
                          roix_stream_t stream);

/*
 * a2 HISTOGRAM, accumulated (+=) into hist:
 *   u16:  nbins = 65536, hist[v] += #{i : x[i] = v}           (raw values; I_max and the 256-bin
 *         norm8 histogram are derived from it exactly by roix_threshold);
 *   fp32: nbins = 256,   hist[k] += #{i : norm8(x[i]) = k}     (requires roix_resolve).
 * hist is uint64, caller-zeroed; for a sharded volume, sum the per-slab histograms (allreduce).
 */
roix_status roix_histogram(const void *x, roix_dtype dtype, uint64_t n, roix_scalars *sc, uint64_t *hist,
                           uint32_t nbins, roix_stream_t stream);

/*
 * Zero hist[0 .. nbins) (device uint64) on `stream` -- the start of a2 for an accumulating histogram
 * (one kernel of this library, so a captured step holds no foreign kernels).  nbins = 0 is a no-op;
 * hist must be 16-byte aligned.
 */
roix_status roix_histogram_clear(uint64_t *hist, uint64_t nbins, roix_stream_t stream);

/*
 * a3 THRESHOLD (Eq. 1 P:255-257 with round-half-up S:82; Otsu P:263-267 with k = 2, smallest t on
 * ties S:170; reading G-8/G-9).  u16: I_max = largest populated bin (1 if none above 0),
 * h8[norm8(v)] += hist[v] with norm8(v) = floor((510 v + I_max) / (2 I_max)).  fp32: hist is already
 * h8.  Otsu maximises the between-class variance exactly (256-bit integer compares).  Writes t8,
 * thr_u16/thr_f32, polarity, i_max (u16) into sc; fewer than two populated norm8 bins sets
 * ROIX_ERR_DEGENERATE.
 */
roix_status roix_threshold(const uint64_t *hist, uint32_t nbins, roix_dtype dtype, roix_polarity polarity,
                           roix_scalars *sc, roix_stream_t stream);

/*
 * NEXT-3 multi-Otsu ("multi-Otsu adaptive thresholding", AC4 S:565).
 * classes = 2: exactly roix_threshold.  classes = 3: the thresholds t1 < t2 maximising the
 * between-class variance sum_k w_k (mu_k - mu_T)^2 over every tuple with three non-empty classes,
 * the lexicographically smallest on ties (exact: 448-bit integer compares); sc->t8_all = t1 | t2 << 8
 * and the ROI threshold sc->t8 = t1 for HIGH (ROI = everything above the lowest threshold) or
 * t2 for LOW (ROI = everything at or below the highest, G-39); thr_u16 / thr_f32 follow
 * t8.  Fewer than `classes` populated norm8 bins sets ROIX_ERR_DEGENERATE.
 */
roix_status roix_threshold_multi(const uint64_t *hist, uint32_t nbins, roix_dtype dtype, roix_polarity polarity,
                                 uint32_t classes, roix_scalars *sc, roix_stream_t stream);

/*
 * NEXT-3 BACKGROUND SUBTRACTION (M(x, y) = I(x, y) - B(x, y), B from calibration scans
 * without the sample; SPEC S:61-69 clamps at 0) and its inverse for reconstruction.  uint16:
 * out[z][y][x] = op(x[z][y][x], B[y][x]) for every frame z < g->nz, one reference frame B[ny][nx]
 * (device) for all frames:
 *   ROIX_BG_SUB  max(0, I - B)   (the paper's M)
 *   ROIX_BG_REV  max(0, B - I)   (transmission frames, where the sample darkens I: G-10, G-40)
 *   ROIX_BG_ADD  min(65535, M + B)  (restores SUB; REV is its own inverse)
 * out may alias x.  16-byte alignment as everywhere; frames of ny*nx % 8 != 0 voxels take a slower
 * per-voxel path.
 */
typedef enum { ROIX_BG_SUB = 0, ROIX_BG_REV = 1, ROIX_BG_ADD = 2 } roix_bg_op;
roix_status roix_background(const uint16_t *x, const uint16_t *B, const roix_geom *g, roix_bg_op op, uint16_t *out,
                            roix_stream_t stream);

/*
 * NEXT-3 PER-FRAME THRESHOLDS (uint16 frame stacks, e.g. detector frames, C3): every z-plane of the
 * slab is its own image, as in the paper's 2-D pipeline -- its own I_max (Eq. 1),
 * norm8 histogram and (multi-)Otsu thresholds.
 *   roix_histogram_frames   hist[z * 65536 + v] += #{voxels of frame z equal to v}, z < g->nz
 *   roix_threshold_frames   frames[z] from frame z's histogram: i_max, t8_all (every threshold, one
 *                           per byte), t8 (the ROI threshold, as roix_threshold_multi) and thr_u16 =
 *                           the first value v with norm8_z(v) > t8; sc->polarity set.  A frame with
 *                           too few populated bins sets ROIX_ERR_DEGENERATE.
 *   roix_morph_frames       roix_morph (u16) with frame z binarised against frames[z].thr_u16.
 */
typedef struct roix_frame {
    uint32_t thr_u16; /* raw threshold: ROI = x >= thr_u16 (HIGH) or x < thr_u16 (LOW) */
    uint32_t t8;      /* ROI threshold on the frame's norm8 scale                       */
    uint32_t t8_all;  /* every threshold, ascending, one per byte                       */
    uint32_t i_max;   /* the frame's I_max (Eq. 1)                                      */
} roix_frame;

roix_status roix_histogram_frames(const uint16_t *x, const roix_geom *g, roix_scalars *sc, uint64_t *hist,
                                  roix_stream_t stream);
roix_status roix_threshold_frames(const uint64_t *hist, uint64_t nframes, roix_polarity polarity, uint32_t classes,
                                  roix_scalars *sc, roix_frame *frames, roix_stream_t stream);

/*
 * a4+a5 BINARISE + OPEN (Eq. 2; G-11).  m = [norm8(x) > t8] (HIGH) or [<= t8] (LOW), evaluated as
 * the equivalent raw compare against thr_*; o = dilate(erode(m)) with the radius-1 cross:
 *   se = 6: 6 face neighbours (3-D);  se = 4: the 4 in-plane neighbours (2-D per z-plane).
 * Out-of-volume neighbours are ignored (erosion border 1, dilation border 0).
 * x holds the slab g (planes z0..z0+nz-1); o_bits receives its ceil(nz*ny*nx/32) words.
 * Sharded 3-D volumes (se = 6, z0 > 0 or z0+nz < gz): halo_lo holds the binarised m of global
 * planes z0-2, z0-1 and halo_hi of z0+nz, z0+nz+1 (each plane packed from bit 0 with
 * ceil(ny*nx/32) words; produced by roix_binarize_planes on the neighbour); planes that do not
 * exist in the global volume are ignored.  NULL halos are allowed only at global volume faces.
 * row_runs (nullable, nz*ny uint32): receives the number of x-runs of o in each row -- the fused
 * first step of roix_label, which then skips its own counting pass.
 * ws/ws_bytes (roix_morph_workspace): holds the binarised mask m between the two kernels.
 * Slabs of >= 2^30 voxels are processed in chunks of whole planes: each chunk is binarised on
 * `stream` and opened on a second, library-owned stream of the current device (forked from and
 * joined back to `stream` with events), so the opening of one chunk runs beside the binarisation of
 * the next.  The call stays stream-ordered on `stream` (and capturable in a CUDA graph); concurrent
 * calls on different streams share that second stream (their enqueue sequences are serialised by a
 * lock, so each call's chunks keep their own dependencies).
 */
roix_status roix_morph_workspace(const roix_geom *g, size_t *ws_bytes);
roix_status roix_morph(const void *x, roix_dtype dtype, const roix_geom *g, uint32_t se, const uint32_t *halo_lo,
                       const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs,
                       void *ws, size_t ws_bytes, roix_stream_t stream);
/*
 * roix_morph plus run records: run_slots (nz*ny*slots_per_row pairs of uint32, 8-byte aligned;
 * needs row_runs) receives, for every row of o, the first slots_per_row x-runs as (x0, x1) with x1
 * exclusive; sc->run_slots is set to slots_per_row when they were written (0 when this form of the
 * opening writes none).  roix_label_slots / roix_label_local_slots then take the runs of every row
 * with at most slots_per_row runs from here instead of reading that row of o again (the opening had
 * the row in registers anyway).  slots_per_row in 1..64.
 */
roix_status roix_morph_slots(const void *x, roix_dtype dtype, const roix_geom *g, uint32_t se, const uint32_t *halo_lo,
                             const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs,
                             uint32_t *run_slots, uint32_t slots_per_row, void *ws, size_t ws_bytes,
                             roix_stream_t stream);

/*
 * a2+a4 fused by speculation (one read of x instead of two).  A 1/64 sample of x gives Otsu a window
 * for the raw threshold; one pass then accumulates the full histogram into `hist` (exactly as
 * roix_histogram) and writes into ws the mask bits that are certain for any threshold inside the
 * window, queueing the voxels inside it.  After roix_threshold (on the -- possibly all-reduced --
 * histogram), roix_morph_prebinarized resolves the queued voxels with the exact threshold, or
 * re-binarises x when the threshold fell outside the window or the queue overflowed, then opens.
 * The mask is exactly that of roix_morph in every case.  ws: roix_histogram_binarize_workspace bytes,
 * the same buffer for both calls.
 */
roix_status roix_histogram_binarize_workspace(const roix_geom *g, size_t *ws_bytes);
roix_status roix_histogram_binarize(const void *x, roix_dtype dtype, const roix_geom *g, roix_polarity polarity,
                                    roix_scalars *sc, uint64_t *hist, uint32_t nbins, void *ws, size_t ws_bytes,
                                    roix_stream_t stream);
roix_status roix_morph_prebinarized(const void *x, roix_dtype dtype, const roix_geom *g, uint32_t se,
                                    const uint32_t *halo_lo, const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits,
                                    uint32_t *row_runs, void *ws, size_t ws_bytes, roix_stream_t stream);

roix_status roix_morph_frames(const uint16_t *x, const roix_geom *g, uint32_t se, const uint32_t *halo_lo,
                             const uint32_t *halo_hi, const roix_frame *frames, roix_scalars *sc, uint32_t *o_bits,
                             uint32_t *row_runs, void *ws, size_t ws_bytes, roix_stream_t stream);

/* Binarise planes [p0, p0+np) of the slab (slab-local plane numbers) into m_bits, each plane
 * packed from bit 0 with ceil(ny*nx/32) words -- the halo planes roix_morph consumes. */
roix_status roix_binarize_planes(const void *x, roix_dtype dtype, const roix_geom *g, uint64_t p0, uint64_t np,
                                 roix_scalars *sc, uint32_t *m_bits, roix_stream_t stream);

/*
 * a6+a7 LABEL + FILTER.  Connected components of o under conn (6, 18, 26: 3-D; 4, 8: in-plane per
 * z-plane), each named by its minimum global linear index (G-14).  Components of size < min_size
 * are dropped (G-13).  min_size = ROIX_KEEP_LARGEST (NEXT-3, "select the largest by area";
 * S:185-193) keeps only the largest component, ties to the smallest label (raster-order anchor).
 * Outputs (device):
 *   keep_bits      K = o AND kept; may alias o_bits (in-place: only dropped voxels are cleared);
 *   comp_min/comp_size/comp_kept  the component table in increasing min index, capacity comp_cap
 *                  (any may be NULL to skip the table); counts in sc->n_components / n_kept;
 *   labels         optional (nullable) uint64 per voxel: the component label, UINT64_MAX for
 *                  background.
 * Works on x-runs of o (maximal stretches of set bits in one row); run_capacity bounds their
 * number (ROIX_ERR_CAPACITY if exceeded).  row_runs: the per-row run counts roix_morph produced
 * for this o (nullable: then they are counted here).  ws/ws_bytes from roix_label_workspace.
 */
#define ROIX_KEEP_LARGEST UINT64_MAX

typedef struct roix_label_out {
    uint32_t *keep_bits;
    uint64_t *comp_min;
    uint64_t *comp_size;
    uint8_t *comp_kept;
    uint64_t comp_cap;
    uint64_t *labels;
} roix_label_out;

roix_status roix_label_workspace(const roix_geom *g, uint64_t run_capacity, size_t *ws_bytes);
roix_status roix_label(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom *g, uint32_t conn,
                       uint64_t min_size, uint64_t run_capacity, void *ws, size_t ws_bytes,
                       const roix_label_out *out, roix_scalars *sc, roix_stream_t stream);
/* roix_label with the run records of roix_morph_slots (same row_runs / run_slots / slots_per_row;
 * used only when sc->run_slots == slots_per_row, i.e. the preceding opening wrote them). */
roix_status roix_label_slots(const uint32_t *o_bits, const uint32_t *row_runs, const uint32_t *run_slots,
                             uint32_t slots_per_row, const roix_geom *g, uint32_t conn, uint64_t min_size,
                             uint64_t run_capacity, void *ws, size_t ws_bytes, const roix_label_out *out,
                             roix_scalars *sc, roix_stream_t stream);

/*
 * Sharded labelling (z-slab decomposition over GPUs).  roix_label above equals
 * roix_label_local followed by roix_label_finish with an empty merge map.  For a volume split into
 * z-slabs (one per rank), each rank:
 *   1. roix_label_local on its slab (runs, union-find, sizes of the slab-local components);
 *   2. roix_label_boundary(side = 1) exports the runs of its last plane (to rank + 1);
 *   3. roix_label_link pairs its first-plane components with the previous rank's last-plane runs;
 *   4. roix_label_boundary_roots lists (label, size) of its components touching either slab face,
 *      in increasing label order;
 *   5. all ranks gather every pair list and root table, and roix_merge_device (or roix_merge on
 *      the host) -- the same deterministic union-by-min on every rank -- maps each boundary label to
 *      its merged label and total size;
 *   6. roix_label_finish applies the map: table entries live on the rank holding the component's
 *      minimum index; small-object removal uses the merged sizes.
 * Every map argument below is device memory: map_label (ascending), map_final, map_total, and the map
 * length *nmap (device uint64; nmap = NULL: an empty map).
 * Labels are global linear indices (uint64).  ws / run_capacity are those of roix_label_local.
 * Keep-largest on a sharded volume (NEXT-3): after roix_merge, roix_label_largest(phase 0) writes the
 * largest size among this slab's owned components to best[0] (device, 2 uint64; phase 0 first resets
 * best to (0, 2^63 - 1 = none)); reduce best[0] with MAX over ranks; phase 1 writes the smallest label of
 * that size to best[1]; reduce best[1] with MIN; roix_label_finish_keep then keeps exactly the
 * component best[1] on every rank (nothing if the volume has no component).
 */
typedef struct roix_brun {
    uint32_t y, x0, x1, pad; /* row within the plane, run [x0, x1)                    */
    uint64_t label;          /* global label (min linear index) of its local component  */
} roix_brun;

roix_status roix_label_local(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom *g, uint32_t conn,
                             uint64_t run_capacity, void *ws, size_t ws_bytes, roix_scalars *sc,
                             roix_stream_t stream);
roix_status roix_label_local_slots(const uint32_t *o_bits, const uint32_t *row_runs, const uint32_t *run_slots,
                                   uint32_t slots_per_row, const roix_geom *g, uint32_t conn, uint64_t run_capacity,
                                   void *ws, size_t ws_bytes, roix_scalars *sc, roix_stream_t stream);
roix_status roix_label_boundary(const void *ws, const roix_geom *g, uint64_t run_capacity, int side, roix_brun *out,
                                uint64_t out_cap, uint64_t *count, roix_scalars *sc, roix_stream_t stream);
roix_status roix_label_link(const void *ws, const roix_geom *g, uint64_t run_capacity, uint32_t conn,
                            const roix_brun *prev, const uint64_t *n_prev, uint64_t *pairs, uint64_t pair_cap,
                            uint64_t *n_pairs, roix_scalars *sc, roix_stream_t stream);
roix_status roix_label_boundary_roots(const void *ws, const roix_geom *g, uint64_t run_capacity, uint64_t *labels,
                                      uint64_t *sizes, uint64_t out_cap, uint64_t *count, roix_scalars *sc,
                                      roix_stream_t stream);
/* HOST memory, no GPU work: pairs[2k], pairs[2k+1] are labels of one component; labels / sizes the
 * boundary components of all slabs.  Outputs (capacity nlabels): the distinct labels in increasing
 * order with their merged label and total size; *nout = their number.  ROIX_E_INVALID if a pair
 * names a label missing from `labels`. */
roix_status roix_merge(const uint64_t *pairs, uint64_t npairs, const uint64_t *labels, const uint64_t *sizes,
                       uint64_t nlabels, uint64_t *out_label, uint64_t *out_final, uint64_t *out_total,
                       uint64_t *nout);
/* The same merge on the device, enqueued on `stream` (every rank runs it on the same input, so the maps
 * agree without a host round trip; the whole sharded step stays capturable).  gathered: G blocks of
 * W = 2 + 2 pair_cap + 2 root_cap uint64 words in rank order, block r = rank r's
 *   [npairs, nroots, pairs[2 pair_cap] (roix_label_link), labels[root_cap], sizes[root_cap]
 *    (roix_label_boundary_roots)];
 * blocks concatenate to an ascending label list (every rank's labels lie in its own slab).  Outputs:
 * map_label / map_final / map_total (capacity G * root_cap) and *nmap (device).  A count above its
 * capacity sets ROIX_ERR_CAPACITY, a pair naming a label missing from the tables ROIX_ERR_FORMAT.
 * ws: roix_merge_workspace(G, root_cap) bytes, 16-byte aligned. */
roix_status roix_merge_workspace(uint32_t G, uint64_t root_cap, size_t *ws_bytes);
roix_status roix_merge_device(const uint64_t *gathered, uint32_t G, uint64_t pair_cap, uint64_t root_cap,
                              uint64_t *map_label, uint64_t *map_final, uint64_t *map_total, uint64_t *nmap, void *ws,
                              size_t ws_bytes, roix_scalars *sc, roix_stream_t stream);
roix_status roix_label_finish(const uint32_t *o_bits, const roix_geom *g, uint64_t min_size, uint64_t run_capacity,
                              void *ws, size_t ws_bytes, const uint64_t *map_label, const uint64_t *map_final,
                              const uint64_t *map_total, const uint64_t *nmap, const roix_label_out *out, roix_scalars *sc,
                              roix_stream_t stream);

roix_status roix_label_largest(void *ws, const roix_geom *g, uint64_t run_capacity, const uint64_t *map_label,
                               const uint64_t *map_final, const uint64_t *map_total, const uint64_t *nmap, uint32_t phase,
                               uint64_t *best, roix_scalars *sc, roix_stream_t stream);
roix_status roix_label_finish_keep(const uint32_t *o_bits, const roix_geom *g, uint64_t run_capacity, void *ws,
                                   size_t ws_bytes, const uint64_t *map_label, const uint64_t *map_final,
                                   const uint64_t *map_total, const uint64_t *nmap, const uint64_t *keep,
                                   const roix_label_out *out, roix_scalars *sc, roix_stream_t stream);

/*
 * a1+a8 EXTRACT.  For the set bits i_0 < i_1 < ... of keep_bits (n voxels), codes_out[j] =
 * RNE(x[i_j] / s) (u16 -> uint16, fp32 -> int32), written at codes_out[offset + j].  Adds the
 * number of set bits to sc->count.  Reads x only where keep_bits has set bits.  More than
 * `capacity` codes sets ROIX_ERR_CAPACITY (nothing is written past capacity).
 * offset: device pointer to a uint64 start position (NULL = 0) -- the rank's global offset when
 * a sharded stream is assembled.  ws/ws_bytes from roix_extract_workspace.
 */
roix_status roix_extract_workspace(uint64_t n, size_t *ws_bytes);
roix_status roix_extract(const void *x, roix_dtype dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                         void *codes_out, uint64_t capacity, const uint64_t *offset, void *ws, size_t ws_bytes,
                         roix_stream_t stream);

/*
 * a1+a8 EXTRACT from the labelling's kept runs (the pipeline's form of roix_extract).  After
 * roix_label (or roix_label_finish) on the same ws, writes exactly what roix_extract(x, K) writes for
 * the K that call produced -- codes_out[offset + j] = RNE(x[i_j] / s) for the kept voxels i_0 < i_1 <
 * ... of the slab -- and adds their number to sc->count, but reads neither K nor any voxel of x
 * outside the kept runs: x is read run by run with 16-byte loads (the kept runs in raster order are
 * the kept voxels in increasing linear index, G-17).  g, run_capacity, ws, ws_bytes: those of the
 * labelling (ws is also scratch here).  capacity / offset / errors: as roix_extract.
 */
roix_status roix_extract_runs(const void *x, roix_dtype dtype, const roix_geom *g, uint64_t run_capacity, void *ws,
                              size_t ws_bytes, roix_scalars *sc, void *codes_out, uint64_t capacity,
                              const uint64_t *offset, roix_stream_t stream);

/*
 * NEXT-1 ROW SPANS: the paper's ROI representation.  For every row
 * i = z*Y + y (global: z counts from the volume's first plane) of keep_bits holding a set bit, in
 * increasing i: the geometry record spans[k] = {i, x_start, x_end} -- x_start the leftmost set column,
 * x_end the rightmost + 1 (exclusive, n_i = x_end - x_start) -- and the pixel section: the codes
 * RNE(x / s) of x[i][x_start .. x_end), interior gaps included, concatenated in codes (uint16 for
 * u16 input, int32 for fp32).  counts (device, 2 uint64): number of records, total section length.
 * Requires roix_resolve (the step s).  More than span_cap records or code_cap codes sets
 * ROIX_ERR_CAPACITY (nothing is written past either capacity).  ws/ws_bytes from
 * roix_row_spans_workspace.  keep_bits / x: the slab g, as roix_label / roix_extract.
 */
typedef struct roix_span {
    uint64_t row;     /* i = z*Y + y                              */
    uint32_t x_start; /* leftmost set column                      */
    uint32_t x_end;   /* rightmost set column + 1 (exclusive)     */
} roix_span;

roix_status roix_row_spans_workspace(const roix_geom *g, size_t *ws_bytes);
roix_status roix_row_spans(const uint32_t *keep_bits, const void *x, roix_dtype dtype, const roix_geom *g,
                           roix_scalars *sc, roix_span *spans, uint64_t span_cap, void *codes, uint64_t code_cap,
                           uint64_t *counts, void *ws, size_t ws_bytes, roix_stream_t stream);

/*
 * NEXT-2 GREEDY QUANTISER: the paper's absolute-error-bounded quantiser (§4.2.3 Steps 1-5,
 * P:340-399) on a uint16 sequence D[0..n) (device): groups are the greedy left-to-right
 * maximal runs whose intervals [D - E, D + E] intersect (range max - min <= 2E); Q[i] = floor((u + l)
 * / 2) = floor((max + min) / 2) of i's group, clipped to [0, qmax] (Step 5: 255 for 8-bit data).
 * group_bits (device, ceil(n/32) words): bit i set where a group starts; *ngroups (device): their
 * number.  E >= 0 and finite (S:299 admits 0: runs of equal values).  |Q - D| <= E for integer E and
 * whenever frac(E) < 1/2 (G-35).  ws/ws_bytes from roix_greedy_workspace.
 */
roix_status roix_greedy_workspace(uint64_t n, size_t *ws_bytes);
roix_status roix_greedy_quantize(const uint16_t *D, uint64_t n, double E, uint32_t qmax, uint16_t *Q, uint32_t *group_bits,
                                 uint64_t *ngroups, void *ws, size_t ws_bytes, roix_stream_t stream);

/*
 * NEXT-4 RECONSTRUCTION ("each row is precisely restored using the preserved metadata";
 * SPEC S:359-367 reconstruct_image without a background: the ROI on a zero canvas).  The decoded value
 * of a code c, with s = sc->s = fl32(2 eb) (set by roix_scalars_init + roix_resolve with the eb the
 * codes were made with; G-37):
 *   u16 input   x^ = min(65535, RNE(c * s)): c * s_int when s is an integer, else the exact binary64
 *               product rounded half to even -- |x - x^| <= eb for integer s (eb + 1/2 otherwise);
 *   fp32 input  x^ = fl32(fl32(c) * s), one correctly rounded fp32 multiply.
 *
 * roix_decode: the mask form (roix_extract's output).  xhat[i] = x^(codes[j]) for the j-th set bit i
 * of keep_bits[0..n) (in increasing i), 0 elsewhere; every voxel of xhat[0..n) (dtype's type) is
 * written.  ncodes: elements readable at codes; more kept voxels than ncodes sets ROIX_ERR_CAPACITY
 * and writes nothing.  ws/ws_bytes from roix_decode_workspace.
 */
roix_status roix_decode_workspace(uint64_t n, size_t *ws_bytes);
roix_status roix_decode(const uint32_t *keep_bits, const void *codes, uint64_t ncodes, roix_dtype dtype, uint64_t n,
                        roix_scalars *sc, void *xhat, void *ws, size_t ws_bytes, roix_stream_t stream);

/*
 * roix_decode_spans: the span form (roix_row_spans' output, the paper's representation).  xhat is the
 * slab g ([nz][ny][nx], dtype's type), every voxel written: row i = z*Y + y (global) of a record gets
 * x^ of its section's codes over [x_start, x_end), every other voxel 0.  counts (device, 2 uint64) =
 * (number of records, total section length) as roix_row_spans wrote them; spans hold span_cap
 * records and codes code_cap codes.  Records must have strictly increasing rows inside the slab and
 * 0 <= x_start < x_end <= nx, and the lengths must sum to counts[1]: else ROIX_ERR_FORMAT; more than
 * span_cap records or code_cap codes: ROIX_ERR_CAPACITY.  Nothing is decoded after either error.
 * ws/ws_bytes from roix_decode_spans_workspace.
 */
roix_status roix_decode_spans_workspace(const roix_geom *g, size_t *ws_bytes);
roix_status roix_decode_spans(const roix_span *spans, uint64_t span_cap, const void *codes, uint64_t code_cap,
                              const uint64_t *counts, roix_dtype dtype, const roix_geom *g, roix_scalars *sc,
                              void *xhat, void *ws, size_t ws_bytes, roix_stream_t stream);

/*
 * NEXT-4 ROI QUALITY METRICS.  roix_confusion: the per-voxel tally of two
 * bit-packed masks of n voxels (device) into counts (device, 4 uint64) = (tp, fp, fn, tn): tp =
 * #(pred & truth), fp = #(pred & ~truth), fn = #(~pred & truth), tn = n - tp - fp - fn.  Pad bits past
 * n are ignored.
 */
roix_status roix_confusion(const uint32_t *pred_bits, const uint32_t *truth_bits, uint64_t n, uint64_t *counts,
                           roix_stream_t stream);

/*
 * roix_overlap_metrics (host only, no GPU work): Eqs. 7-14 from counts (host, 4 uint64: tp, fp, fn, tn)
 * into out (host, 7 doubles): dsc = 2tp/(2tp+fp+fn), iou = tp/(tp+fp+fn), sensitivity = tp/(tp+fn),
 * specificity = tn/(tn+fp), accuracy = (tp+tn)/N, kappa = ((tp+tn) - f_c)/(N - f_c) with f_c =
 * ((tn+fn)(tn+fp) + (fp+tp)(fn+tp))/N, auc = 1 - (fp/(fp+tn) + fn/(fn+tp))/2; N = tp+fp+fn+tn.  Ratios
 * of exact 128-bit integers; a zero denominator gives NaN.
 */
roix_status roix_overlap_metrics(const uint64_t *counts, double *out);

#ifdef __cplusplus
}
#endif
#endif /* ROIX_H */
