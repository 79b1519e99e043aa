// kernels.cuh -- host-side launch entry points of the libroix kernels (called by api.cu).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

#include "roix.h"

int num_sms();  // SM count of the current device (cached)

// The labelling's x-runs (run order = raster order of their first voxel), as a7 left them.
struct RunsView {
    const uint64_t *n_runs;                       // device: number of runs
    const uint32_t *x0, *x1, *rrow, *parent;      // run [x0, x1) of slab row rrow; parent = its local root
    const uint8_t *kept;                          // kept flag, valid at roots
    uint32_t *err_snap;                           // error bits before the gather (its own must not stop it)
};

cudaError_t launch_scalars_init(roix_scalars *sc, float eb, cudaStream_t st);
cudaError_t launch_range(const float *x, uint64_t n, roix_scalars *sc, cudaStream_t st);
cudaError_t launch_resolve(roix_scalars *sc, int dtype, double rel_eb, cudaStream_t st);

cudaError_t launch_quantize(const void *x, int dtype, uint64_t n, roix_scalars *sc, void *codes, cudaStream_t st);

cudaError_t launch_hist_clear(uint64_t *hist, uint64_t nbins, cudaStream_t st);
cudaError_t launch_hist_u16(const uint16_t *x, uint64_t n, roix_scalars *sc, uint64_t *hist, cudaStream_t st);
cudaError_t launch_hist_f32(const float *x, uint64_t n, roix_scalars *sc, uint64_t *hist, cudaStream_t st);

cudaError_t launch_threshold(const uint64_t *hist, int dtype, int polarity, roix_scalars *sc, cudaStream_t st,
                             int classes = 2);

size_t morph_workspace_bytes(const roix_geom &g);
cudaError_t launch_morph(const void *x, int dtype, const roix_geom &g, uint32_t se, const uint32_t *halo_lo,
                         const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs, void *ws,
                         int prebinarized, cudaStream_t st, const roix_frame *frames = nullptr,
                         uint2 *run_slots = nullptr, uint32_t rs = 0);

cudaError_t launch_spec(const uint64_t *shist, int dtype, int polarity, roix_scalars *sc, cudaStream_t st);
size_t fused_workspace_bytes(const roix_geom &g);
cudaError_t launch_histogram_binarize(const void *x, int dtype, const roix_geom &g, int polarity, roix_scalars *sc,
                                      uint64_t *hist, void *ws, cudaStream_t st);
cudaError_t launch_spec_resolve(const void *x, int dtype, const roix_geom &g, roix_scalars *sc, void *ws,
                                cudaStream_t st);
cudaError_t launch_binarize_planes(const void *x, int dtype, const roix_geom &g, uint64_t p0, uint64_t np,
                                   roix_scalars *sc, uint32_t *m_bits, cudaStream_t st);

size_t label_workspace_bytes(const roix_geom &g, uint64_t cap);
cudaError_t launch_label(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom &g, uint32_t conn,
                         uint64_t min_size, uint64_t cap, void *ws, const roix_label_out &out, roix_scalars *sc,
                         cudaStream_t st, const uint2 *run_slots = nullptr, uint32_t rs = 0);

size_t extract_workspace_bytes(uint64_t n);
cudaError_t launch_extract(const void *x, int dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                           void *codes, uint64_t capacity, const uint64_t *offset, void *ws, cudaStream_t st);

cudaError_t launch_label_local(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom &g, uint32_t conn,
                               uint64_t cap, void *ws, roix_scalars *sc, cudaStream_t st, const uint2 *run_slots = nullptr,
                               uint32_t rs = 0);
cudaError_t launch_label_finish(const uint32_t *o_bits, const roix_geom &g, uint64_t min_size, uint64_t cap, void *ws,
                                const uint64_t *map_label, const uint64_t *map_final, const uint64_t *map_total,
                                const uint64_t *nmap, const roix_label_out &out, roix_scalars *sc, cudaStream_t st,
                                const uint64_t *keep = nullptr);
cudaError_t launch_label_largest(const roix_geom &g, uint64_t cap, void *ws, const uint64_t *map_label,
                                 const uint64_t *map_final, const uint64_t *map_total, const uint64_t *nmap, uint64_t *best,
                                 int phase, roix_scalars *sc, cudaStream_t st);
cudaError_t launch_label_boundary(const void *ws, const roix_geom &g, uint64_t cap, int side, roix_brun *out,
                                  uint64_t out_cap, uint64_t *count, roix_scalars *sc, cudaStream_t st);
cudaError_t launch_label_link(const void *ws, const roix_geom &g, uint64_t cap, uint32_t conn, const roix_brun *prev,
                              const uint64_t *n_prev, uint64_t *pairs, uint64_t pair_cap, uint64_t *n_pairs,
                              roix_scalars *sc, cudaStream_t st);
cudaError_t launch_label_boundary_roots(const void *ws, const roix_geom &g, uint64_t cap, uint64_t *labels,
                                        uint64_t *sizes, uint64_t out_cap, uint64_t *count, roix_scalars *sc,
                                        cudaStream_t st);


cudaError_t launch_runx(const void *x, int dtype, uint64_t n, uint64_t nx, const RunsView &R, uint64_t cap, uint32_t *klen,
                        uint64_t *koff, uint64_t *scan_tmp, roix_scalars *sc, void *codes,
                        uint64_t capacity, const uint64_t *offset, cudaStream_t st);
cudaError_t launch_extract_runs(const void *x, int dtype, const roix_geom &g, uint64_t cap, void *ws, roix_scalars *sc,
                                void *codes, uint64_t capacity, const uint64_t *offset, cudaStream_t st);

size_t row_spans_workspace_bytes(const roix_geom &g);
cudaError_t launch_row_spans(const uint32_t *K, const void *x, int dtype, const roix_geom &g, roix_scalars *sc,
                             roix_span *spans, uint64_t span_cap, void *codes, uint64_t code_cap, uint64_t *counts,
                             void *ws, cudaStream_t st);

size_t greedy_workspace_bytes(uint64_t n);
cudaError_t launch_greedy(const uint16_t *D, uint64_t n, double E, uint32_t qmax, uint16_t *Q, uint32_t *group_bits,
                          uint64_t *ngroups, void *ws, cudaStream_t st);

size_t decode_workspace_bytes(uint64_t n);
cudaError_t launch_decode(const uint32_t *K, const void *codes, uint64_t ncodes, int dtype, uint64_t n,
                          roix_scalars *sc, void *xhat, void *ws, cudaStream_t st);
size_t decode_spans_workspace_bytes(const roix_geom &g);
cudaError_t launch_decode_spans(const roix_span *spans, uint64_t span_cap, const void *codes, uint64_t code_cap,
                                const uint64_t *counts, int dtype, const roix_geom &g, roix_scalars *sc, void *xhat,
                                void *ws, cudaStream_t st);
cudaError_t launch_confusion(const uint32_t *pred, const uint32_t *truth, uint64_t n, uint64_t *counts,
                             cudaStream_t st);

cudaError_t launch_hist_u16_frames(const uint16_t *x, uint64_t nframes, uint64_t A, roix_scalars *sc, uint64_t *hist,
                                   cudaStream_t st);
cudaError_t launch_threshold_frames(const uint64_t *hist, uint64_t nframes, int polarity, int classes,
                                    roix_scalars *sc, roix_frame *frames, cudaStream_t st);
cudaError_t launch_background(const uint16_t *x, const uint16_t *B, const roix_geom &g, int op, uint16_t *out,
                              cudaStream_t st);

size_t merge_workspace_bytes(uint32_t G, uint64_t root_cap);
cudaError_t launch_merge(const uint64_t *gathered, uint32_t G, uint64_t pair_cap, uint64_t root_cap,
                         uint64_t *map_label, uint64_t *map_final, uint64_t *map_total, uint64_t *nmap, void *ws,
                         roix_scalars *sc, cudaStream_t st);
