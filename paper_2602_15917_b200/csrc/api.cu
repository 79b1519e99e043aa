// api.cu -- the C ABI of libroix (include/roix.h): argument validation, workspace sizing and launches
// on the caller's stream.  No allocation, no synchronisation.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <mutex>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "kernels.cuh"
#include "roix.h"

namespace {

thread_local char g_err[512] = "";

roix_status fail(roix_status s, const char *fmt, const char *what) {
    snprintf(g_err, sizeof(g_err), fmt, what);
    return s;
}
roix_status invalid(const char *what) { return fail(ROIX_E_INVALID, "invalid argument: %s", what); }
roix_status unsupported(const char *what) { return fail(ROIX_E_UNSUPPORTED, "unsupported: %s", what); }
roix_status cuda(cudaError_t e, const char *where) {
    if (e == cudaSuccess) return ROIX_OK;
    snprintf(g_err, sizeof(g_err), "%s: %s", where, cudaGetErrorString(e));
    return ROIX_E_CUDA;
}
bool aligned16(const void *p) { return ((uintptr_t)p & 15u) == 0; }

// NVTX range around an enqueuing call (a profiler's timeline shows which C-ABI call issued which
// kernels; without a profiler attached the push / pop are no-ops)
struct Range {
    explicit Range(const char *name) { nvtxRangePushA(name); }
    ~Range() { nvtxRangePop(); }
};
bool dtype_ok(roix_dtype d) { return d == ROIX_U16 || d == ROIX_F32; }
bool geom_ok(const roix_geom *g) {
    if (!g) return false;
    if (g->nz == 0 || g->ny == 0 || g->nx == 0) return false;
    if (g->z0 + g->nz > g->gz) return false;
    // linear indices are uint64; keep nz*ny*nx and the bit count well inside
    long double n = (long double)g->nz * g->ny * g->nx;
    return n < 1.0e18L;
}

}  // namespace

int num_sms() {
    static int sms = 0;
    static std::once_flag once;
    std::call_once(once, [] {
        int dev = 0;
        cudaGetDevice(&dev);
        if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
    });
    return sms;
}

extern "C" {

const char *roix_status_string(roix_status s) {
    switch (s) {
    case ROIX_OK: return "ok";
    case ROIX_E_INVALID: return "invalid argument";
    case ROIX_E_UNSUPPORTED: return "unsupported";
    case ROIX_E_CUDA: return "CUDA error";
    }
    return "unknown status";
}

const char *roix_last_error(void) { return g_err; }
int roix_version(void) { return ROIX_VERSION; }
size_t roix_scalars_size(void) { return sizeof(roix_scalars); }

roix_status roix_scalars_init(roix_scalars *sc, float eb_abs, roix_stream_t stream) {
    if (!sc) return invalid("sc is NULL");
    if (!(eb_abs >= 0.0f) || !std::isfinite(eb_abs)) return invalid("eb_abs must be finite and >= 0");
    return cuda(launch_scalars_init(sc, eb_abs, (cudaStream_t)stream), "roix_scalars_init");
}

roix_status roix_range(const float *x, uint64_t n, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_range");
    if (!sc) return invalid("sc is NULL");
    if (n == 0) return ROIX_OK;
    if (!x || !aligned16(x)) return invalid("x must be a 16-byte aligned device pointer");
    return cuda(launch_range(x, n, sc, (cudaStream_t)stream), "roix_range");
}

roix_status roix_resolve(roix_scalars *sc, roix_dtype dtype, double rel_eb, roix_stream_t stream) {
    const Range nvtx_range("roix_resolve");
    if (!sc) return invalid("sc is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (!(rel_eb >= 0.0) || !std::isfinite(rel_eb)) return invalid("rel_eb must be finite and >= 0");
    if (rel_eb > 0.0 && dtype != ROIX_F32) return unsupported("relative eb needs fp32 input");
    return cuda(launch_resolve(sc, (int)dtype, rel_eb, (cudaStream_t)stream), "roix_resolve");
}

roix_status roix_quantize(const void *x, roix_dtype dtype, uint64_t n, roix_scalars *sc, void *codes,
                          roix_stream_t stream) {
    const Range nvtx_range("roix_quantize");
    if (!sc) return invalid("sc is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (n == 0) return ROIX_OK;
    if (!x || !codes || !aligned16(x) || !aligned16(codes)) return invalid("x / codes must be 16-byte aligned");
    return cuda(launch_quantize(x, (int)dtype, n, sc, codes, (cudaStream_t)stream), "roix_quantize");
}

roix_status roix_histogram(const void *x, roix_dtype dtype, uint64_t n, roix_scalars *sc, uint64_t *hist,
                           uint32_t nbins, roix_stream_t stream) {
    const Range nvtx_range("roix_histogram");
    if (!sc || !hist) return invalid("sc / hist is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if ((dtype == ROIX_U16 && nbins != 65536) || (dtype == ROIX_F32 && nbins != 256))
        return invalid("nbins must be 65536 (u16) or 256 (fp32)");
    if (n == 0) return ROIX_OK;
    if (!x || !aligned16(x)) return invalid("x must be a 16-byte aligned device pointer");
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == ROIX_U16) return cuda(launch_hist_u16((const uint16_t *)x, n, sc, hist, st), "roix_histogram");
    return cuda(launch_hist_f32((const float *)x, n, sc, hist, st), "roix_histogram");
}

roix_status roix_histogram_clear(uint64_t *hist, uint64_t nbins, roix_stream_t stream) {
    if (nbins == 0) return ROIX_OK;
    if (!hist || !aligned16(hist)) return invalid("hist must be a 16-byte aligned device pointer");
    return cuda(launch_hist_clear(hist, nbins, (cudaStream_t)stream), "roix_histogram_clear");
}

roix_status roix_threshold(const uint64_t *hist, uint32_t nbins, roix_dtype dtype, roix_polarity polarity,
                           roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_threshold");
    if (!sc || !hist) return invalid("sc / hist is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if ((dtype == ROIX_U16 && nbins != 65536) || (dtype == ROIX_F32 && nbins != 256))
        return invalid("nbins must be 65536 (u16) or 256 (fp32)");
    if (polarity != ROIX_POL_HIGH && polarity != ROIX_POL_LOW) return invalid("polarity");
    return cuda(launch_threshold(hist, (int)dtype, (int)polarity, sc, (cudaStream_t)stream), "roix_threshold");
}

roix_status roix_threshold_multi(const uint64_t *hist, uint32_t nbins, roix_dtype dtype, roix_polarity polarity,
                                 uint32_t classes, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_threshold_multi");
    if (classes != 2 && classes != 3) return unsupported("classes must be 2 or 3");
    if (!sc || !hist) return invalid("sc / hist is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if ((dtype == ROIX_U16 && nbins != 65536) || (dtype == ROIX_F32 && nbins != 256))
        return invalid("nbins must be 65536 (u16) or 256 (fp32)");
    if (polarity != ROIX_POL_HIGH && polarity != ROIX_POL_LOW) return invalid("polarity");
    return cuda(launch_threshold(hist, (int)dtype, (int)polarity, sc, (cudaStream_t)stream, (int)classes),
                "roix_threshold_multi");
}

static roix_status check_halos(const roix_geom *g, uint32_t se, const uint32_t *lo, const uint32_t *hi) {
    if (se != 6) return ROIX_OK;
    if (g->z0 > 0 && !lo) return invalid("halo_lo required: the slab does not start at the volume face");
    if (g->z0 + g->nz < g->gz && !hi) return invalid("halo_hi required: the slab does not end at the volume face");
    return ROIX_OK;
}

roix_status roix_morph_workspace(const roix_geom *g, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    *ws_bytes = morph_workspace_bytes(*g);
    return ROIX_OK;
}

roix_status roix_morph_slots(const void *x, roix_dtype dtype, const roix_geom *g, uint32_t se, const uint32_t *halo_lo,
                             const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs,
                             uint32_t *run_slots, uint32_t slots_per_row, void *ws, size_t ws_bytes,
                             roix_stream_t stream) {
    const Range nvtx_range("roix_morph_slots");
    if (!sc || !o_bits || !ws) return invalid("sc / o_bits / ws is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (!geom_ok(g)) return invalid("geometry");
    if (se != 6 && se != 4) return unsupported("se must be 6 (3-D cross) or 4 (in-plane cross)");
    if (!x || !aligned16(x) || !aligned16(o_bits)) return invalid("x / o_bits must be 16-byte aligned");
    if (run_slots && (!row_runs || slots_per_row == 0 || slots_per_row > 64 || ((uintptr_t)run_slots & 7u)))
        return invalid("run_slots needs row_runs, 1 <= slots_per_row <= 64 and 8-byte alignment");
    roix_status s = check_halos(g, se, halo_lo, halo_hi);
    if (s != ROIX_OK) return s;
    if (g->nx > (1u << 30)) return unsupported("rows longer than 2^30 voxels");
    if (ws_bytes < morph_workspace_bytes(*g) || !aligned16(ws)) return invalid("workspace (see roix_morph_workspace)");
    return cuda(launch_morph(x, (int)dtype, *g, se, halo_lo, halo_hi, sc, o_bits, row_runs, ws, 0, (cudaStream_t)stream,
                             nullptr, (uint2 *)run_slots, run_slots ? slots_per_row : 0),
                "roix_morph");
}

roix_status roix_morph(const void *x, roix_dtype dtype, const roix_geom *g, uint32_t se, const uint32_t *halo_lo,
                       const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits, uint32_t *row_runs, void *ws,
                       size_t ws_bytes, roix_stream_t stream) {
    return roix_morph_slots(x, dtype, g, se, halo_lo, halo_hi, sc, o_bits, row_runs, nullptr, 0, ws, ws_bytes, stream);
}

roix_status roix_morph_frames(const uint16_t *x, const roix_geom *g, uint32_t se, const uint32_t *halo_lo,
                             const uint32_t *halo_hi, const roix_frame *frames, roix_scalars *sc, uint32_t *o_bits,
                             uint32_t *row_runs, void *ws, size_t ws_bytes, roix_stream_t stream) {
    const Range nvtx_range("roix_morph_frames");
    if (!sc || !o_bits || !ws || !frames) return invalid("sc / o_bits / ws / frames is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    if (se != 6 && se != 4) return unsupported("se must be 6 (3-D cross) or 4 (in-plane cross)");
    if (!x || !aligned16(x) || !aligned16(o_bits)) return invalid("x / o_bits must be 16-byte aligned");
    roix_status s = check_halos(g, se, halo_lo, halo_hi);
    if (s != ROIX_OK) return s;
    if (g->nx > (1u << 30)) return unsupported("rows longer than 2^30 voxels");
    if (ws_bytes < morph_workspace_bytes(*g) || !aligned16(ws)) return invalid("workspace (see roix_morph_workspace)");
    return cuda(launch_morph(x, ROIX_U16, *g, se, halo_lo, halo_hi, sc, o_bits, row_runs, ws, 0, (cudaStream_t)stream,
                             frames),
                "roix_morph_frames");
}

roix_status roix_background(const uint16_t *x, const uint16_t *B, const roix_geom *g, roix_bg_op op, uint16_t *out,
                            roix_stream_t stream) {
    const Range nvtx_range("roix_background");
    if (!geom_ok(g)) return invalid("geometry");
    if (op != ROIX_BG_SUB && op != ROIX_BG_REV && op != ROIX_BG_ADD) return invalid("op");
    if (g->nz * g->ny * g->nx == 0) return ROIX_OK;
    if (!x || !B || !out || !aligned16(x) || !aligned16(B) || !aligned16(out))
        return invalid("x / B / out must be 16-byte aligned device pointers");
    return cuda(launch_background(x, B, *g, (int)op, out, (cudaStream_t)stream), "roix_background");
}

roix_status roix_histogram_frames(const uint16_t *x, const roix_geom *g, roix_scalars *sc, uint64_t *hist,
                                  roix_stream_t stream) {
    const Range nvtx_range("roix_histogram_frames");
    if (!sc || !hist) return invalid("sc / hist is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    if (g->nz * g->ny * g->nx && (!x || !aligned16(x))) return invalid("x must be a 16-byte aligned device pointer");
    return cuda(launch_hist_u16_frames(x, g->nz, g->ny * g->nx, sc, hist, (cudaStream_t)stream),
                "roix_histogram_frames");
}

roix_status roix_threshold_frames(const uint64_t *hist, uint64_t nframes, roix_polarity polarity, uint32_t classes,
                                  roix_scalars *sc, roix_frame *frames, roix_stream_t stream) {
    const Range nvtx_range("roix_threshold_frames");
    if (classes != 2 && classes != 3) return unsupported("classes must be 2 or 3");
    if (!sc || (nframes && (!hist || !frames))) return invalid("sc / hist / frames is NULL");
    if (polarity != ROIX_POL_HIGH && polarity != ROIX_POL_LOW) return invalid("polarity");
    return cuda(launch_threshold_frames(hist, nframes, (int)polarity, (int)classes, sc, frames, (cudaStream_t)stream),
                "roix_threshold_frames");
}

roix_status roix_histogram_binarize_workspace(const roix_geom *g, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    *ws_bytes = fused_workspace_bytes(*g);
    return ROIX_OK;
}

roix_status roix_histogram_binarize(const void *x, roix_dtype dtype, const roix_geom *g, roix_polarity polarity,
                                    roix_scalars *sc, uint64_t *hist, uint32_t nbins, void *ws, size_t ws_bytes,
                                    roix_stream_t stream) {
    const Range nvtx_range("roix_histogram_binarize");
    if (!sc || !hist || !ws) return invalid("sc / hist / ws is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (!geom_ok(g)) return invalid("geometry");
    if ((dtype == ROIX_U16 && nbins != 65536) || (dtype == ROIX_F32 && nbins != 256))
        return invalid("nbins must be 65536 (u16) or 256 (fp32)");
    if (polarity != ROIX_POL_HIGH && polarity != ROIX_POL_LOW) return invalid("polarity");
    if (!x || !aligned16(x) || !aligned16(ws)) return invalid("x / ws must be 16-byte aligned");
    if (ws_bytes < fused_workspace_bytes(*g)) return invalid("workspace (see roix_histogram_binarize_workspace)");
    return cuda(launch_histogram_binarize(x, (int)dtype, *g, (int)polarity, sc, hist, ws, (cudaStream_t)stream),
                "roix_histogram_binarize");
}

roix_status roix_morph_prebinarized(const void *x, roix_dtype dtype, const roix_geom *g, uint32_t se,
                                    const uint32_t *halo_lo, const uint32_t *halo_hi, roix_scalars *sc, uint32_t *o_bits,
                                    uint32_t *row_runs, void *ws, size_t ws_bytes, roix_stream_t stream) {
    const Range nvtx_range("roix_morph_prebinarized");
    if (!sc || !o_bits || !ws) return invalid("sc / o_bits / ws is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (!geom_ok(g)) return invalid("geometry");
    if (se != 6 && se != 4) return unsupported("se must be 6 (3-D cross) or 4 (in-plane cross)");
    if (!x || !aligned16(x) || !aligned16(o_bits)) return invalid("x / o_bits must be 16-byte aligned");
    roix_status s = check_halos(g, se, halo_lo, halo_hi);
    if (s != ROIX_OK) return s;
    if (ws_bytes < fused_workspace_bytes(*g)) return invalid("workspace (see roix_histogram_binarize_workspace)");
    return cuda(launch_morph(x, (int)dtype, *g, se, halo_lo, halo_hi, sc, o_bits, row_runs, ws, 1, (cudaStream_t)stream),
                "roix_morph_prebinarized");
}

roix_status roix_binarize_planes(const void *x, roix_dtype dtype, const roix_geom *g, uint64_t p0, uint64_t np,
                                 roix_scalars *sc, uint32_t *m_bits, roix_stream_t stream) {
    const Range nvtx_range("roix_binarize_planes");
    if (!sc || !m_bits) return invalid("sc / m_bits is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (!geom_ok(g)) return invalid("geometry");
    if (p0 + np > g->nz) return invalid("planes outside the slab");
    if (np == 0) return ROIX_OK;
    if (!x || !aligned16(x)) return invalid("x must be 16-byte aligned");
    return cuda(launch_binarize_planes(x, (int)dtype, *g, p0, np, sc, m_bits, (cudaStream_t)stream),
                "roix_binarize_planes");
}

roix_status roix_label_workspace(const roix_geom *g, uint64_t run_capacity, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    if (run_capacity == 0 || run_capacity >= 0xffffffffull) return invalid("run_capacity must be in [1, 2^32-1)");
    if (g->nz * g->ny >= 0xffffffffull) return unsupported("more than 2^32-1 rows per slab");
    *ws_bytes = label_workspace_bytes(*g, run_capacity);
    return ROIX_OK;
}

roix_status roix_label_slots(const uint32_t *o_bits, const uint32_t *row_runs, const uint32_t *run_slots,
                             uint32_t slots_per_row, const roix_geom *g, uint32_t conn, uint64_t min_size,
                             uint64_t run_capacity, void *ws, size_t ws_bytes, const roix_label_out *out,
                             roix_scalars *sc, roix_stream_t stream) {
    if (!sc || !o_bits || !out || !ws) return invalid("sc / o_bits / out / ws is NULL");
    if (!aligned16(o_bits) || (out->keep_bits && !aligned16(out->keep_bits)) || (row_runs && !aligned16(row_runs)))
        return invalid("o_bits / keep_bits / row_runs must be 16-byte aligned");
    if (run_slots && (!row_runs || slots_per_row == 0 || slots_per_row > 64 || ((uintptr_t)run_slots & 7u)))
        return invalid("run_slots needs row_runs, 1 <= slots_per_row <= 64 and 8-byte alignment");
    if (!geom_ok(g)) return invalid("geometry");
    if (conn != 4 && conn != 8 && conn != 6 && conn != 18 && conn != 26) return unsupported("conn (4, 8, 6, 18, 26)");
    size_t need = 0;
    roix_status s = roix_label_workspace(g, run_capacity, &need);
    if (s != ROIX_OK) return s;
    if (ws_bytes < need) return invalid("workspace too small (see roix_label_workspace)");
    if (out->comp_min && (!out->comp_size || out->comp_cap == 0)) return invalid("comp_size / comp_cap");
    if (g->z0 != 0 || g->nz != g->gz) {
        if (conn != 4 && conn != 8) return unsupported("sharded 3-D labelling: use roix_label_local ... finish");
    }
    return cuda(launch_label(o_bits, row_runs, *g, conn, min_size, run_capacity, ws, *out, sc, (cudaStream_t)stream,
                             (const uint2 *)run_slots, run_slots ? slots_per_row : 0),
                "roix_label");
}

roix_status roix_label(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom *g, uint32_t conn,
                       uint64_t min_size, uint64_t run_capacity, void *ws, size_t ws_bytes,
                       const roix_label_out *out, roix_scalars *sc, roix_stream_t stream) {
    return roix_label_slots(o_bits, row_runs, nullptr, 0, g, conn, min_size, run_capacity, ws, ws_bytes, out, sc,
                            stream);
}

static roix_status label_common(const roix_geom *g, uint64_t cap, const void *ws, size_t ws_bytes) {
    if (!ws) return invalid("ws is NULL");
    size_t need = 0;
    roix_status s = roix_label_workspace(g, cap, &need);
    if (s != ROIX_OK) return s;
    if (ws_bytes < need) return invalid("workspace too small (see roix_label_workspace)");
    return ROIX_OK;
}

roix_status roix_label_local_slots(const uint32_t *o_bits, const uint32_t *row_runs, const uint32_t *run_slots,
                                   uint32_t slots_per_row, const roix_geom *g, uint32_t conn, uint64_t run_capacity,
                                   void *ws, size_t ws_bytes, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_label_local_slots");
    if (!sc || !o_bits) return invalid("sc / o_bits is NULL");
    if (!aligned16(o_bits) || (row_runs && !aligned16(row_runs)))
        return invalid("o_bits / row_runs must be 16-byte aligned");
    if (run_slots && (!row_runs || slots_per_row == 0 || slots_per_row > 64 || ((uintptr_t)run_slots & 7u)))
        return invalid("run_slots needs row_runs, 1 <= slots_per_row <= 64 and 8-byte alignment");
    if (conn != 4 && conn != 8 && conn != 6 && conn != 18 && conn != 26) return unsupported("conn (4, 8, 6, 18, 26)");
    roix_status s = label_common(g, run_capacity, ws, ws_bytes);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_local(o_bits, row_runs, *g, conn, run_capacity, ws, sc, (cudaStream_t)stream,
                                   (const uint2 *)run_slots, run_slots ? slots_per_row : 0),
                "roix_label_local");
}

roix_status roix_label_local(const uint32_t *o_bits, const uint32_t *row_runs, const roix_geom *g, uint32_t conn,
                             uint64_t run_capacity, void *ws, size_t ws_bytes, roix_scalars *sc,
                             roix_stream_t stream) {
    return roix_label_local_slots(o_bits, row_runs, nullptr, 0, g, conn, run_capacity, ws, ws_bytes, sc, stream);
}

roix_status roix_label_finish(const uint32_t *o_bits, const roix_geom *g, uint64_t min_size, uint64_t run_capacity,
                              void *ws, size_t ws_bytes, const uint64_t *map_label, const uint64_t *map_final,
                              const uint64_t *map_total, const uint64_t *nmap, const roix_label_out *out, roix_scalars *sc,
                              roix_stream_t stream) {
    const Range nvtx_range("roix_label_finish");
    if (!sc || !o_bits || !out) return invalid("sc / o_bits / out is NULL");
    if (nmap && (!map_label || !map_final || !map_total)) return invalid("merge map");
    if (out->comp_min && (!out->comp_size || out->comp_cap == 0)) return invalid("comp_size / comp_cap");
    if (min_size == ROIX_KEEP_LARGEST) return invalid("keep-largest on a sharded volume: use roix_label_finish_keep");
    roix_status s = label_common(g, run_capacity, ws, ws_bytes);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_finish(o_bits, *g, min_size, run_capacity, ws, map_label, map_final, map_total, nmap, *out,
                                    sc, (cudaStream_t)stream),
                "roix_label_finish");
}

roix_status roix_label_largest(void *ws, const roix_geom *g, uint64_t run_capacity, const uint64_t *map_label,
                               const uint64_t *map_final, const uint64_t *map_total, const uint64_t *nmap, uint32_t phase,
                               uint64_t *best, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_label_largest");
    if (!sc || !best) return invalid("sc / best is NULL");
    if (phase > 1) return invalid("phase must be 0 or 1");
    if (nmap && (!map_label || !map_final || !map_total)) return invalid("merge map");
    roix_status s = label_common(g, run_capacity, ws, (size_t)-1);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_largest(*g, run_capacity, ws, map_label, map_final, map_total, nmap, best, (int)phase, sc,
                                     (cudaStream_t)stream),
                "roix_label_largest");
}

roix_status roix_label_finish_keep(const uint32_t *o_bits, const roix_geom *g, uint64_t run_capacity, void *ws,
                                   size_t ws_bytes, const uint64_t *map_label, const uint64_t *map_final,
                                   const uint64_t *map_total, const uint64_t *nmap, const uint64_t *keep,
                                   const roix_label_out *out, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_label_finish_keep");
    if (!sc || !o_bits || !out || !keep) return invalid("sc / o_bits / out / keep is NULL");
    if (nmap && (!map_label || !map_final || !map_total)) return invalid("merge map");
    if (out->comp_min && (!out->comp_size || out->comp_cap == 0)) return invalid("comp_size / comp_cap");
    roix_status s = label_common(g, run_capacity, ws, ws_bytes);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_finish(o_bits, *g, 0, run_capacity, ws, map_label, map_final, map_total, nmap, *out, sc,
                                    (cudaStream_t)stream, keep),
                "roix_label_finish_keep");
}

roix_status roix_merge_workspace(uint32_t G, uint64_t root_cap, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (G == 0 || (uint64_t)G * root_cap >= 0xffffffffull) return invalid("G * root_cap must be in [1, 2^32-1)");
    *ws_bytes = merge_workspace_bytes(G, root_cap);
    return ROIX_OK;
}

roix_status roix_merge_device(const uint64_t *gathered, uint32_t G, uint64_t pair_cap, uint64_t root_cap,
                              uint64_t *map_label, uint64_t *map_final, uint64_t *map_total, uint64_t *nmap, void *ws,
                              size_t ws_bytes, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_merge_device");
    if (!gathered || !map_label || !map_final || !map_total || !nmap || !ws || !sc)
        return invalid("gathered / map / nmap / ws / sc is NULL");
    size_t need = 0;
    roix_status s = roix_merge_workspace(G, root_cap, &need);
    if (s != ROIX_OK) return s;
    if (ws_bytes < need || !aligned16(ws)) return invalid("workspace (see roix_merge_workspace)");
    return cuda(launch_merge(gathered, G, pair_cap, root_cap, map_label, map_final, map_total, nmap, ws, sc,
                             (cudaStream_t)stream),
                "roix_merge_device");
}

roix_status roix_label_boundary(const void *ws, const roix_geom *g, uint64_t run_capacity, int side, roix_brun *out,
                                uint64_t out_cap, uint64_t *count, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_label_boundary");
    if (!sc || !count || (out_cap && !out)) return invalid("sc / count / out is NULL");
    if (side != 0 && side != 1) return invalid("side must be 0 (first plane) or 1 (last plane)");
    roix_status s = label_common(g, run_capacity, ws, (size_t)-1);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_boundary(ws, *g, run_capacity, side, out, out_cap, count, sc, (cudaStream_t)stream),
                "roix_label_boundary");
}

roix_status roix_label_link(const void *ws, const roix_geom *g, uint64_t run_capacity, uint32_t conn,
                            const roix_brun *prev, const uint64_t *n_prev, uint64_t *pairs, uint64_t pair_cap,
                            uint64_t *n_pairs, roix_scalars *sc, roix_stream_t stream) {
    const Range nvtx_range("roix_label_link");
    if (!sc || !prev || !n_prev || !n_pairs || (pair_cap && !pairs)) return invalid("NULL pointer");
    if (conn != 6 && conn != 18 && conn != 26) return unsupported("cross-slab links need a 3-D conn (6, 18, 26)");
    roix_status s = label_common(g, run_capacity, ws, (size_t)-1);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_link(ws, *g, run_capacity, conn, prev, n_prev, pairs, pair_cap, n_pairs, sc,
                                  (cudaStream_t)stream),
                "roix_label_link");
}

roix_status roix_label_boundary_roots(const void *ws, const roix_geom *g, uint64_t run_capacity, uint64_t *labels,
                                      uint64_t *sizes, uint64_t out_cap, uint64_t *count, roix_scalars *sc,
                                      roix_stream_t stream) {
    const Range nvtx_range("roix_label_boundary_roots");
    if (!sc || !count || (out_cap && (!labels || !sizes))) return invalid("NULL pointer");
    roix_status s = label_common(g, run_capacity, ws, (size_t)-1);
    if (s != ROIX_OK) return s;
    return cuda(launch_label_boundary_roots(ws, *g, run_capacity, labels, sizes, out_cap, count, sc,
                                            (cudaStream_t)stream),
                "roix_label_boundary_roots");
}

// Host union-find over the boundary components of all slabs: union by minimum label, so every
// merged component is named by its minimum global linear index (G-14) whatever the pair order.
roix_status roix_merge(const uint64_t *pairs, uint64_t npairs, const uint64_t *labels, const uint64_t *sizes,
                       uint64_t nlabels, uint64_t *out_label, uint64_t *out_final, uint64_t *out_total,
                       uint64_t *nout) {
    if (!nout || (nlabels && (!labels || !sizes || !out_label || !out_final || !out_total)) || (npairs && !pairs))
        return invalid("NULL pointer");
    std::vector<std::pair<uint64_t, uint64_t>> ls(nlabels);
    for (uint64_t i = 0; i < nlabels; i++) ls[i] = {labels[i], sizes[i]};
    std::sort(ls.begin(), ls.end());
    std::vector<uint64_t> L, S;
    for (auto &p : ls)
        if (L.empty() || L.back() != p.first) {
            L.push_back(p.first);
            S.push_back(p.second);
        }
    const size_t m = L.size();
    std::vector<uint64_t> parent(m);
    for (size_t i = 0; i < m; i++) parent[i] = i;
    auto find = [&](uint64_t a) {
        while (parent[a] != a) {
            parent[a] = parent[parent[a]];
            a = parent[a];
        }
        return a;
    };
    auto index = [&](uint64_t lab, uint64_t *out) {
        auto it = std::lower_bound(L.begin(), L.end(), lab);
        if (it == L.end() || *it != lab) return false;
        *out = (uint64_t)(it - L.begin());
        return true;
    };
    for (uint64_t k = 0; k < npairs; k++) {
        uint64_t a, b;
        if (!index(pairs[2 * k], &a) || !index(pairs[2 * k + 1], &b)) return invalid("pair label not in the tables");
        a = find(a);
        b = find(b);
        if (a == b) continue;
        if (a < b) parent[b] = a;   // indices are in label order: the smaller label wins
        else parent[a] = b;
    }
    std::vector<uint64_t> tot(m, 0);
    for (size_t i = 0; i < m; i++) tot[find(i)] += S[i];
    for (size_t i = 0; i < m; i++) {
        const uint64_t r = find(i);
        out_label[i] = L[i];
        out_final[i] = L[r];
        out_total[i] = tot[r];
    }
    *nout = m;
    return ROIX_OK;
}

roix_status roix_extract_workspace(uint64_t n, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    *ws_bytes = extract_workspace_bytes(n);
    return ROIX_OK;
}

roix_status roix_extract(const void *x, roix_dtype dtype, uint64_t n, const uint32_t *keep_bits, roix_scalars *sc,
                         void *codes_out, uint64_t capacity, const uint64_t *offset, void *ws, size_t ws_bytes,
                         roix_stream_t stream) {
    const Range nvtx_range("roix_extract");
    if (!sc || !keep_bits || !ws) return invalid("sc / keep_bits / ws is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (n == 0) return ROIX_OK;
    if (!x || !aligned16(x)) return invalid("x must be 16-byte aligned");
    if (!aligned16(keep_bits)) return invalid("keep_bits must be 16-byte aligned");
    if (capacity > 0 && (!codes_out || !aligned16(codes_out))) return invalid("codes_out must be 16-byte aligned");
    if (ws_bytes < extract_workspace_bytes(n)) return invalid("workspace too small (see roix_extract_workspace)");
    return cuda(launch_extract(x, (int)dtype, n, keep_bits, sc, codes_out, capacity, offset, ws, (cudaStream_t)stream),
                "roix_extract");
}

roix_status roix_extract_runs(const void *x, roix_dtype dtype, const roix_geom *g, uint64_t run_capacity, void *ws,
                              size_t ws_bytes, roix_scalars *sc, void *codes_out, uint64_t capacity,
                              const uint64_t *offset, roix_stream_t stream) {
    const Range nvtx_range("roix_extract_runs");
    if (!sc) return invalid("sc is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    roix_status s = label_common(g, run_capacity, ws, ws_bytes);
    if (s != ROIX_OK) return s;
    if (!x || !aligned16(x)) return invalid("x must be 16-byte aligned");
    if (capacity > 0 && (!codes_out || !aligned16(codes_out))) return invalid("codes_out must be 16-byte aligned");
    return cuda(launch_extract_runs(x, (int)dtype, *g, run_capacity, ws, sc, codes_out, capacity, offset,
                                    (cudaStream_t)stream),
                "roix_extract_runs");
}

roix_status roix_row_spans_workspace(const roix_geom *g, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    if (g->nz * g->ny >= 0xffffffffull) return unsupported("more than 2^32-1 rows per slab");
    if (g->nx >= 0xffffffffull) return unsupported("rows longer than 2^32-1 voxels");
    *ws_bytes = row_spans_workspace_bytes(*g);
    return ROIX_OK;
}

roix_status roix_row_spans(const uint32_t *keep_bits, const void *x, roix_dtype dtype, const roix_geom *g,
                           roix_scalars *sc, roix_span *spans, uint64_t span_cap, void *codes, uint64_t code_cap,
                           uint64_t *counts, void *ws, size_t ws_bytes, roix_stream_t stream) {
    const Range nvtx_range("roix_row_spans");
    if (!sc || !keep_bits || !counts || !ws) return invalid("sc / keep_bits / counts / ws is NULL");
    if (!aligned16(keep_bits)) return invalid("keep_bits must be 16-byte aligned");
    if (!dtype_ok(dtype)) return invalid("dtype");
    size_t need = 0;
    roix_status s = roix_row_spans_workspace(g, &need);
    if (s != ROIX_OK) return s;
    if (ws_bytes < need) return invalid("workspace too small (see roix_row_spans_workspace)");
    if (!x || !aligned16(x)) return invalid("x must be 16-byte aligned");
    if ((span_cap && !spans) || (code_cap && !codes)) return invalid("spans / codes is NULL");
    return cuda(launch_row_spans(keep_bits, x, (int)dtype, *g, sc, spans, span_cap, codes, code_cap, counts, ws,
                                 (cudaStream_t)stream),
                "roix_row_spans");
}

roix_status roix_greedy_workspace(uint64_t n, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    *ws_bytes = greedy_workspace_bytes(n);
    return ROIX_OK;
}

roix_status roix_greedy_quantize(const uint16_t *D, uint64_t n, double E, uint32_t qmax, uint16_t *Q, uint32_t *group_bits,
                                 uint64_t *ngroups, void *ws, size_t ws_bytes, roix_stream_t stream) {
    const Range nvtx_range("roix_greedy_quantize");
    if (!ngroups || !ws || !group_bits) return invalid("ngroups / group_bits / ws is NULL");
    if (!(E >= 0.0) || !std::isfinite(E)) return invalid("E must be finite and >= 0");
    if (qmax > 65535) return invalid("qmax must be <= 65535");
    if (n && (!D || !Q)) return invalid("D / Q is NULL");
    if (ws_bytes < greedy_workspace_bytes(n)) return invalid("workspace too small (see roix_greedy_workspace)");
    return cuda(launch_greedy(D, n, E, qmax, Q, group_bits, ngroups, ws, (cudaStream_t)stream), "roix_greedy_quantize");
}

roix_status roix_decode_workspace(uint64_t n, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    *ws_bytes = decode_workspace_bytes(n);
    return ROIX_OK;
}

roix_status roix_decode(const uint32_t *keep_bits, const void *codes, uint64_t ncodes, roix_dtype dtype, uint64_t n,
                        roix_scalars *sc, void *xhat, void *ws, size_t ws_bytes, roix_stream_t stream) {
    const Range nvtx_range("roix_decode");
    if (!sc || !ws) return invalid("sc / ws is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    if (ws_bytes < decode_workspace_bytes(n)) return invalid("workspace too small (see roix_decode_workspace)");
    if (n && (!keep_bits || !aligned16(keep_bits) || !xhat || !aligned16(xhat)))
        return invalid("keep_bits / xhat must be 16-byte aligned device pointers");
    if (ncodes && (!codes || !aligned16(codes))) return invalid("codes must be a 16-byte aligned device pointer");
    return cuda(launch_decode(keep_bits, codes, ncodes, (int)dtype, n, sc, xhat, ws, (cudaStream_t)stream),
                "roix_decode");
}

roix_status roix_decode_spans_workspace(const roix_geom *g, size_t *ws_bytes) {
    if (!ws_bytes) return invalid("ws_bytes is NULL");
    if (!geom_ok(g)) return invalid("geometry");
    if (g->nz * g->ny >= 0xffffffffull) return unsupported("more than 2^32-1 rows per slab");
    if (g->nx >= 0xffffffffull) return unsupported("rows longer than 2^32-1 voxels");
    *ws_bytes = decode_spans_workspace_bytes(*g);
    return ROIX_OK;
}

roix_status roix_decode_spans(const roix_span *spans, uint64_t span_cap, const void *codes, uint64_t code_cap,
                              const uint64_t *counts, roix_dtype dtype, const roix_geom *g, roix_scalars *sc,
                              void *xhat, void *ws, size_t ws_bytes, roix_stream_t stream) {
    const Range nvtx_range("roix_decode_spans");
    if (!sc || !counts || !ws) return invalid("sc / counts / ws is NULL");
    if (!dtype_ok(dtype)) return invalid("dtype");
    size_t need = 0;
    roix_status s = roix_decode_spans_workspace(g, &need);
    if (s != ROIX_OK) return s;
    if (ws_bytes < need) return invalid("workspace too small (see roix_decode_spans_workspace)");
    if (!xhat || !aligned16(xhat)) return invalid("xhat must be a 16-byte aligned device pointer");
    if ((span_cap && !spans) || (code_cap && !codes)) return invalid("spans / codes is NULL");
    return cuda(launch_decode_spans(spans, span_cap, codes, code_cap, counts, (int)dtype, *g, sc, xhat, ws,
                                    (cudaStream_t)stream),
                "roix_decode_spans");
}

roix_status roix_confusion(const uint32_t *pred_bits, const uint32_t *truth_bits, uint64_t n, uint64_t *counts,
                           roix_stream_t stream) {
    const Range nvtx_range("roix_confusion");
    if (!counts) return invalid("counts is NULL");
    if (n && (!pred_bits || !truth_bits || !aligned16(pred_bits) || !aligned16(truth_bits)))
        return invalid("pred_bits / truth_bits must be 16-byte aligned device pointers");
    return cuda(launch_confusion(pred_bits, truth_bits, n, counts, (cudaStream_t)stream), "roix_confusion");
}

static double ratio128(__int128 num, __int128 den) {
    if (den == 0) return std::nan("");
    return (double)((long double)num / (long double)den);
}

roix_status roix_overlap_metrics(const uint64_t *counts, double *out) {
    const Range nvtx_range("roix_overlap_metrics");
    if (!counts || !out) return invalid("counts / out is NULL");
    const __int128 tp = counts[0], fp = counts[1], fn = counts[2], tn = counts[3];
    const __int128 N = tp + fp + fn + tn;
    out[0] = ratio128(2 * tp, 2 * tp + fp + fn);   // Eq. 7 DSC
    out[1] = ratio128(tp, tp + fp + fn);           // Eq. 8 IoU
    out[2] = ratio128(tp, tp + fn);                // Eq. 9 sensitivity
    out[3] = ratio128(tn, tn + fp);                // Eq. 10 specificity
    out[4] = ratio128(tp + tn, N);                 // Eq. 11 accuracy
    // Eq. 12-13: kappa = ((tp+tn) - S/N) / (N - S/N) = (N(tp+tn) - S) / (N^2 - S), S = N f_c
    const __int128 S = (tn + fn) * (tn + fp) + (fp + tp) * (fn + tp);
    out[5] = N == 0 ? std::nan("") : ratio128(N * (tp + tn) - S, N * N - S);
    // Eq. 14: auc = 1 - (fp/(fp+tn) + fn/(fn+tp))/2 = (2AB - fp B - fn A) / (2AB), A = fp+tn, B = fn+tp
    const __int128 A = fp + tn, B = fn + tp;
    out[6] = (A == 0 || B == 0) ? std::nan("") : ratio128(2 * A * B - fp * B - fn * A, 2 * A * B);
    return ROIX_OK;
}

}  // extern "C"
