// synth.cu -- seeded synthetic X-CT phantoms (the input recipe of DESIGN.md §5).
//
// This is the INPUT GENERATOR shared by the product tests/bench and the oracle tests.  It holds
// none of the method's arithmetic (no quantiser, histogram, threshold, morphology or labelling).
// Every voxel value is a pure function of (config, seed, object list, global linear index), so a
// z-slab generated on any rank is bit-identical to the same planes of the whole volume.
//
// Randomness: Philox4x32-10 (Salmon et al., SC'11) with counter = (i_lo, i_hi, stream, 0) and
// key = (seed, 0x524f4958 "ROIX"); Gaussians by Box-Muller on two 24-bit uniforms.
#include <cstdint>
#include <cuda_runtime.h>

extern "C" {

struct synth_obj {        // an ellipsoid: centre, rotation R (row-major, body->world), 1/r^2
    float c[3];           // (z, y, x) in voxel units of the GLOBAL volume
    float R[9];
    float inv_r2[3];
    float mu;             // object intensity parameter
    float bbox[6];        // zlo, zhi, ylo, yhi, xlo, xhi (inclusive, voxel units)
};

struct synth_params {
    int mode;             // 1 ell_poisson (C1), 2 ell_gauss (C5), 3 f32 texture (C2), 4 frames (C3), 5 cyl+pores (C4),
                          // 6 the C3 flat field without the sample (a noise-free calibration frame)
    uint32_t seed;
    uint64_t gz, ny, nx;  // global volume
    uint64_t z0, nz;      // slab to generate
    int nobj;
    const synth_obj *obj; // device
    float p[16];          // mode parameters
    int nring;
    const float *ring;    // device: (R_j, w_j, sigma_j) triples
    uint32_t *truth;      // device, optional (NULL): ground-truth ROI bits of the slab, packed like the
                          // product's masks (bit i%32 of word i/32, slab-local i); the caller zeroes it
};
}

namespace {

__device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                                       uint32_t out[4]) {
#pragma unroll
    for (int r = 0; r < 10; r++) {
        uint32_t hi0 = __umulhi(0xD2511F53u, c0), lo0 = 0xD2511F53u * c0;
        uint32_t hi1 = __umulhi(0xCD9E8D57u, c2), lo1 = 0xCD9E8D57u * c2;
        uint32_t n0 = hi1 ^ c1 ^ k0, n2 = hi0 ^ c3 ^ k1;
        c0 = n0; c1 = lo1; c2 = n2; c3 = lo0;
        k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
    }
    out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

__device__ __forceinline__ float u24(uint32_t r) { return (float)(r >> 8) * (1.0f / 16777216.0f); }

// two standard normals for voxel i in stream s
__device__ __forceinline__ void normals(uint64_t i, uint32_t s, uint32_t seed, float &z1, float &z2) {
    uint32_t r[4];
    philox((uint32_t)i, (uint32_t)(i >> 32), s, 0u, seed, 0x524f4958u, r);
    float u1 = ((float)(r[0] >> 8) + 1.0f) * (1.0f / 16777216.0f);  // (0, 1]
    float u2 = u24(r[1]);
    float rad = sqrtf(-2.0f * logf(u1));
    float sn, cs;
    sincospif(2.0f * u2, &sn, &cs);
    z1 = rad * cs;
    z2 = rad * sn;
}

__device__ __forceinline__ float hash_unit(uint32_t a, uint32_t b, uint32_t c, uint32_t seed) {
    uint32_t r[4];
    philox(a, b, c, 0x7e57u, seed, 0x4c415454u, r);
    return u24(r[0]);
}

__device__ __forceinline__ bool inside(const synth_obj &o, float z, float y, float x) {
    float dz = z - o.c[0], dy = y - o.c[1], dx = x - o.c[2];
    // body coordinates q = R^T d
    float q0 = o.R[0] * dz + o.R[3] * dy + o.R[6] * dx;
    float q1 = o.R[1] * dz + o.R[4] * dy + o.R[7] * dx;
    float q2 = o.R[2] * dz + o.R[5] * dy + o.R[8] * dx;
    return q0 * q0 * o.inv_r2[0] + q1 * q1 * o.inv_r2[1] + q2 * q2 * o.inv_r2[2] <= 1.0f;
}

__device__ __forceinline__ float smooth(float t) { return t * t * (3.0f - 2.0f * t); }

// value noise in [-1, 1]: hashed lattice values, trilinear interpolation with smoothstep weights
__device__ float value_noise(float z, float y, float x, float cell, uint32_t oct, uint32_t seed) {
    float fz = z / cell, fy = y / cell, fx = x / cell;
    float iz = floorf(fz), iy = floorf(fy), ix = floorf(fx);
    float tz = smooth(fz - iz), ty = smooth(fy - iy), tx = smooth(fx - ix);
    float acc = 0.0f;
#pragma unroll
    for (int c = 0; c < 8; c++) {
        int dz = c >> 2, dy = (c >> 1) & 1, dx = c & 1;
        float w = (dz ? tz : 1.0f - tz) * (dy ? ty : 1.0f - ty) * (dx ? tx : 1.0f - tx);
        uint32_t a = (uint32_t)((int)iz + dz) + oct * 0x10000u, b = (uint32_t)((int)iy + dy), d = (uint32_t)((int)ix + dx);
        acc += w * (2.0f * hash_unit(a, b, d, seed) - 1.0f);
    }
    return acc;
}

__device__ __forceinline__ uint16_t clamp_u16(float v, float hi) {
    v = rintf(v);
    v = fminf(fmaxf(v, 0.0f), hi);
    return (uint16_t)v;
}

constexpr int MAXL = 256;  // objects kept per row after culling

// One CTA per (z, y) row of the slab.  Objects whose bounding box contains the row are collected
// in order (painter's order: the later object wins) into shared memory.
__global__ void synth_rows(synth_params P, void *out) {
    __shared__ int list[MAXL];
    __shared__ int nlist;
    const uint64_t row = blockIdx.x + (uint64_t)blockIdx.y * gridDim.x;
    if (row >= P.nz * P.ny) return;
    const uint64_t zl = row / P.ny, y = row % P.ny, z = P.z0 + zl;
    const float fz = (float)z, fy = (float)y;
    if (threadIdx.x == 0) nlist = 0;
    __syncthreads();
    if (P.mode != 4) {
        // ordered compaction, one warp
        if (threadIdx.x < 32) {
            int base = 0;
            int lo = 0, hi = P.nobj;
            if (P.mode == 5) {  // pores sorted by centre z; only |cz - z| <= p[5] can touch this row
                float zr = P.p[5];
                int a = 0, b = P.nobj;
                while (a < b) { int m = (a + b) / 2; if (P.obj[m].c[0] < fz - zr) a = m + 1; else b = m; }
                lo = a;
                a = lo; b = P.nobj;
                while (a < b) { int m = (a + b) / 2; if (P.obj[m].c[0] <= fz + zr) a = m + 1; else b = m; }
                hi = a;
            }
            for (int k0 = lo; k0 < hi; k0 += 32) {
                int k = k0 + threadIdx.x;
                bool hit = false;
                if (k < hi) {
                    const synth_obj &o = P.obj[k];
                    hit = fz >= o.bbox[0] && fz <= o.bbox[1] && fy >= o.bbox[2] && fy <= o.bbox[3];
                }
                unsigned b = __ballot_sync(0xffffffffu, hit);
                if (hit) {
                    int pos = base + __popc(b & ((1u << threadIdx.x) - 1u));
                    if (pos < MAXL) list[pos] = k;
                }
                base += __popc(b);
            }
            if (threadIdx.x == 0) nlist = base < MAXL ? base : MAXL;
        }
        __syncthreads();
    }
    const int nl = nlist;
    const uint64_t rowbase = row * P.nx;                       // slab-local linear index of x = 0
    const uint64_t gbase = (z * P.ny + y) * P.nx;              // global linear index of x = 0
    for (uint64_t x0 = 0; x0 < P.nx; x0 += blockDim.x) {
        const uint64_t x = x0 + threadIdx.x;
        const bool valid = x < P.nx;
        bool truth = false;   // ground truth: the voxel belongs to the phantom's region of interest
        const uint64_t gi = gbase + x;
        const float fx = (float)x;
        float z1, z2;
        normals(gi, 0u, P.seed, z1, z2);
        int hit = -1;
        if (P.mode == 5) {
            for (int k = 0; k < nl; k++) {
                const synth_obj &o = P.obj[list[k]];
                if (fx >= o.bbox[4] && fx <= o.bbox[5] && inside(o, fz, fy, fx)) { hit = list[k]; break; }
            }
        } else if (P.mode != 4) {
            for (int k = nl - 1; k >= 0; k--) {
                const synth_obj &o = P.obj[list[k]];
                if (fx >= o.bbox[4] && fx <= o.bbox[5] && inside(o, fz, fy, fx)) { hit = list[k]; break; }
            }
        }
        switch (P.mode) {
        case 1: {  // C1: Poisson(lambda) ~ lambda + sqrt(lambda) z2, 12-bit
            float lam = hit < 0 ? P.p[0] + P.p[1] * z1 : P.obj[hit].mu + P.p[2] * z1;
            lam = fmaxf(lam, 0.0f);
            if (valid) ((uint16_t *)out)[rowbase + x] = clamp_u16(lam + sqrtf(lam) * z2, P.p[3]);
            truth = hit >= 0;
        } break;
        case 2: {  // C5: Gaussian background / inclusions, 16-bit
            float v = (hit < 0 ? P.p[0] : P.obj[hit].mu) + P.p[1] * z1;
            if (valid) ((uint16_t *)out)[rowbase + x] = clamp_u16(v, 65535.0f);
            truth = hit >= 0;
        } break;
        case 3: {  // C2: fp32 attenuation, textured objects, ring artefacts
            float v;
            if (hit < 0) v = P.p[0] + P.p[1] * z1;
            else {
                float t = (4.0f / 7.0f) * value_noise(fz, fy, fx, 32.0f, 0u, P.seed) +
                          (2.0f / 7.0f) * value_noise(fz, fy, fx, 16.0f, 1u, P.seed) +
                          (1.0f / 7.0f) * value_noise(fz, fy, fx, 8.0f, 2u, P.seed);
                v = P.obj[hit].mu + P.p[2] * t;
            }
            float dy = fy - P.p[3], dx = fx - P.p[4];
            float rho = sqrtf(dy * dy + dx * dx);
            float ring = 0.0f;
            for (int j = 0; j < P.nring; j++)
                if (fabsf(rho - P.ring[3 * j]) <= 0.5f * P.ring[3 * j + 1]) ring += P.ring[3 * j + 2];
            if (valid) ((float *)out)[rowbase + x] = v + P.p[5] * ring;
            truth = hit >= 0;
        } break;
        case 4: {  // C3: detector frames, flat field with a rotating elliptical sample shadow
            float g = 0.97f + 0.06f * hash_unit((uint32_t)y, (uint32_t)x, 0x6a1u, P.seed);
            float th = 3.14159265358979f * fz / P.p[0];
            float A = P.p[1], Bh = P.p[2];
            float a = sqrtf(A * A * cosf(th) * cosf(th) + Bh * Bh * sinf(th) * sinf(th));
            float ry = (fy - P.p[4]) / P.p[3], rx = (fx - P.p[5]) / a;
            float r2 = ry * ry + rx * rx;
            float E = r2 < 1.0f ? g * (P.p[6] - P.p[7] * sqrtf(1.0f - r2)) : P.p[8] * g;
            if (valid) ((uint16_t *)out)[rowbase + x] = clamp_u16(E + sqrtf(E) * z1, P.p[9]);
            truth = r2 < 1.0f;   // the sample's shadow
        } break;
        case 6: {  // C3 calibration: the gain-varied open beam, no sample, no noise
            float g = 0.97f + 0.06f * hash_unit((uint32_t)y, (uint32_t)x, 0x6a1u, P.seed);
            if (valid) ((uint16_t *)out)[rowbase + x] = clamp_u16(P.p[8] * g, P.p[9]);
        } break;
        case 5: {  // C4: porous cylinder in air
            float dy = fy - P.p[0], dx = fx - P.p[1];
            float v;
            const bool cyl = dy * dy + dx * dx <= P.p[2] * P.p[2];
            if (cyl) v = hit >= 0 ? 300.0f + 50.0f * z1 : 2500.0f + 100.0f * z1;
            else v = 200.0f + 40.0f * z1;
            if (valid) ((uint16_t *)out)[rowbase + x] = clamp_u16(v, 65535.0f);
            truth = cyl && hit < 0;   // the solid matrix (pores and air are background)
        } break;
        }
        if (P.truth) {   // 32 consecutive voxels per warp: their bits land in at most two words
            const unsigned b = __ballot_sync(0xffffffffu, valid && truth);
            if ((threadIdx.x & 31u) == 0 && b) {
                const uint64_t li = rowbase + x;
                const uint32_t sh = (uint32_t)(li & 31);
                atomicOr(&P.truth[li >> 5], b << sh);
                if (sh && (b >> (32 - sh))) atomicOr(&P.truth[(li >> 5) + 1], b >> (32 - sh));
            }
        }
    }
}

}  // namespace

extern "C" int synth_generate(const synth_params *P, void *out, void *stream) {
    uint64_t rows = P->nz * P->ny;
    if (rows == 0) return 0;
    dim3 grid((unsigned)(rows < 65535 ? rows : 65535), (unsigned)((rows + 65534) / 65535));
    synth_rows<<<grid, 256, 0, (cudaStream_t)stream>>>(*P, out);
    return (int)cudaGetLastError();
}

extern "C" int synth_obj_size(void) { return (int)sizeof(synth_obj); }
