// k_background.cu -- NEXT-3 background subtraction (M(x, y) = I(x, y) - B(x, y), "a
// pixel-by-pixel subtraction from the original"; SPEC S:61-69 clamps at 0) and its inverse for the
// reconstruction ("combined with the precomputed background"), on uint16 frame stacks: one
// reference frame B[Y][X] for every frame z of x[Z][Y][X].
//   ROIX_BG_SUB  max(0, I - B)    ROIX_BG_REV  max(0, B - I)    ROIX_BG_ADD  min(65535, I + B)
// Per 32-bit word the two halves go through the saturating SIMD ops __vsubus2 / __vaddus2.  Frames that
// are whole 16-byte units (Y X % 8 == 0): 16-byte vectors, B read once (k_background_vec); else one CTA
// row per frame (blockIdx.y) voxel by voxel.
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

template <int OP>
__device__ __forceinline__ uint32_t bg_word(uint32_t x, uint32_t b) {
    if constexpr (OP == ROIX_BG_SUB) return __vsubus2(x, b);
    else if constexpr (OP == ROIX_BG_REV) return __vsubus2(b, x);
    else return __vaddus2(x, b);
}

// Thread = one 16-byte group i of the frame, looping over every frame z: B[i] is loaded once and
// reused (a C3 frame is 270 MB, twice the L2: a frame-major order would re-read B from HBM per frame).
// Four frames in flight per thread.
template <int OP>
__global__ void __launch_bounds__(256) k_background_vec(const uint16_t *x, const uint16_t *__restrict__ B,
                                                        uint64_t A, uint64_t nz, uint16_t *out) {
    const uint64_t n8 = A / 8, A8 = A / 8;
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x);
    const uint4 *b4 = reinterpret_cast<const uint4 *>(B);
    uint4 *o4 = reinterpret_cast<uint4 *>(out);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 b = __ldcs(b4 + i);
        uint64_t z = 0;
        for (; z + 4 <= nz; z += 4) {
            uint4 v[4];
#pragma unroll
            for (int k = 0; k < 4; k++) v[k] = __ldcs(x4 + (z + k) * A8 + i);
#pragma unroll
            for (int k = 0; k < 4; k++)
                __stcs(o4 + (z + k) * A8 + i, make_uint4(bg_word<OP>(v[k].x, b.x), bg_word<OP>(v[k].y, b.y),
                                                         bg_word<OP>(v[k].z, b.z), bg_word<OP>(v[k].w, b.w)));
        }
        for (; z < nz; z++) {
            const uint4 v = __ldcs(x4 + z * A8 + i);
            __stcs(o4 + z * A8 + i, make_uint4(bg_word<OP>(v.x, b.x), bg_word<OP>(v.y, b.y), bg_word<OP>(v.z, b.z),
                                               bg_word<OP>(v.w, b.w)));
        }
    }
}

template <int OP>
__global__ void __launch_bounds__(256) k_background_scalar(const uint16_t *x,
                                                           const uint16_t *__restrict__ B, uint64_t A, uint16_t *out) {
    const uint64_t z = blockIdx.y;
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < A; i += (uint64_t)gridDim.x * blockDim.x)
        out[z * A + i] = (uint16_t)bg_word<OP>(x[z * A + i], B[i]);
}

}  // namespace roix

using namespace roix;

cudaError_t launch_background(const uint16_t *x, const uint16_t *B, const roix_geom &g, int op, uint16_t *out,
                              cudaStream_t st) {
    const uint64_t A = g.ny * g.nx;
    if (A == 0 || g.nz == 0) return cudaSuccess;
    if (A % 8 == 0) {
        const unsigned grid = (unsigned)max((uint64_t)1, min((A / 8 + 255) / 256, (uint64_t)num_sms() * 8));
        switch (op) {
        case ROIX_BG_SUB: k_background_vec<ROIX_BG_SUB><<<grid, 256, 0, st>>>(x, B, A, g.nz, out); break;
        case ROIX_BG_REV: k_background_vec<ROIX_BG_REV><<<grid, 256, 0, st>>>(x, B, A, g.nz, out); break;
        default: k_background_vec<ROIX_BG_ADD><<<grid, 256, 0, st>>>(x, B, A, g.nz, out); break;
        }
        return cudaGetLastError();
    }
    const uint64_t target = (uint64_t)num_sms() * 8;   // CTAs over all frames
    const unsigned per = (unsigned)max((uint64_t)1, min((A + 255) / 256, (target + g.nz - 1) / g.nz));
    for (uint64_t z0 = 0; z0 < g.nz; z0 += 65535) {
        const dim3 grid(per, (unsigned)min(g.nz - z0, (uint64_t)65535));
        const uint16_t *xz = x + z0 * A;
        uint16_t *oz = out + z0 * A;
        switch (op) {
        case ROIX_BG_SUB: k_background_scalar<ROIX_BG_SUB><<<grid, 256, 0, st>>>(xz, B, A, oz); break;
        case ROIX_BG_REV: k_background_scalar<ROIX_BG_REV><<<grid, 256, 0, st>>>(xz, B, A, oz); break;
        default: k_background_scalar<ROIX_BG_ADD><<<grid, 256, 0, st>>>(xz, B, A, oz); break;
        }
    }
    return cudaGetLastError();
}
