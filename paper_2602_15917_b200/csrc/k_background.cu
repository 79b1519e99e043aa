// k_background.cu -- NEXT-3 background subtraction (M(x, y) = I(x, y) - B(x, y), "a
// pixel-by-pixel subtraction from the original"; SPEC S:61-69 clamps at 0) and its inverse for the
// reconstruction ("combined with the precomputed background"), on uint16 frame stacks: one
// reference frame B[Y][X] for every frame z of x[Z][Y][X].
//   ROIX_BG_SUB  max(0, I - B)    ROIX_BG_REV  max(0, B - I)    ROIX_BG_ADD  min(65535, I + B)
// Per 32-bit word the two halves go through the saturating SIMD ops __vsubus2 / __vaddus2.  One CTA row
// per frame (blockIdx.y), so B is indexed by the offset inside the frame (no division); 16-byte
// vectors when frames are whole 16-byte units (Y X % 8 == 0), else voxel by voxel.
#include "common.cuh"
#include "kernels.cuh"

namespace roix {

template <int OP>
__device__ __forceinline__ uint32_t bg_word(uint32_t x, uint32_t b) {
    if constexpr (OP == ROIX_BG_SUB) return __vsubus2(x, b);
    else if constexpr (OP == ROIX_BG_REV) return __vsubus2(b, x);
    else return __vaddus2(x, b);
}

template <int OP>
__global__ void __launch_bounds__(256) k_background_vec(const uint16_t *__restrict__ x, const uint16_t *__restrict__ B,
                                                        uint64_t A, uint16_t *out) {
    const uint64_t z = blockIdx.y, n8 = A / 8;
    const uint4 *x4 = reinterpret_cast<const uint4 *>(x + z * A);
    const uint4 *b4 = reinterpret_cast<const uint4 *>(B);
    uint4 *o4 = reinterpret_cast<uint4 *>(out + z * A);
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n8; i += (uint64_t)gridDim.x * blockDim.x) {
        const uint4 v = __ldcs(x4 + i), b = __ldg(b4 + i);
        __stcs(o4 + i, make_uint4(bg_word<OP>(v.x, b.x), bg_word<OP>(v.y, b.y), bg_word<OP>(v.z, b.z),
                                  bg_word<OP>(v.w, b.w)));
    }
}

template <int OP>
__global__ void __launch_bounds__(256) k_background_scalar(const uint16_t *__restrict__ x,
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
    const bool vec = A % 8 == 0;
    const uint64_t work = vec ? A / 8 : A;
    const uint64_t target = (uint64_t)num_sms() * 8;   // CTAs over all frames
    const unsigned per = (unsigned)max((uint64_t)1, min((work + 255) / 256, (target + g.nz - 1) / g.nz));
    for (uint64_t z0 = 0; z0 < g.nz; z0 += 65535) {
        const dim3 grid(per, (unsigned)min(g.nz - z0, (uint64_t)65535));
        const uint16_t *xz = x + z0 * A;
        uint16_t *oz = out + z0 * A;
#define ROIX_BG(OP)                                                                       \
    if (vec) k_background_vec<OP><<<grid, 256, 0, st>>>(xz, B, A, oz);                      \
    else k_background_scalar<OP><<<grid, 256, 0, st>>>(xz, B, A, oz);
        switch (op) {
        case ROIX_BG_SUB: ROIX_BG(ROIX_BG_SUB) break;
        case ROIX_BG_REV: ROIX_BG(ROIX_BG_REV) break;
        default: ROIX_BG(ROIX_BG_ADD) break;
        }
#undef ROIX_BG
    }
    return cudaGetLastError();
}
