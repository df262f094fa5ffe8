// kernels_inverse.cu -- steps 3 and 4 of WASABI.
//  K5 inverse_kernel: L-level inverse Haar of one 64 x 64 tile in shared
//     memory (tile and band edges are multiples of 2^L, so every block is self-contained: no halo),
//     butterflies a=((LL+HL)+(LH+HH))/2, b=((LL-HL)+(LH-HH))/2, c=((LL+HL)-(LH+HH))/2,
//     d=((LL-HL)-(LH-HH))/2 (R-A6); optionally fused with the print quantisation.
//  K6 quantize_kernel: standalone step 4 on an existing u.
// Step 4 (R-A14, R-A15): I = Re(u conj(R)), R = exp(i k r),
//     r = sqrt((x-x_r)^2 + (y-y_r)^2 + z_r^2); the phase is reduced in fp64 (r/lambda up to ~1e6
//     cycles; fp32 would be off by > 0.2 rad) and only the reduced fraction goes to fp32 sincospi.
// HBM-bound: 16 B/px (read psi, write u), +0.125 B/px bits.
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "internal.h"
#include "device_common.cuh"

namespace wasabi {
namespace {

constexpr int kT = 64;
constexpr int kS = kT + 2;  // float2 row stride (keeps float4 alignment of rows)

__global__ void __launch_bounds__(256) inverse_kernel(const float2 *psi, float2 *u, int64_t n_h, int64_t row0, int L,
                                                      QArgs q, uint8_t *__restrict__ bits, int write_u, int do_bits) {
    __shared__ __align__(16) float2 s[kT * kS];
    const int64_t X0 = (int64_t)blockIdx.x * kT, Yl0 = (int64_t)blockIdx.y * kT;  // band-local rows
    const float4 *src = reinterpret_cast<const float4 *>(psi);
    // load 64 rows x 64 complex (32 float4 per row), coalesced
#pragma unroll
    for (int i = 0; i < 8; i++) {
        const int f = threadIdx.x + 256 * i;
        const int row = f >> 5, c4 = f & 31;
        const float4 v = src[((Yl0 + row) * n_h + X0) / 2 + c4];
        *reinterpret_cast<float4 *>(&s[row * kS + 2 * c4]) = v;
    }
    __syncthreads();
    inverse_haar_tile_blk4(s, kT, kS, L, threadIdx.x, 256);
    if (write_u) {
        float4 *dst = reinterpret_cast<float4 *>(u);
#pragma unroll
        for (int i = 0; i < 8; i++) {
            const int f = threadIdx.x + 256 * i;
            const int row = f >> 5, c4 = f & 31;
            dst[((Yl0 + row) * n_h + X0) / 2 + c4] = *reinterpret_cast<const float4 *>(&s[row * kS + 2 * c4]);
        }
    }
    if (do_bits) {
        // 64 rows x 8 bytes per tile; thread -> 2 bytes
        for (int bi = threadIdx.x; bi < kT * 8; bi += 256) {
            const int row = bi >> 3, xb = bi & 7;
            const int64_t Y = row0 + Yl0 + row;
            float2 v[8];
#pragma unroll
            for (int i = 0; i < 8; i++) v[i] = s[row * kS + xb * 8 + i];
            const unsigned byte = print_byte(v, X0 + xb * 8, ref_row(Y, q), q);
            bits[(Yl0 + row) * (n_h / 8) + X0 / 8 + xb] = (uint8_t)byte;
        }
    }
}

__global__ void __launch_bounds__(256) quantize_kernel(const float2 *__restrict__ u, int64_t rows, int64_t n_h,
                                                       int64_t row0, QArgs q, uint8_t *__restrict__ bits) {
    const int64_t nbytes = rows * (n_h / 8);
    for (int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; b < nbytes; b += (int64_t)gridDim.x * blockDim.x) {
        const int64_t yl = b / (n_h / 8), xb = b % (n_h / 8);
        const float4 *p = reinterpret_cast<const float4 *>(u + yl * n_h + xb * 8);
        float2 v[8];
#pragma unroll
        for (int i = 0; i < 4; i++) {
            const float4 f = p[i];
            v[2 * i] = make_float2(f.x, f.y);
            v[2 * i + 1] = make_float2(f.z, f.w);
        }
        bits[b] = (uint8_t)print_byte(v, xb * 8, ref_row(row0 + yl, q), q);
    }
}

}  // namespace

cudaError_t launch_inverse(const float2 *psi, float2 *u, int64_t rows, int64_t n_h, int64_t row0, int levels,
                           const double *print4, double pitch, uint8_t *bits, cudaStream_t s) {
    const QArgs q = make_qargs(print4, pitch, n_h);
    dim3 grid((unsigned)(n_h / kT), (unsigned)(rows / kT));
    if (grid.x == 0 || grid.y == 0) return cudaSuccess;
    count_launches(1);
    inverse_kernel<<<grid, 256, 0, s>>>(psi, u, n_h, row0, levels, q, bits, u != nullptr, bits != nullptr);
    return cudaGetLastError();
}

cudaError_t launch_quantize(const float2 *u, int64_t rows, int64_t n_h, int64_t row0, const double *print4,
                            double pitch, uint8_t *bits, cudaStream_t s) {
    const QArgs q = make_qargs(print4, pitch, n_h);
    const int64_t nbytes = rows * (n_h / 8);
    if (nbytes == 0) return cudaSuccess;
    const int64_t blocks = std::min<int64_t>((nbytes + 255) / 256, 148 * 64);
    count_launches(1);
    quantize_kernel<<<(unsigned)blocks, 256, 0, s>>>(u, rows, n_h, row0, q, bits);
    return cudaGetLastError();
}

}  // namespace wasabi
