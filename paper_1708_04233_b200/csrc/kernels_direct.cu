// kernels_direct.cu -- the conventional method on the GPU: quantised direct
// sum of Eq.(1) by PSF stamping (the N-LUT-like form the paper compares against,
// PAPER.md:129, :164-167):  u(X, Y) = sum_j a_j f_{iz_j}(X - ix_j, Y - iy_j)  with the same
// quantisation (R-A3, R-A9) and the same PSF tables f_d = exp(ikr) circ(.) (R-A2) as
// WASABI, but without the wavelet shrinkage.  Used as the PSNR reference for the C5 sweep (R-A18)
// and as the same-box conventional baseline.
//   K7a psf_dense_kernel: dense fp32 PSF tables (fp64 phase), one per depth.
//   K7b stamp_kernel: one CTA per 64x64 tile, each thread owns 16 pixels in registers and gathers
//       f from the dense table for every point of the tile's bin (bin order = accumulation order).
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "device_common.cuh"

namespace wasabi {
namespace {

__global__ void __launch_bounds__(256) psf_dense_kernel(const DenseDesc *__restrict__ dd, int n_depth,
                                                        float2 *__restrict__ out, double k, double pitch,
                                                        int64_t total_ctas) {
    // CTA -> (depth, 64x64 tile) by linear search over the (small) depth list
    int64_t b = blockIdx.x;
    int d = 0;
    while (d + 1 < n_depth && dd[d + 1].cta_base <= b) d++;
    const DenseDesc D = dd[d];
    const int local = (int)(b - D.cta_base);
    const int tiles = (D.side + 63) / 64;
    const int X0 = (local % tiles) * 64, Y0 = (local / tiles) * 64;
    const int H = D.side / 2;
    const double R2 = __dmul_rn(D.R, D.R), z2 = __dmul_rn(D.z, D.z);
    for (int i = threadIdx.x; i < 64 * 64; i += 256) {
        const int X = X0 + (i & 63), Y = Y0 + (i >> 6);
        if (X >= D.side || Y >= D.side) continue;
        const long long dx = X - H, dy = Y - H;
        float2 v = make_float2(0.f, 0.f);
        if ((dx == 0 && dy == 0) || (double)(dx * dx + dy * dy) < R2) {
            const double xp = __dmul_rn((double)dx, pitch), yp = __dmul_rn((double)dy, pitch);
            const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xp, xp), __dmul_rn(yp, yp)), z2));
            double s, c;
            sincos(__dmul_rn(k, r), &s, &c);
            v = make_float2((float)c, (float)s);
        }
        out[D.off + (int64_t)Y * D.side + X] = v;
    }
}

constexpr int kT = 64;

__global__ void __launch_bounds__(256) stamp_kernel(const void *__restrict__ d_bins, const DenseDesc *__restrict__ dd,
                                                    const float2 *__restrict__ dense, int tiles_x, int64_t row0,
                                                    int64_t n_h, int T, float2 *__restrict__ u) {
    __shared__ int4 pts[256];
    const char *bb = reinterpret_cast<const char *>(d_bins);
    const BinHeader *bh = reinterpret_cast<const BinHeader *>(bb);
    const int4 *__restrict__ pconv = reinterpret_cast<const int4 *>(bb + bh->pts_off);
    const unsigned long long *__restrict__ bptr = reinterpret_cast<const unsigned long long *>(bb + bh->ptr_off);
    const uint32_t *__restrict__ bidx = reinterpret_cast<const uint32_t *>(bb + bh->idx_off);
    const int64_t t = blockIdx.x;
    const int bin_x0 = (int)(t % tiles_x) * T;
    const int bin_y0 = (int)(row0 + (t / tiles_x) * (int64_t)T);
    const int x = threadIdx.x & 63, yb = threadIdx.x >> 6;   // pixels (x, yb + 4k), k = 0..15
    const unsigned long long b0 = bptr[t], b1 = bptr[t + 1];
    for (int sub = 0; sub < (T / kT) * (T / kT); sub++) {    // 64x64 sub-tiles of the bin tile
    const int tile_x0 = bin_x0 + (sub % (T / kT)) * kT, tile_y0 = bin_y0 + (sub / (T / kT)) * kT;
    float ar[16], ai[16];
#pragma unroll
    for (int k = 0; k < 16; k++) { ar[k] = 0.f; ai[k] = 0.f; }
    for (unsigned long long pb = b0; pb < b1; pb += 256) {
        const int np = (int)min(256ull, b1 - pb);
        __syncthreads();
        if ((int)threadIdx.x < np) pts[threadIdx.x] = pconv[bidx[pb + threadIdx.x]];
        __syncthreads();
        for (int j = 0; j < np; j++) {
            const int4 q = pts[j];
            const DenseDesc D = dd[q.z];
            const int H = D.side / 2;
            const float a = __int_as_float(q.w);
            const int cx = tile_x0 + x - q.x + H;            // table column of my pixel
            if ((unsigned)cx >= (unsigned)D.side) continue;
            const float2 *row = dense + D.off + cx;
#pragma unroll
            for (int k = 0; k < 16; k++) {
                const int cy = tile_y0 + yb + 4 * k - q.y + H;
                if ((unsigned)cy < (unsigned)D.side) {
                    const float2 f = __ldg(row + (int64_t)cy * D.side);
                    ar[k] = fmaf(a, f.x, ar[k]);
                    ai[k] = fmaf(a, f.y, ai[k]);
                }
            }
        }
    }
#pragma unroll
    for (int k = 0; k < 16; k++)
        u[(int64_t)(tile_y0 + yb + 4 * k - row0) * n_h + tile_x0 + x] = make_float2(ar[k], ai[k]);
    }
}

// K7c exact_kernel: the exact Eq.(1) -- continuous (x_j, y_j, z_j), no depth or
// position quantisation -- on the diffraction-limited window rho < |z_j| tan(theta) (+ the rho = 0
// pixel), the D1 reference of the C5 PSNR (R-A18).  Bins by the PSF disc (wasabi_bin_points_psf; their
// reach covers the continuous point: R of the level's far edge + 1 px).  One CTA per 64x64 tile, each
// thread owns 16 pixels in registers; per (pixel, point) the window test and the distance are fp64
// (the oracle's sequence), the phase is the fp64 quarter-cycle count 4 r / lambda and (cos, sin) its
// fp32 minimax split (< 1e-7), accumulated in fp32 in bin (point) order.
struct ExArgs {
    double pitch, tn, k4;              // p, tan(theta), 4/lambda
    int64_t half, row0, n_h;
    int tiles_x, T;
};

__global__ void __launch_bounds__(256) exact_kernel(const void *__restrict__ d_bins, const float4 *__restrict__ pts,
                                                    ExArgs A, float2 *__restrict__ u) {
    __shared__ double4 sp[128];      // x_j / p, y_j / p, z_j^2, R_j^2 (pixel units)
    __shared__ double2 sm[128];      // x_j, y_j (metres)
    __shared__ float sa[128];
    const char *bb = reinterpret_cast<const char *>(d_bins);
    const BinHeader *bh = reinterpret_cast<const BinHeader *>(bb);
    const unsigned long long *__restrict__ bptr = reinterpret_cast<const unsigned long long *>(bb + bh->ptr_off);
    const uint32_t *__restrict__ bidx = reinterpret_cast<const uint32_t *>(bb + bh->idx_off);
    const int64_t t = blockIdx.x;
    const int bin_x0 = (int)(t % A.tiles_x) * A.T;
    const int bin_y0 = (int)(A.row0 + (t / A.tiles_x) * (int64_t)A.T);
    const int x = threadIdx.x & 63, yb = threadIdx.x >> 6;
    const unsigned long long b0 = bptr[t], b1 = bptr[t + 1];
    for (int sub = 0; sub < (A.T / kT) * (A.T / kT); sub++) {
        const int tile_x0 = bin_x0 + (sub % (A.T / kT)) * kT, tile_y0 = bin_y0 + (sub / (A.T / kT)) * kT;
        const int64_t X = tile_x0 + x;
        const double ex0 = (double)(X - A.half), xh = __dmul_rn(ex0, A.pitch);
        float ar[16], ai[16];
#pragma unroll
        for (int k = 0; k < 16; k++) { ar[k] = 0.f; ai[k] = 0.f; }
        for (unsigned long long pb = b0; pb < b1; pb += 128) {
            const int np = (int)min(128ull, b1 - pb);
            __syncthreads();
            if ((int)threadIdx.x < np) {
                const float4 q = pts[bidx[pb + threadIdx.x]];
                // the oracle's sequence (orc_direct_d1): x / p, y / p and R = |z| tan(theta) / p by division
                const double R = __ddiv_rn(__dmul_rn(fabs((double)q.z), A.tn), A.pitch);
                sp[threadIdx.x] = make_double4(__ddiv_rn((double)q.x, A.pitch), __ddiv_rn((double)q.y, A.pitch),
                                               __dmul_rn((double)q.z, (double)q.z), __dmul_rn(R, R));
                sm[threadIdx.x] = make_double2((double)q.x, (double)q.y);
                sa[threadIdx.x] = q.w;
            }
            __syncthreads();
            for (int j = 0; j < np; j++) {
                const double4 P = sp[j];
                const double2 M = sm[j];
                const float a = sa[j];
                const double ex = __dsub_rn(ex0, P.x), ex2 = __dmul_rn(ex, ex);
                const double ddx = __dsub_rn(xh, M.x), ddx2 = __dmul_rn(ddx, ddx);
#pragma unroll
                for (int k = 0; k < 16; k++) {
                    const double ey0 = (double)(tile_y0 + yb + 4 * k - A.half);
                    const double ey = __dsub_rn(ey0, P.y);
                    const double rho2 = __dadd_rn(ex2, __dmul_rn(ey, ey));
                    if (rho2 < P.w || rho2 == 0.0) {
                        const double ddy = __dsub_rn(__dmul_rn(ey0, A.pitch), M.y);
                        const double r = sqrt_nonneg(__dadd_rn(__dadd_rn(ddx2, __dmul_rn(ddy, ddy)), P.z));
                        const float2 cs = cis_quarter(__dmul_rn(r, A.k4));
                        ar[k] = fmaf(a, cs.x, ar[k]);
                        ai[k] = fmaf(a, cs.y, ai[k]);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 16; k++)
            u[(int64_t)(tile_y0 + yb + 4 * k - A.row0) * A.n_h + tile_x0 + x] = make_float2(ar[k], ai[k]);
    }
}

}  // namespace

cudaError_t launch_exact(const void *d_bins, const float4 *pts, int tiles_x, int tiles_y, int64_t row0, int64_t n_h,
                         int T, double pitch, double tan_theta, double wavelength, float2 *u, cudaStream_t s) {
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    if (n_tiles <= 0) return cudaSuccess;
    ExArgs A;
    A.pitch = pitch; A.tn = tan_theta; A.k4 = 4.0 / wavelength;
    A.half = n_h / 2; A.row0 = row0; A.n_h = n_h; A.tiles_x = tiles_x; A.T = T;
    count_launches(1);
    exact_kernel<<<(unsigned)n_tiles, 256, 0, s>>>(d_bins, pts, A, u);
    return cudaGetLastError();
}

cudaError_t launch_psf_dense(const DenseDesc *d_desc, int n_depth, float2 *out, double k, double pitch,
                             int64_t total_ctas, cudaStream_t s) {
    if (total_ctas <= 0) return cudaSuccess;
    count_launches(1);
    psf_dense_kernel<<<(unsigned)total_ctas, 256, 0, s>>>(d_desc, n_depth, out, k, pitch, total_ctas);
    return cudaGetLastError();
}

cudaError_t launch_stamp(const void *d_bins, const DenseDesc *d_desc, const float2 *dense, int tiles_x, int tiles_y,
                         int64_t row0, int64_t n_h, int T, float2 *u, cudaStream_t s) {
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    if (n_tiles <= 0) return cudaSuccess;
    count_launches(1);
    stamp_kernel<<<(unsigned)n_tiles, 256, 0, s>>>(d_bins, d_desc, dense, tiles_x, row0, n_h, T, u);
    return cudaGetLastError();
}

}  // namespace wasabi
