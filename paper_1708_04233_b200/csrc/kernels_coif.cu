// kernels_coif.cu -- the coiflet mode (WASABI_FLAG_COIFLET, reading R-A21):
// "we used coiflets as the wavelets at level 3".  coif1 filter bank on the infinite
// grid with zero extension, interleaved layout (R-A6):
//   analysis  a[m] = sum_k h0[k] x[2m + k - 2],  d[m] = sum_k h1[k] x[2m + k - 2]
//   synthesis x[n] = sum_m h0[n - 2m + 2] a[m] + h1[n - 2m + 2] d[m]
// a level-l step works on the samples at multiples of s = 2^(l-1); a[m] -> sample 2m, d[m] -> 2m + 1.
//   step 1: psf_f64_kernel (PSF into an fp64 work table), fb_fwd_pass_kernel (per level: rows A->B,
//           columns B->A, fp64, taps summed in order k = 0..5 with _rn operations -- the same IEEE
//           sequence as the specification, so the fp32 rank keys match bit for bit), coef_keys_kernel.
//   step 3: fb_inv_line_kernel: per level (L..1) columns then rows, in place on the psi band that
//           carries a halo of kCoifHalo rows (one CTA per line; the line's level samples in shared
//           memory; fp32).  Samples outside the band / hologram are zero (R-A21 boundary).
// Off the fused hot path: the coiflet inverse is not block-local, so this mode runs superpose on the
// halo band, then the line passes, then quantise.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace wasabi {
namespace {

template <typename T>
__device__ __forceinline__ const T *at(const void *t, int64_t off) {
    return reinterpret_cast<const T *>(reinterpret_cast<const char *>(t) + off);
}

__device__ __forceinline__ int find_le(const int64_t *base, int n, int64_t b) {   // largest i: base[i] <= b
    int lo = 0, hi = n;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (base[mid] <= b) lo = mid; else hi = mid;
    }
    return lo;
}

constexpr int kTile = 64;

// PSF u_z = exp(i k r) circ(.) (R-A2) in fp64 into the work table (centre (H, H)).
__global__ void __launch_bounds__(256) psf_f64_kernel(const void *tables, double2 *__restrict__ work, double k,
                                                      double pitch, int n_tab) {
    const TableHeader &h = *reinterpret_cast<const TableHeader *>(tables);
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    const KDesc *kd = at<KDesc>(tables, h.kdesc_off);
    const int32_t *cbase = at<int32_t>(tables, h.ctabase_off);
    int lo = 0, hi = n_tab;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (cbase[mid] <= (int)blockIdx.x) lo = mid; else hi = mid;
    }
    const int d = lo;
    const DDesc D = dd[d];
    const int H = kd[d].H, side = D.side;
    const int local = (int)blockIdx.x - D.cta_base;
    const int X0 = (local % D.tiles) * kTile, Y0 = (local / D.tiles) * kTile;
    const double R2 = __dmul_rn(D.R, D.R), z2 = __dmul_rn(D.z, D.z);
    for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
        const int X = X0 + (i & (kTile - 1)), Y = Y0 + (i >> 6);
        if (X >= side || Y >= side) continue;
        const long long dx = X - H, dy = Y - H;
        double2 v = make_double2(0.0, 0.0);
        if ((dx == 0 && dy == 0) || ((double)(dx * dx + dy * dy) < R2)) {
            const double xp = __dmul_rn((double)dx, pitch), yp = __dmul_rn((double)dy, pitch);
            const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xp, xp), __dmul_rn(yp, yp)), z2));
            double s, c;
            sincos(__dmul_rn(k, r), &s, &c);
            v = make_double2(c, s);
        }
        work[D.coef_off + (int64_t)Y * side + X] = v;
    }
}

struct Filt {
    double h0[6], h1[6];
};

// One analysis pass of level l over all tables: thread = (table, line j, pair m).  rows = 1: lines
// are rows Y = s j, samples X = s n; rows = 0: lines are columns.  Reads src, writes dst (level grid).
__global__ void __launch_bounds__(256) fb_fwd_pass_kernel(const void *tables, const double2 *__restrict__ src,
                                                          double2 *__restrict__ dst, const int64_t *__restrict__ pre,
                                                          int n_tab, int l, int rows, Filt F) {
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= pre[n_tab]) return;
    const TableHeader &h = *reinterpret_cast<const TableHeader *>(tables);
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    const int t = find_le(pre, n_tab, g);
    const DDesc D = dd[t];
    const int side = D.side, s = 1 << (l - 1), N = side >> (l - 1);
    const int64_t local = g - pre[t];
    const int j = (int)(local / (N / 2)), m = (int)(local % (N / 2));
    const double2 *in = src + D.coef_off;
    double2 *out = dst + D.coef_off;
    // sample n of line j
    auto idx = [&](int n) -> int64_t {
        return rows ? (int64_t)(s * j) * side + (int64_t)s * n : (int64_t)(s * n) * side + (int64_t)s * j;
    };
    double ar = 0.0, ai = 0.0, dr = 0.0, di = 0.0;
#pragma unroll
    for (int k = 0; k < 6; k++) {
        const int i = 2 * m + k - 2;
        if (i < 0 || i >= N) continue;
        const double2 x = in[idx(i)];
        ar = __dadd_rn(ar, __dmul_rn(F.h0[k], x.x));
        ai = __dadd_rn(ai, __dmul_rn(F.h0[k], x.y));
        dr = __dadd_rn(dr, __dmul_rn(F.h1[k], x.x));
        di = __dadd_rn(di, __dmul_rn(F.h1[k], x.y));
    }
    out[idx(2 * m)] = make_double2(ar, ai);
    out[idx(2 * m + 1)] = make_double2(dr, di);
}

// fp32 value and rank key bits of fp32_RN(re^2 + im^2) (R-A13) from the fp64 coefficients.
__global__ void __launch_bounds__(256) coef_keys_kernel(const double2 *__restrict__ work, float2 *__restrict__ val,
                                                        uint32_t *__restrict__ key, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const double2 v = work[i];
    val[i] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
    key[i] = __float_as_uint(__double2float_rn(__dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y))));
}

// One synthesis pass of level l on the band psi (rows x n_h, in place): CTA = line.  rows = 0:
// line = column X = s j, samples along Y; rows = 1: line = row Y = s j.
__global__ void __launch_bounds__(256) fb_inv_line_kernel(float2 *__restrict__ psi, int64_t nrows, int64_t n_h, int l,
                                                          int rows, Filt F) {
    extern __shared__ float2 line[];
    const int s = 1 << (l - 1);
    const int j = blockIdx.x;
    const int64_t len = rows ? n_h : nrows;
    const int N = (int)(len / s);
    auto idx = [&](int n) -> int64_t {
        return rows ? (int64_t)(s * j) * n_h + (int64_t)s * n : (int64_t)s * n * n_h + (int64_t)s * j;
    };
    for (int n = threadIdx.x; n < N; n += blockDim.x) line[n] = psi[idx(n)];
    __syncthreads();
    float h0[6], h1[6];
#pragma unroll
    for (int k = 0; k < 6; k++) { h0[k] = (float)F.h0[k]; h1[k] = (float)F.h1[k]; }
    for (int n = threadIdx.x; n < N; n += blockDim.x) {
        float xr = 0.f, xi = 0.f;
        const int m_hi = (n + 2) >> 1;
#pragma unroll
        for (int q = 0; q < 3; q++) {
            const int m = m_hi - q, k = n - 2 * m + 2;
            if (m < 0 || 2 * m + 1 >= N || k < 0 || k > 5) continue;
            const float2 a = line[2 * m], d = line[2 * m + 1];
            xr = fmaf(h0[k], a.x, fmaf(h1[k], d.x, xr));
            xi = fmaf(h0[k], a.y, fmaf(h1[k], d.y, xi));
        }
        psi[idx(n)] = make_float2(xr, xi);
    }
}

}  // namespace

// coif1 (R-A21): h0 = sqrt(2)/32 [1-s, 5+s, 14+2s, 14-2s, 1-s, -3+s], s = sqrt(7); h1[k] = (-1)^k h0[5-k].
static Filt coif1() {
    Filt F;
    const double s7 = sqrt(7.0), c = sqrt(2.0) / 32.0;
    const double v[6] = {1.0 - s7, 5.0 + s7, 14.0 + 2.0 * s7, 14.0 - 2.0 * s7, 1.0 - s7, -3.0 + s7};
    for (int k = 0; k < 6; k++) F.h0[k] = v[k] * c;
    for (int k = 0; k < 6; k++) F.h1[k] = ((k & 1) ? -1.0 : 1.0) * F.h0[5 - k];
    return F;
}

cudaError_t launch_coif_tables(const TableHeader &h, const void *d_tables, double2 *work, double2 *tmp,
                               const int64_t *d_pre, const int64_t *h_pre_last, float2 *val, uint32_t *key,
                               int64_t n_coef, double k, double pitch, int L, cudaStream_t s) {
    const Filt F = coif1();
    const int nt = h.n_depth;
    count_launches(1);
    psf_f64_kernel<<<(unsigned)h.total_ctas, 256, 0, s>>>(d_tables, work, k, pitch, nt);
    for (int l = 1; l <= L; l++) {
        const int64_t n = h_pre_last[l - 1];
        const unsigned blocks = (unsigned)((n + 255) / 256);
        if (!blocks) continue;
        const int64_t *pre = d_pre + (int64_t)(l - 1) * (nt + 1);
        count_launches(2);
        fb_fwd_pass_kernel<<<blocks, 256, 0, s>>>(d_tables, work, tmp, pre, nt, l, 1, F);
        fb_fwd_pass_kernel<<<blocks, 256, 0, s>>>(d_tables, tmp, work, pre, nt, l, 0, F);
    }
    if (n_coef > 0) {
        count_launches(1);
        coef_keys_kernel<<<(unsigned)((n_coef + 255) / 256), 256, 0, s>>>(work, val, key, n_coef);
    }
    return cudaGetLastError();
}

cudaError_t launch_coif_inverse(float2 *psi, int64_t nrows, int64_t n_h, int L, cudaStream_t s) {
    const Filt F = coif1();
    const int max_len = (int)(nrows > n_h ? nrows : n_h);
    const int smem = max_len * (int)sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(fb_inv_line_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    for (int l = L; l >= 1; l--) {
        const int sgrid = 1 << (l - 1);
        const unsigned ncols = (unsigned)(n_h / sgrid), nrow = (unsigned)(nrows / sgrid);
        count_launches(2);
        fb_inv_line_kernel<<<ncols, 256, (int)(nrows / sgrid) * (int)sizeof(float2), s>>>(psi, nrows, n_h, l, 0, F);
        fb_inv_line_kernel<<<nrow, 256, (int)(n_h / sgrid) * (int)sizeof(float2), s>>>(psi, nrows, n_h, l, 1, F);
    }
    return cudaGetLastError();
}

}  // namespace wasabi
