// kernels_coif.cu -- the coiflet mode (WASABI_FLAG_COIFLET, reading R-A21):
// "we used coiflets as the wavelets at level 3".  coif1 filter bank on the infinite
// grid with zero extension, interleaved layout (R-A6):
//   analysis  a[m] = sum_k h0[k] x[2m + k - 2],  d[m] = sum_k h1[k] x[2m + k - 2]
//   synthesis x[n] = sum_m h0[n - 2m + 2] a[m] + h1[n - 2m + 2] d[m]
// a level-l step works on the samples at multiples of s = 2^(l-1); a[m] -> sample 2m, d[m] -> 2m + 1.
//   step 1: psf_f64_kernel (PSF into an fp64 work table), fb_fwd_pass_kernel (per level: rows A->B,
//           columns B->A, fp64, taps summed in order k = 0..5 with _rn operations -- the same IEEE
//           sequence as the specification, so the fp32 rank keys match bit for bit), coef_keys_kernel.
//   step 3 (+4): coif_synth_tile_kernel<L>: per 64 x 64 output tile, psi plus a halo in shared memory,
//           the L levels of column and row passes in place, then the print bits and u (psi only read);
//           or fb_inv_cols_kernel / fb_inv_rows_kernel: per level (L..1) columns then rows, in place on
//           the psi band that carries a halo of one tile row (rolling window of pairs along the lines
//           in shared memory; fp32), then quantize_kernel.  Samples outside the band / hologram are
//           zero (R-A21 boundary); both give bit-identical u and bits.
// The coiflet inverse is not block-local (its halo crosses tiles), so this mode superposes psi on the
// halo band first (no superpose -> inverse fusion as in the Haar path).
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "device_common.cuh"

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
    // rows: adjacent threads take adjacent pairs of a row; columns: adjacent columns at the same pair
    // (coalesced along the row in both cases)
    const int j = rows ? (int)(local / (N / 2)) : (int)(local % N);
    const int m = rows ? (int)(local % (N / 2)) : (int)(local / N);
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

// One synthesis pass of level l on the band psi (nrows x n_h, in place), as a rolling window along
// the lines.  Output samples 2p and 2p + 1 need pairs p - 1, p, p + 1 (pair m = samples 2m, 2m + 1;
// k = n - 2m + 2 in [0, 5]); a CTA owns its lines, loads blocks of kBP pairs, keeps the last two
// pairs of the previous block, and writes outputs only over pairs it has already read: in place
// without races.  Columns: 32 adjacent lines per CTA (coalesced across lines); rows: one line per
// CTA with the threads along it.  Samples beyond the band / hologram are zero (R-A21).
constexpr int kBP = 32;

__device__ __forceinline__ float2 synth(const float2 *a, const float2 *d, int q, int stride, const float *h0,
                                        const float *h1, int odd) {
    // pairs q - 1, q, q + 1 of the window (p - 1, p, p + 1), k = 4, 2, 0 (even) / 5, 3, 1 (odd)
    float2 x = make_float2(0.f, 0.f);
#pragma unroll
    for (int t = 0; t < 3; t++) {
        const int k = 4 - 2 * t + odd;
        const float2 A = a[(q + t) * stride], D = d[(q + t) * stride];
        x.x = fmaf(h0[k], A.x, fmaf(h1[k], D.x, x.x));
        x.y = fmaf(h0[k], A.y, fmaf(h1[k], D.y, x.y));
    }
    return x;
}

__global__ void __launch_bounds__(256) fb_inv_cols_kernel(float2 *__restrict__ psi, int64_t nrows, int64_t n_h, int l,
                                                          Filt F) {
    __shared__ float2 sa[kBP + 2][32], sd[kBP + 2][32];
    const int s = 1 << (l - 1), tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
    const int ncol = (int)(n_h / s), np = (int)(nrows / s) / 2;
    const int j = blockIdx.x * 32 + tx;
    const bool colok = j < ncol;
    float h0[6], h1[6];
#pragma unroll
    for (int k = 0; k < 6; k++) { h0[k] = (float)F.h0[k]; h1[k] = (float)F.h1[k]; }
    auto at = [&](int n) -> int64_t { return (int64_t)s * n * n_h + (int64_t)s * j; };
    if (ty < 2) { sa[ty][tx] = make_float2(0.f, 0.f); sd[ty][tx] = make_float2(0.f, 0.f); }   // pairs -2, -1
    for (int p0 = 0; p0 <= np; p0 += kBP) {
        for (int q = ty; q < kBP; q += 8) {           // pairs p0 .. p0 + kBP - 1 -> window rows 2..
            const int p = p0 + q;
            float2 A = make_float2(0.f, 0.f), D = A;
            if (colok && p < np) { A = psi[at(2 * p)]; D = psi[at(2 * p + 1)]; }
            sa[q + 2][tx] = A; sd[q + 2][tx] = D;
        }
        __syncthreads();
        // outputs for pairs p = p0 - 1 + q (window rows q .. q + 2 hold p - 1 .. p + 1)
        for (int q = ty; q < kBP; q += 8) {
            const int p = p0 - 1 + q;
            if (!colok || p < 0 || p >= np) continue;
            psi[at(2 * p)] = synth(&sa[0][tx], &sd[0][tx], q, 32, h0, h1, 0);
            psi[at(2 * p + 1)] = synth(&sa[0][tx], &sd[0][tx], q, 32, h0, h1, 1);
        }
        __syncthreads();
        if (ty < 2) { sa[ty][tx] = sa[kBP + ty][tx]; sd[ty][tx] = sd[kBP + ty][tx]; }
        __syncthreads();
    }
}

constexpr int kRP = 256;
__global__ void __launch_bounds__(256) fb_inv_rows_kernel(float2 *__restrict__ psi, int64_t nrows, int64_t n_h, int l,
                                                          Filt F) {
    __shared__ float2 sa[kRP + 2], sd[kRP + 2];
    const int s = 1 << (l - 1), t = threadIdx.x;
    const int np = (int)(n_h / s) / 2;
    const int64_t row = (int64_t)s * blockIdx.x * n_h;
    float h0[6], h1[6];
#pragma unroll
    for (int k = 0; k < 6; k++) { h0[k] = (float)F.h0[k]; h1[k] = (float)F.h1[k]; }
    if (t < 2) { sa[t] = make_float2(0.f, 0.f); sd[t] = make_float2(0.f, 0.f); }
    for (int p0 = 0; p0 <= np; p0 += kRP) {
        const int p = p0 + t;
        float2 A = make_float2(0.f, 0.f), D = A;
        if (p < np) { A = psi[row + (int64_t)s * (2 * p)]; D = psi[row + (int64_t)s * (2 * p + 1)]; }
        sa[t + 2] = A; sd[t + 2] = D;
        __syncthreads();
        const int po = p0 - 1 + t;
        if (po >= 0 && po < np) {
            psi[row + (int64_t)s * (2 * po)] = synth(sa, sd, t, 1, h0, h1, 0);
            psi[row + (int64_t)s * (2 * po + 1)] = synth(sa, sd, t, 1, h0, h1, 1);
        }
        __syncthreads();
        if (t < 2) { sa[t] = sa[kRP + t]; sd[t] = sd[kRP + t]; }
        __syncthreads();
    }
}

// ---- fused coif1 synthesis + quantise, one 64 x 64 output tile per CTA (psi read once) ----
// The tile's psi is loaded with a halo of a_L pixels per side into shared memory (row pitch R + 1
// cells, odd: conflict-free along rows and columns), zero outside the psi band and the hologram (the
// R-A21 boundary, as the line passes).  Level l = L..1 (grid s = 2^(l-1)) runs its column pass then
// its row pass in place over the square [-a_l, 64 + a_l), a_L = 3 (2^L - 1) rounded up to 2^L and
// a_(l-1) = a_l - 3 s rounded down to 2^(l-1): an output sample depends on the samples within
// [-2 s, +3 s], so after level 1 the square [-3, 67) is exact.  Lines are split into segments of
// pairs, one per thread; a thread reads its neighbours' boundary pairs before a barrier and then rolls
// along its segment (old values of pairs p - 1, p, p + 1 in registers), so the in-place passes have no
// races.  Every output sample is computed with synth()'s operation sequence from the same inputs as
// fb_inv_cols/rows_kernel: u and the bits are bit-identical to the line passes + quantize_kernel.
constexpr int kCT = 64;        // output tile side
#ifndef WASABI_COIF_GROUP
#define WASABI_COIF_GROUP 32   // tile order: 10.66 -> 10.36 ms per 16384-row C4 band (8: 10.42, 16: 10.38, 64: 10.35)
#endif
#ifndef WASABI_COIF_THREADS
#define WASABI_COIF_THREADS 384   // 12 warps x 2 CTAs per SM: measured best of 256..512 (2.79 -> 2.69 ms per 4096-row C4 band)
#endif
constexpr int kCThreads = WASABI_COIF_THREADS;

// a_l of level l for an L-level synthesis: a_L = 3 (2^L - 1) rounded up to 2^L (the halo), a_(l-1) =
// a_l - 3 s_l rounded down to a multiple of 2^(l-1) (the next level's pair size)
__host__ __device__ constexpr int coif_a(int L, int l) {
    int a = (3 * ((1 << L) - 1) + (1 << L) - 1) / (1 << L) * (1 << L);
    for (int k = L; k > l; k--) a = (a - 3 * (1 << (k - 1))) / (1 << (k - 1)) * (1 << (k - 1));
    return a;
}
__host__ __device__ constexpr int coif_seg(int nl, int np) {   // segments per line: lines x seg <= threads
    int seg = 1;
    while (nl * (seg + 1) <= kCThreads && seg + 1 <= np) seg++;
    return seg;
}

// One synthesis pass of level l (grid S = 2^(l-1)) over the square [-A, 64 + A): PASS 0 = columns
// (lines are columns, samples along y), 1 = rows.  reg: the region, origin (-HP, -HP), pitch P cells.
// Thread -> (line j = tid % nl, segment g = tid / nl): a warp's lanes work on adjacent lines at the
// same sample (conflict-free shared accesses at S = 1).  Samples outside [vlo, vhi) along the line,
// and lines outside [llo, lhi), are never written (R-A21 zeros).
template <int PASS, int S, int A, int HP, int P>
__device__ __forceinline__ void coif_pass(float2 *reg, const float *h0, const float *h1, int vlo, int vhi, int llo,
                                          int lhi) {
    constexpr int nl = (kCT + 2 * A) / S, np = nl / 2;
    constexpr int seg = coif_seg(nl, np), per = (np + seg - 1) / seg;
    const int tid = threadIdx.x;
    const bool active = tid < nl * seg;
    const int j = tid % nl, g = tid / nl;
    const int p_beg = g * per, p_end = active ? min(np, p_beg + per) : 0;
    const int across = -A + S * j;
    // sample n of the line: base[n * st]
    constexpr int st = PASS == 0 ? S * P : S;
    float2 *base = PASS == 0 ? reg + (HP - A) * P + (across + HP) : reg + (across + HP) * P + (HP - A);
    // writable samples n in [nlo, nhi): along-line coordinate -A + S n in [vlo, vhi), line inside [llo, lhi)
    int nlo = 0, nhi = 0;
    if (across >= llo && across < lhi) {
        nlo = max(0, (vlo + A + S - 1) / S);
        nhi = min(nl, (vhi + A + S - 1) / S);
    }
    const float2 z = make_float2(0.f, 0.f);
    float2 lA = z, lD = z, rA = z, rD = z;   // old pairs p_beg - 1 and p_end (zero beyond the square)
    if (p_beg < p_end) {
        if (p_beg > 0) { lA = base[(2 * p_beg - 2) * st]; lD = base[(2 * p_beg - 1) * st]; }
        if (p_end < np) { rA = base[(2 * p_end) * st]; rD = base[(2 * p_end + 1) * st]; }
    }
    __syncthreads();
    if (p_beg < p_end) {
        float2 *q = base + 2 * p_beg * st;                    // pair p
        float2 A0 = lA, D0 = lD;                              // pair p - 1 (old)
        float2 A1 = q[0], D1 = q[st];                         // pair p (old)
        const bool all = nlo <= 2 * p_beg && 2 * p_end <= nhi;
        for (int p = p_beg; p < p_end; p++, q += 2 * st) {
            float2 A2 = rA, D2 = rD;                          // pair p + 1 (old)
            if (p + 1 < p_end) { A2 = q[2 * st]; D2 = q[3 * st]; }
            float2 o[2];
#pragma unroll
            for (int odd = 0; odd < 2; odd++) {               // synth(): k = 4 - 2 t + odd, t = 0..2
                float2 x = z;
                const float2 As[3] = {A0, A1, A2}, Ds[3] = {D0, D1, D2};
#pragma unroll
                for (int t = 0; t < 3; t++) {
                    const int k = 4 - 2 * t + odd;
                    x.x = fmaf(h0[k], As[t].x, fmaf(h1[k], Ds[t].x, x.x));
                    x.y = fmaf(h0[k], As[t].y, fmaf(h1[k], Ds[t].y, x.y));
                }
                o[odd] = x;
            }
            if (all) {
                q[0] = o[0];
                q[st] = o[1];
            } else {
                if (2 * p >= nlo && 2 * p < nhi) q[0] = o[0];
                if (2 * p + 1 >= nlo && 2 * p + 1 < nhi) q[st] = o[1];
            }
            A0 = A1; D0 = D1; A1 = A2; D1 = D2;
        }
    }
    __syncthreads();
}

template <int L, int l>
__device__ __forceinline__ void coif_levels(float2 *reg, const float *h0, const float *h1, int ylo, int yhi, int xlo,
                                            int xhi) {
    constexpr int HP = coif_a(L, L), P = kCT + 2 * HP + 1, A = coif_a(L, l), S = 1 << (l - 1);
    coif_pass<0, S, A, HP, P>(reg, h0, h1, ylo, yhi, xlo, xhi);
    coif_pass<1, S, A, HP, P>(reg, h0, h1, xlo, xhi, ylo, yhi);
    if constexpr (l > 1) coif_levels<L, l - 1>(reg, h0, h1, ylo, yhi, xlo, xhi);
}

template <int L>
__global__ void __launch_bounds__(kCThreads) coif_synth_tile_kernel(const float2 *__restrict__ psi, int64_t e0,
                                                                    int64_t e1, int64_t row0, int64_t n_h, Filt F,
                                                                    QArgs qa, float2 *__restrict__ u,
                                                                    uint8_t *__restrict__ bits) {
    extern __shared__ float2 reg[];
    constexpr int hp = coif_a(L, L), R = kCT + 2 * hp, P = R + 1;
    static_assert(coif_a(L, 1) >= 3, "coif1 halo: the square of level 1 must cover [-3, 67)");
    const int tid = threadIdx.x, lane = tid & 31;
    const int tiles_x = (int)(n_h / kCT);
    int64_t tx, ty;
    if (WASABI_COIF_GROUP > 0) {   // groups of G tile rows, column-major inside a group: the vertical halo
        const int64_t tiles_y = (gridDim.x + tiles_x - 1) / tiles_x;   // rows of the band (grid = tiles_x x tiles_y)
        const int64_t per = (int64_t)WASABI_COIF_GROUP * tiles_x;      // neighbours' psi is re-read from L2
        const int64_t g = blockIdx.x / per, rem = blockIdx.x - g * per;
        const int gh = (int)min((int64_t)WASABI_COIF_GROUP, tiles_y - g * WASABI_COIF_GROUP);
        ty = g * WASABI_COIF_GROUP + rem % gh;
        tx = rem / gh;
    } else {
        tx = blockIdx.x % tiles_x;
        ty = blockIdx.x / tiles_x;
    }
    const int64_t tile_x0 = tx * kCT;
    const int64_t tile_y0 = row0 + ty * kCT;
    float h0[6], h1[6];
#pragma unroll
    for (int k = 0; k < 6; k++) { h0[k] = (float)F.h0[k]; h1[k] = (float)F.h1[k]; }
    // R-A21 boundary: samples outside the psi band rows [e0, e1) and the hologram columns are zero at
    // every level (as in the line passes, whose lines end there): loaded as zero, never written
    const int ylo = (int)max((int64_t)-hp, e0 - tile_y0), yhi = (int)min((int64_t)(kCT + hp), e1 - tile_y0);
    const int xlo = (int)max((int64_t)-hp, -tile_x0), xhi = (int)min((int64_t)(kCT + hp), n_h - tile_x0);
    // load (asynchronous 8-byte copies, zero-filled outside): a warp per region row
    const uint32_t rsa = (uint32_t)__cvta_generic_to_shared(reg);
    if (ylo == -hp && yhi == kCT + hp && xlo == -hp && xhi == kCT + hp) {   // interior tile: no checks
        const float2 *src = psi + (tile_y0 - hp - e0) * n_h + tile_x0 - hp + lane;
        for (int y = tid >> 5; y < R; y += kCThreads / 32) {
            uint32_t dst = rsa + 8u * (uint32_t)(y * P + lane);
            const float2 *sr = src + (int64_t)y * n_h;
#pragma unroll
            for (int x = 0; x < R; x += 32, dst += 256u)
                if (x + lane < R) asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(sr + x) : "memory");
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    } else {
        for (int y = (tid >> 5) - hp; y < kCT + hp; y += kCThreads / 32) {
            const bool rok = y >= ylo && y < yhi;
            const float2 *src = psi + (tile_y0 + y - e0) * n_h + tile_x0;
            uint32_t dst = rsa + 8u * (uint32_t)((y + hp) * P + lane);
            for (int x = lane - hp; x < kCT + hp; x += 32, dst += 256u) {
                const bool ok = rok && x >= xlo && x < xhi;
                asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(dst), "l"(ok ? src + x : psi),
                             "r"(ok ? 8 : 0) : "memory");
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
    coif_levels<L, L>(reg, h0, h1, ylo, yhi, xlo, xhi);
    // step 4 on the tile (same print_byte as quantize_kernel) and the u write
    auto cell = [&](int y, int x) -> const float2 & { return reg[(y + hp) * P + (x + hp)]; };
    if (bits) {
        for (int b = tid; b < kCT * (kCT / 8); b += kCThreads) {   // lanes on adjacent rows: no bank conflicts
            const int y = b % kCT, xb = b / kCT;
            float2 v[8];
#pragma unroll
            for (int i = 0; i < 8; i++) v[i] = cell(y, xb * 8 + i);
            const int64_t Y = tile_y0 + y;
            bits[(Y - row0) * (n_h / 8) + tile_x0 / 8 + xb] = (uint8_t)print_byte(v, tile_x0 + xb * 8, ref_row(Y, qa), qa);
        }
    }
    if (u) {
        float2 *out = u + (tile_y0 - row0) * n_h + tile_x0;
        for (int y = tid >> 5; y < kCT; y += kCThreads / 32) {
            __stcs(out + y * n_h + lane, cell(y, lane));
            __stcs(out + y * n_h + lane + 32, cell(y, lane + 32));
        }
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
    for (int l = L; l >= 1; l--) {
        const int sgrid = 1 << (l - 1);
        const unsigned ncols = (unsigned)(n_h / sgrid), nrow = (unsigned)(nrows / sgrid);
        count_launches(2);
        fb_inv_cols_kernel<<<(ncols + 31) / 32, 256, 0, s>>>(psi, nrows, n_h, l, F);
        fb_inv_rows_kernel<<<nrow, 256, 0, s>>>(psi, nrows, n_h, l, F);
    }
    return cudaGetLastError();
}

}  // namespace wasabi

namespace wasabi {
// Fused coif1 synthesis + quantise of band [row0, row1) from the halo band psi [e0, e1) (read only).
cudaError_t launch_coif_fused(const float2 *psi, int64_t e0, int64_t e1, int64_t row0, int64_t row1, int64_t n_h,
                              int L, const double *print4, double pitch, float2 *u, uint8_t *bits, cudaStream_t s) {
    const Filt F = coif1();
    const QArgs qa = make_qargs(print4, pitch, n_h);
    const int hp = coif_a(L, L), R = kCT + 2 * hp;
    const int smem = R * (R + 1) * (int)sizeof(float2);
    const int64_t tiles = (n_h / kCT) * ((row1 - row0) / kCT);
    auto go = [&](auto kern) -> cudaError_t {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        if (tiles > 0) {
            count_launches(1);
            kern<<<(unsigned)tiles, kCThreads, smem, s>>>(psi, e0, e1, row0, n_h, F, qa, u, bits);
        }
        return cudaGetLastError();
    };
    switch (L) {
        case 1: return go(coif_synth_tile_kernel<1>);
        case 2: return go(coif_synth_tile_kernel<2>);
        case 3: return go(coif_synth_tile_kernel<3>);
        case 4: return go(coif_synth_tile_kernel<4>);
        default: return cudaErrorInvalidValue;
    }
}
}  // namespace wasabi
