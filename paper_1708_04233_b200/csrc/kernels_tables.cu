// kernels_tables.cu -- step 1 of WASABI: per-depth PSF, forward Haar, top-N_r
// selection and the LUT with its per-level band index.  Compiled with --fmad=false and explicit
// _rn intrinsics on the key path so that the fp32 rank keys are computed with the same IEEE
// operation sequence as the specification (K1/K2).  Off the per-frame hot loop:
// one launch set per parameter set.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace wasabi {
namespace {

__device__ __forceinline__ const TableHeader &hdr(const void *t) {
    return *reinterpret_cast<const TableHeader *>(t);
}
template <typename T>
__device__ __forceinline__ const T *at(const void *t, int64_t off) {
    return reinterpret_cast<const T *>(reinterpret_cast<const char *>(t) + off);
}
template <typename T>
__device__ __forceinline__ T *atw(void *t, int64_t off) {
    return reinterpret_cast<T *>(reinterpret_cast<char *>(t) + off);
}

__device__ __forceinline__ int kdh(const void *t, int d) {
    return at<KDesc>(t, hdr(t).kdesc_off)[d].H;
}

// CTA -> table: largest d with cta_base[d] <= b (cta_base has n_tables + 1 entries).
__device__ __forceinline__ int find_depth(const int32_t *base, int n, int64_t b) {
    int lo = 0, hi = n;  // invariant base[lo] <= b < base[hi]
    while (hi - lo > 1) {
        int mid = (lo + hi) >> 1;
        if (base[mid] <= b) lo = mid; else hi = mid;
    }
    return lo;
}

constexpr int kTile = 64;

// K1: one CTA per 64x64 region of one depth table.  PSF u_z = exp(i k r) circ(.) with r =
// sqrt((dx p)^2 + (dy p)^2 + z^2), support S = {dx^2+dy^2 < R^2} U {0}
// (R-A2), then L forward Haar levels in shared memory in fp64 with the butterfly order
// LL=((a+b)+(c+d))/2, HL=((a-b)+(c-d))/2, LH=((a+b)-(c+d))/2, HH=((a-b)-(c-d))/2 (R-A6).
// Output: fp32 value and the rank key bits of fp32_RN(re^2 + im^2) (R-A13).
__global__ void __launch_bounds__(256) psf_haar_kernel(const void *tables, float2 *__restrict__ coef_val,
                                                       uint32_t *__restrict__ coef_key, double k, double pitch,
                                                       int L, int n_depth) {
    extern __shared__ double2 f[];  // 64 x 64
    const TableHeader &h = hdr(tables);
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    const int32_t *cbase = at<int32_t>(tables, h.ctabase_off);
    const int d = find_depth(cbase, n_depth, blockIdx.x);
    const DDesc D = dd[d];
    const int local = (int)blockIdx.x - D.cta_base;
    const int X0 = (local % D.tiles) * kTile, Y0 = (local / D.tiles) * kTile;
    const int side = D.side;
    const int Cx = kdh(tables, d) + D.cx, Cy = kdh(tables, d) + D.cy;   // PSF centre (R-A20: offset class)
    const double R2 = __dmul_rn(D.R, D.R);
    const double z2 = __dmul_rn(D.z, D.z);

    for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
        const int x = i & (kTile - 1), y = i >> 6;
        const int X = X0 + x, Y = Y0 + y;
        double2 v = make_double2(0.0, 0.0);
        if (X < side && Y < side) {
            const long long dx = X - Cx, dy = Y - Cy;
            const bool in = (dx == 0 && dy == 0) || ((double)(dx * dx + dy * dy) < R2);
            if (in) {
                const double xp = __dmul_rn((double)dx, pitch), yp = __dmul_rn((double)dy, pitch);
                const double r = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(xp, xp), __dmul_rn(yp, yp)), z2));
                double s, c;
                sincos(__dmul_rn(k, r), &s, &c);
                v = make_double2(c, s);
            }
        }
        f[i] = v;
    }
    __syncthreads();
    for (int l = 1; l <= L; l++) {
        const int bs = 1 << l, st = bs >> 1, nqs = kTile >> l;
        for (int q = threadIdx.x; q < nqs * nqs; q += blockDim.x) {
            const int bx = (q % nqs) << l, by = (q / nqs) << l;
            double2 *pa = &f[by * kTile + bx], *pb = pa + st, *pc = pa + st * kTile, *pd = pc + st;
            const double2 a = *pa, b = *pb, c = *pc, e = *pd;
            double2 LL, HL, LH, HH;
            LL.x = __dadd_rn(__dadd_rn(a.x, b.x), __dadd_rn(c.x, e.x)) * 0.5;
            HL.x = __dadd_rn(__dsub_rn(a.x, b.x), __dsub_rn(c.x, e.x)) * 0.5;
            LH.x = __dsub_rn(__dadd_rn(a.x, b.x), __dadd_rn(c.x, e.x)) * 0.5;
            HH.x = __dsub_rn(__dsub_rn(a.x, b.x), __dsub_rn(c.x, e.x)) * 0.5;
            LL.y = __dadd_rn(__dadd_rn(a.y, b.y), __dadd_rn(c.y, e.y)) * 0.5;
            HL.y = __dadd_rn(__dsub_rn(a.y, b.y), __dsub_rn(c.y, e.y)) * 0.5;
            LH.y = __dsub_rn(__dadd_rn(a.y, b.y), __dadd_rn(c.y, e.y)) * 0.5;
            HH.y = __dsub_rn(__dsub_rn(a.y, b.y), __dsub_rn(c.y, e.y)) * 0.5;
            *pa = LL; *pb = HL; *pc = LH; *pd = HH;
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
        const int x = i & (kTile - 1), y = i >> 6;
        const int X = X0 + x, Y = Y0 + y;
        if (X < side && Y < side) {
            const double2 v = f[i];
            const int64_t o = D.coef_off + (int64_t)Y * side + X;
            coef_val[o] = make_float2(__double2float_rn(v.x), __double2float_rn(v.y));
            const double m2 = __dadd_rn(__dmul_rn(v.x, v.x), __dmul_rn(v.y, v.y));
            coef_key[o] = __float_as_uint(__double2float_rn(m2));
        }
    }
}

// Selection state per depth: {prefix, mask, remaining k} of the composite 64-bit key
// (kappa_bits << 32) | ~linear_index: larger key = larger |c|^2, then smaller index (R-A13).
struct SelState {
    unsigned long long prefix, mask, k;
};

// K2a: radix-select histogram pass (8 passes of 8 bits, MSB first) over keys matching the prefix.
__global__ void __launch_bounds__(256) select_hist_kernel(const void *tables, const uint32_t *__restrict__ coef_key,
                                                          unsigned int *__restrict__ hist,
                                                          const SelState *__restrict__ st, int n_depth, int pass) {
    __shared__ unsigned int sh[256];
    const TableHeader &h = hdr(tables);
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    const int32_t *cbase = at<int32_t>(tables, h.ctabase_off);
    const int d = find_depth(cbase, n_depth, blockIdx.x);
    const DDesc D = dd[d];
    const int local = (int)blockIdx.x - D.cta_base;
    const int X0 = (local % D.tiles) * kTile, Y0 = (local / D.tiles) * kTile;
    const int side = D.side;
    const SelState s = st[d];
    if (s.k == 0) return;   // this depth's threshold is already exact (select_pick_kernel)
    const int shift = 56 - 8 * pass;
    sh[threadIdx.x] = 0;
    __syncthreads();
    for (int i = threadIdx.x; i < kTile * kTile; i += blockDim.x) {
        const int X = X0 + (i & (kTile - 1)), Y = Y0 + (i >> 6);
        if (X < side && Y < side) {
            const uint32_t lin = (uint32_t)(Y * side + X);
            const unsigned long long key = ((unsigned long long)coef_key[D.coef_off + (int64_t)Y * side + X] << 32) |
                                           (unsigned long long)(~lin);
            if ((key & s.mask) == s.prefix) atomicAdd(&sh[(key >> shift) & 255u], 1u);
        }
    }
    __syncthreads();
    const unsigned int c = sh[threadIdx.x];
    if (c) atomicAdd(&hist[d * 256 + threadIdx.x], c);
}

// K2b: per depth (one warp), choose the digit containing the k-th largest key; zero the histogram.
// Lane t holds digits 255 - 8 t .. 248 - 8 t (descending); a warp scan of the lane sums finds the lane
// whose digits reach the k-th key, that lane scans its own 8: digit b = the largest with
// sum(hist[b..255]) >= k, as the serial scan from 255 down.
__global__ void select_pick_kernel(unsigned int *hist, SelState *st, int n_depth, int pass) {
    const int d = (int)((blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
    if (d >= n_depth) return;
    SelState s = st[d];
    if (s.k == 0) return;   // done in an earlier pass (warp-uniform)
    const int shift = 56 - 8 * pass;
    unsigned int h[8];
    unsigned long long tot = 0;
#pragma unroll
    for (int q = 0; q < 8; q++) { h[q] = hist[d * 256 + 255 - 8 * lane - q]; tot += h[q]; }
    unsigned long long incl = tot;   // inclusive scan over lanes (descending digits)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const unsigned long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    const unsigned reach = __ballot_sync(0xffffffffu, incl >= s.k);
    const int src = __ffs(reach) - 1;          // first lane whose prefix reaches k (k <= the total: exists)
    unsigned long long cum = 0, cnt = 0;
    int digit = 0;
    if (lane == src) {
        cum = incl - tot;                      // keys in the digits above this lane's
        for (int q = 0; q < 8; q++) {
            if (cum + h[q] >= s.k) { digit = 255 - 8 * lane - q; cnt = h[q]; break; }
            cum += h[q];
        }
    }
#pragma unroll
    for (int q = 0; q < 8; q++) hist[d * 256 + 255 - 8 * lane - q] = 0;
    if (lane != src) return;
    s.k -= cum;
    s.prefix |= (unsigned long long)digit << shift;
    s.mask |= 0xFFull << shift;
    // every key under the new prefix is kept: key >= prefix (lower digits 0) is already the exact
    // top-N_r set, so the remaining passes skip this depth (k = 0 marks it)
    if (cnt == s.k) s.k = 0;
    st[d] = s;
}

__global__ void select_init_kernel(const void *tables, SelState *st, int n_depth) {
    const int d = blockIdx.x * blockDim.x + threadIdx.x;
    if (d >= n_depth) return;
    const TableHeader &h = hdr(tables);
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    st[d].prefix = 0;
    st[d].mask = 0;
    st[d].k = (unsigned long long)dd[d].n_r;
}

// K2c: per (depth, level, band, Xb) group, count (pass 0) or scatter (pass 1) the kept
// coefficients in (Yb, subband) order as 16-byte entries (internal.h pack_entry_pos).
__global__ void __launch_bounds__(256) groups_kernel(void *tables, const float2 *__restrict__ coef_val,
                                                     const uint32_t *__restrict__ coef_key,
                                                     const SelState *__restrict__ st, int n_depth, int L, int T,
                                                     int pass) {
    const TableHeader &h = hdr(tables);
    const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    int d = 0, ek = 0, q = 0;      // this group's depth and kept reach (R-A19, pass 0)
    if (g < h.total_ptrs) {
        const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
        const KDesc *kd = at<KDesc>(tables, h.kdesc_off);
        int32_t *ptr = atw<int32_t>(tables, h.ptr_off);
        // depth: largest d with group_base <= g
        int lo = 0, hi = n_depth;
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (dd[mid].group_base <= g) lo = mid; else hi = mid;
        }
        d = lo;
        const DDesc D = dd[d];
        const KDesc K = kd[d];
        int l = 1;
        while (l < L && K.ptr_base[l] <= g) l++;
        const int side = D.side;
        const int nb = side >> l, hb = band_blocks(T, l);
        const int64_t local = g - K.ptr_base[l - 1];
        const int band = (int)(local / (nb + 1)), Xb = (int)(local % (nb + 1));
        if (Xb == nb) {  // dummy slot: band end
            if (pass == 0) ptr[g] = 0;
        } else {
            const unsigned long long thr = st[d].prefix;
            const int st_px = 1 << (l - 1);
            const int yb1 = min(band * hb + hb, nb);
            int out = pass ? ptr[g] : 0;
            int cnt = 0;
            uint4 *ent = atw<uint4>(tables, h.ent_off);
            for (int Yb = band * hb; Yb < yb1; Yb++) {
                for (int sb = (l == L ? 0 : 1); sb < 4; sb++) {
                    const int sbx = sb & 1, sby = sb >> 1;
                    const int X = (Xb << l) + sbx * st_px, Y = (Yb << l) + sby * st_px;
                    const uint32_t lin = (uint32_t)(Y * side + X);
                    const int64_t o = D.coef_off + (int64_t)Y * side + X;
                    const unsigned long long key = ((unsigned long long)coef_key[o] << 32) | (unsigned long long)(~lin);
                    if (key >= thr) {
                        if (pass) {
                            const float2 v = coef_val[o];
                            ent[out] = make_uint4(pack_entry_pos(X, Y, l), __float_as_uint(v.x), __float_as_uint(v.y), 0u);
                            out++;
                        } else {
                            // target within |dX| + 2^(l-1) of the point per axis (s_l(i) - i in (-h, h]);
                            // offset-class tables: exactly (dX - cx, dY - cy) from the point (R-A20)
                            const bool ex = h.cls_bits != 0;
                            const int ax = ex ? abs(X - K.H - D.cx) : abs(X - K.H) + st_px;
                            const int ay = ex ? abs(Y - K.H - D.cy) : abs(Y - K.H) + st_px;
                            ek = max(ek, max(ax, ay));
                            q = max(q, ax * ax + ay * ay);
                        }
                        cnt++;
                    }
                }
            }
            if (pass == 0) ptr[g] = cnt;
        }
    }
    if (pass == 0) {
        // per-depth max of the reach: one atomic per warp when the warp is within one depth
        KDesc *kdw = atw<KDesc>(tables, h.kdesc_off);
        const int dmin = __reduce_min_sync(0xffffffffu, d), dmax = __reduce_max_sync(0xffffffffu, d);
        if (dmin == dmax) {
            ek = __reduce_max_sync(0xffffffffu, ek);
            q = __reduce_max_sync(0xffffffffu, q);
            if ((threadIdx.x & 31) == 0 && q > 0) { atomicMax(&kdw[d].Ek, ek); atomicMax(&kdw[d].Q, q); }
        } else if (q > 0) {
            atomicMax(&kdw[d].Ek, ek);
            atomicMax(&kdw[d].Q, q);
        }
    }
}

// K2d: the superposition kernel's window LUT (internal.h), built per canonical entry: each kept entry
// (level l, X, Y) of table d belongs, for every variant v of its level, to band k = (Y - v q_l) / 32 + 1
// and column group X >> lg_l.  Pass 0 counts (atomics on the slot counters), pass 1 places it at a
// slot cursor (atomics on a copy of the scanned pointers).  The order inside a group is then
// arbitrary: a window range belongs to one point, whose targets are distinct, so every result is
// bitwise the same whatever that order (R-A11 holds per pixel).  C4: 3e6 entries x ~11 variants.
__global__ void __launch_bounds__(256) ventries_kernel(void *tables, int n_tab, int L, int S, int pass,
                                                       int32_t *__restrict__ cursor) {
    const TableHeader &h = hdr(tables);
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= h.total_entries) return;
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    const KDesc *kd = at<KDesc>(tables, h.kdesc_off);
    const int32_t *ptr = at<int32_t>(tables, h.ptr_off);
    const uint4 en = at<uint4>(tables, h.ent_off)[e];
    // table of entry e: largest d with ptr[group_base_d] <= e (canonical entries are in table order)
    int lo = 0, hi = n_tab;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ptr[dd[mid].group_base] <= e) lo = mid; else hi = mid;
    }
    const int d = lo, side = dd[d].side;
    const int X = (int)(en.x & 0x3fffu), Y = (int)((en.x >> 14) & 0x3fffu), l = (int)(en.x >> 28);
    const int lq = win_lq(l, h.cls_bits), nv = win_variants(l, h.cls_bits), nband = win_bands(side);
    const int ncol = win_cols(side, l), xg = X >> win_lg(l);
    int32_t *vptr = atw<int32_t>(tables, h.vptr_off);
    float2 *vval = atw<float2>(tables, h.vval_off);
    uint16_t *vpos = atw<uint16_t>(tables, h.vpos_off);
    for (int v = 0; v < nv; v++) {
        const int k = ((Y - (v << lq)) >> 5) + 1;            // floor division (arithmetic shift)
        const int bs = (v << lq) + kWinRows * (k - 1);
        const int64_t slot = kd[d].vptr_base[l - 1] + (int64_t)(v * nband + k) * (ncol + 1) + xg;
        if (pass == 0) {
            atomicAdd(&vptr[slot], 1);
        } else {
            const int out = atomicAdd(&cursor[slot], 1);
            vval[out] = make_float2(__uint_as_float(en.y), __uint_as_float(en.z));
            vpos[out] = (uint16_t)((Y - bs) * S + X);
        }
    }
}

// K2e (gather mode, wasabi.h WASABI_FLAG_GATHER): every kept canonical entry (level l, X, Y) of table d
// written at its Mallat position (internal.h mallat_index) of d's dense wavelet table (side_d^2
// complex64, zeroed beforehand).
__global__ void __launch_bounds__(256) dense_fill_kernel(void *tables, int n_tab, int L) {
    const TableHeader &h = hdr(tables);
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= h.total_entries) return;
    const DDesc *dd = at<DDesc>(tables, h.ddesc_off);
    const int32_t *ptr = at<int32_t>(tables, h.ptr_off);
    const uint4 en = at<uint4>(tables, h.ent_off)[e];
    int lo = 0, hi = n_tab;
    while (hi - lo > 1) {
        const int mid = (lo + hi) >> 1;
        if (ptr[dd[mid].group_base] <= e) lo = mid; else hi = mid;
    }
    const int X = (int)(en.x & 0x3fffu), Y = (int)((en.x >> 14) & 0x3fffu);
    float2 *dense = atw<float2>(tables, h.dense_off);
    dense[dd[lo].coef_off + mallat_index(X, Y, dd[lo].side, L)] = make_float2(__uint_as_float(en.y), __uint_as_float(en.z));
}

}  // namespace

cudaError_t launch_dense_fill(const TableHeader &h, void *d_tables, cudaStream_t s) {
    const unsigned blocks = (unsigned)((h.total_entries + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    count_launches(1);
    dense_fill_kernel<<<blocks, 256, 0, s>>>(d_tables, h.n_depth, h.levels);
    return cudaGetLastError();
}

cudaError_t launch_ventries(const TableHeader &h, void *d_tables, int pass, int32_t *cursor, cudaStream_t s) {
    const unsigned blocks = (unsigned)((h.total_entries + 255) / 256);
    if (blocks == 0) return cudaSuccess;
    count_launches(1);
    ventries_kernel<<<blocks, 256, 0, s>>>(d_tables, h.n_depth, h.levels, h.S, pass, cursor);
    return cudaGetLastError();
}


cudaError_t launch_psf_haar(const TableHeader &h, const void *d_tables, float2 *coef_val, uint32_t *coef_key,
                            double k, double pitch, int levels, int n_depth, cudaStream_t s) {
    const int smem = kTile * kTile * sizeof(double2);
    cudaError_t e = cudaFuncSetAttribute(psf_haar_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    count_launches(1);
    psf_haar_kernel<<<(unsigned)h.total_ctas, 256, smem, s>>>(d_tables, coef_val, coef_key, k, pitch, levels,
                                                              n_depth);
    return cudaGetLastError();
}

cudaError_t launch_select(const TableHeader &h, const void *d_tables, const uint32_t *coef_key, unsigned int *hist,
                          unsigned long long *sel_state, int n_depth, cudaStream_t s) {
    SelState *st = reinterpret_cast<SelState *>(sel_state);
    cudaError_t e = cudaMemsetAsync(hist, 0, sizeof(unsigned int) * 256 * (size_t)n_depth, s);
    if (e != cudaSuccess) return e;
    count_launches(1);
    select_init_kernel<<<(n_depth + 127) / 128, 128, 0, s>>>(d_tables, st, n_depth);
    for (int pass = 0; pass < 8; pass++) {
        count_launches(1);
        select_hist_kernel<<<(unsigned)h.total_ctas, 256, 0, s>>>(d_tables, coef_key, hist, st, n_depth, pass);
        count_launches(1);
        select_pick_kernel<<<(n_depth * 32 + 127) / 128, 128, 0, s>>>(hist, st, n_depth, pass);   // a warp per depth
    }
    return cudaGetLastError();
}

cudaError_t launch_groups(const TableHeader &h, void *d_tables, const float2 *coef_val, const uint32_t *coef_key,
                          const unsigned long long *sel_state, int pass, cudaStream_t s) {
    const SelState *st = reinterpret_cast<const SelState *>(sel_state);
    const unsigned blocks = (unsigned)((h.total_ptrs + 255) / 256);
    count_launches(1);
    groups_kernel<<<blocks, 256, 0, s>>>(d_tables, coef_val, coef_key, st, h.n_depth, h.levels, h.tile, pass);
    return cudaGetLastError();
}

}  // namespace wasabi
