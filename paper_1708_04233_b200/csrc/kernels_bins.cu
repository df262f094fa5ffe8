// kernels_bins.cu -- step 2a of WASABI: point conversion and the tile-binning counting sort
// (the paper re-bases all points per N_h x N_h sub-hologram; here every point
// is listed in the T x T tiles its PSF footprint overlaps, within the caller's row band).
//   K3a convert + count (fp64 conversion, R-A3/R-A9/R-A17), K3b scan, K3c scatter (atomic
//   slots), K3d per-tile sort so each bin lists points in ascending index order (R-A11) --
//   deterministic bins, and a deterministic per-pixel accumulation order downstream.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace wasabi {
namespace {

__device__ __forceinline__ long long floor_div(long long a, long long b) {
    long long q = a / b;
    if ((a % b != 0) && (a < 0)) q--;
    return q;
}

struct BinArgs {
    int64_t n;
    int64_t n_h, row0, row1;
    int T, tiles_x, tiles_y, n_depth, cls_bits;
    int psf;              // 1: footprint = the whole PSF disc (Ed, Qd; bins of the direct sum)
    double pitch, z_min, dz;
};

// Per-point conversion (fp64, same IEEE sequence as the specification):
//   ix = floor(x/p + 1/2) + N_h/2, iy likewise (R-A9);
//   t = (z - z_min)/dz, valid iff -1/2 <= t <= N_z - 1/2, iz = clamp(ceil(t - 1/2)) (R-A3, R-A17);
//   a must be finite and > 0.
__device__ __forceinline__ bool convert_point(const float4 p, const BinArgs &A, int &ix, int &iy, int &iz) {
    if (!isfinite(p.x) || !isfinite(p.y) || !isfinite(p.z) || !isfinite(p.w) || !(p.w > 0.0f)) return false;
    const double u = (double)p.x / A.pitch, v = (double)p.y / A.pitch;
    if (!(fabs(u) <= 1073741824.0) || !(fabs(v) <= 1073741824.0)) return false;
    ix = (int)((long long)floor(u + 0.5) + A.n_h / 2);
    iy = (int)((long long)floor(v + 0.5) + A.n_h / 2);
    if (A.n_depth <= 1) { iz = 0; return true; }
    const double t = ((double)p.z - A.z_min) / A.dz;
    if (t < -0.5 || t > (double)(A.n_depth - 1) + 0.5) return false;
    long long q = (long long)ceil(t - 0.5);
    if (q < 0) q = 0;
    if (q > A.n_depth - 1) q = A.n_depth - 1;
    iz = (int)q;
    return true;
}

// Tile range of a point's footprint square [ix-E, ix+E] x [iy-E, iy+E] within the band (E = Ek).
// (T is 64 or 128, wasabi_params validation: floor division is an arithmetic shift)
__device__ __forceinline__ void tile_range(int ix, int iy, int E, const BinArgs &A, int &tx0, int &tx1, int &ty0,
                                           int &ty1) {
    const int sh = A.T == 64 ? 6 : 7;
    tx0 = (int)max(0LL, ((long long)ix - E) >> sh);
    tx1 = (int)min((long long)A.tiles_x - 1, ((long long)ix + E) >> sh);
    ty0 = (int)max(0LL, ((long long)iy - E - A.row0) >> sh);
    ty1 = (int)min((long long)A.tiles_y - 1, ((long long)iy + E - A.row0) >> sh);
}

// Squared distance from coordinate i to the tile span [t0, t0 + T - 1] along one axis (0 inside).
// With the square test of tile_range this is the footprint of R-A19: a tile is listed iff its
// pixel nearest to (ix, iy) lies within squared distance Q of the point.
__device__ __forceinline__ int sq_gap(int i, int t0, int T) {
    const int g = i < t0 ? t0 - i : (i > t0 + T - 1 ? i - (t0 + T - 1) : 0);
    return g * g;
}

// The tiles of a point's footprint (R-A19): the square [ix - Ek, ix + Ek]^2 clipped to the band,
// then the squared-distance test.  Warp-cooperative: the 32 points of a warp are taken one at a time
// and the lanes walk that point's tile box (a footprint is ~10 x 10 tiles at C4), so the atomics of
// a point are issued in parallel instead of one after the other by one thread.
template <typename F>
__device__ __forceinline__ void warp_footprint(int4 q, bool valid, const KDesc *__restrict__ kd, const BinArgs &A,
                                               int lane, F &&f) {
    unsigned vm = __ballot_sync(0xffffffffu, valid);
    while (vm) {
        const int src = __ffs(vm) - 1;
        vm &= vm - 1u;
        const int ix = __shfl_sync(0xffffffffu, q.x, src), iy = __shfl_sync(0xffffffffu, q.y, src);
        const int iz = __shfl_sync(0xffffffffu, q.z, src);
        const int tb = table_of(ix, iy, iz, A.cls_bits);
        const int Q = A.psf ? __ldg(&kd[tb].Qd) : __ldg(&kd[tb].Q);
        int tx0, tx1, ty0, ty1;
        tile_range(ix, iy, A.psf ? __ldg(&kd[tb].Ed) : __ldg(&kd[tb].Ek), A, tx0, tx1, ty0, ty1);
        const int w = tx1 - tx0 + 1, hgt = ty1 - ty0 + 1;
        if (w <= 0 || hgt <= 0) continue;              // footprint entirely outside the band
        const int nbox = w * hgt;
        // box cell i = lane + 32 k -> (row i / w, column i % w), stepped without a division per cell
        const int q32 = 32 / w, r32 = 32 - q32 * w;
        int qy = lane / w, rx = lane - qy * w;
        for (int i = lane; i < nbox; i += 32) {
            const int ty = ty0 + qy, tx = tx0 + rx;
            const int rem = Q - sq_gap(iy, (int)A.row0 + ty * A.T, A.T);
            if (rem >= 0 && sq_gap(ix, tx * A.T, A.T) <= rem) f((int64_t)ty * A.tiles_x + tx, src);
            qy += q32;
            rx += r32;
            if (rx >= w) { rx -= w; qy++; }
        }
    }
}

__global__ void __launch_bounds__(256) convert_count_kernel(const float4 *__restrict__ pts, BinArgs A,
                                                            const KDesc *__restrict__ kd, int4 *__restrict__ pout,
                                                            uint32_t *__restrict__ cnt, BinHeader *bh) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool valid = false;
    int4 q = make_int4(0, 0, -1, 0);
    if (j < A.n) {
        const float4 p = pts[j];
        int ix = 0, iy = 0, iz = 0;
        valid = convert_point(p, A, ix, iy, iz);
        q = make_int4(ix, iy, valid ? iz : -1, __float_as_int(p.w));
        pout[j] = q;
    }
    const int lane = threadIdx.x & 31;
    warp_footprint(q, valid, kd, A, lane, [&](int64_t t, int) { atomicAdd(&cnt[t], 1u); });
    const unsigned vb = __ballot_sync(0xffffffffu, valid);
    const unsigned ib = __ballot_sync(0xffffffffu, j < A.n && !valid);
    if (lane == 0) {
        if (vb) atomicAdd(&bh->n_valid, (unsigned long long)__popc(vb));
        if (ib) atomicAdd(&bh->n_skipped, (unsigned long long)__popc(ib));
    }
}

// cursor mode (every bin position < 2^32): fill[t] starts at ptr[t] (init_cursor_kernel) and the
// atomic returns the entry's absolute position -- no per-pair load of ptr[t]
__global__ void __launch_bounds__(256) scatter_kernel(BinArgs A, const KDesc *__restrict__ kd,
                                                      const int4 *__restrict__ pconv,
                                                      const unsigned long long *__restrict__ ptr,
                                                      uint32_t *__restrict__ fill, uint32_t *__restrict__ idx,
                                                      int cursor) {
    const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int4 q = j < A.n ? pconv[j] : make_int4(0, 0, -1, 0);
    const int64_t j0 = j - (threadIdx.x & 31);           // point index of lane 0
    if (cursor) {
        warp_footprint(q, q.z >= 0, kd, A, threadIdx.x & 31, [&](int64_t t, int src) {
            idx[atomicAdd(&fill[t], 1u)] = (uint32_t)(j0 + src);
        });
    } else {
        warp_footprint(q, q.z >= 0, kd, A, threadIdx.x & 31, [&](int64_t t, int src) {
            const uint32_t slot = atomicAdd(&fill[t], 1u);
            idx[ptr[t] + slot] = (uint32_t)(j0 + src);
        });
    }
}

__global__ void __launch_bounds__(256) init_cursor_kernel(const unsigned long long *__restrict__ ptr,
                                                          uint32_t *__restrict__ cur, int64_t n) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (t < n) cur[t] = (uint32_t)ptr[t];
}

// Warp-per-tile bitonic sort for bins of <= 1024 entries, in registers: element i = 32 e + lane
// (E = m / 32 per lane, m = the next power of two >= max(n, 32)); stages with partner distance
// j < 32 exchange through shuffles, j >= 32 between a lane's own registers.  Larger bins are queued.
constexpr int kSmallBin = 1024;
template <int E>
__device__ __forceinline__ void warp_sort_bin(uint32_t *__restrict__ idx, unsigned long long b, int n, int lane) {
    uint32_t v[E];
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int i = 32 * e + lane;
        v[e] = i < n ? idx[b + i] : 0xffffffffu;
    }
#pragma unroll
    for (int k = 2; k <= 32 * E; k <<= 1) {
#pragma unroll
        for (int j = k >> 1; j > 0; j >>= 1) {
            if (j >= 32) {
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const int p = e ^ (j >> 5);
                    if (p > e) {
                        const bool up = ((32 * e + lane) & k) == 0;
                        const uint32_t x = v[e], y = v[p];
                        if ((x > y) == up) { v[e] = y; v[p] = x; }
                    }
                }
            } else {
#pragma unroll
                for (int e = 0; e < E; e++) {
                    const uint32_t o = __shfl_xor_sync(0xffffffffu, v[e], j);
                    const bool up = ((32 * e + lane) & k) == 0;
                    const bool lower = (lane & j) == 0;
                    v[e] = (lower == up) ? min(v[e], o) : max(v[e], o);
                }
            }
        }
    }
#pragma unroll
    for (int e = 0; e < E; e++) {
        const int i = 32 * e + lane;
        if (i < n) idx[b + i] = v[e];
    }
}

__global__ void __launch_bounds__(256) sort_small_kernel(int64_t n_tiles, const unsigned long long *__restrict__ ptr,
                                                         uint32_t *__restrict__ idx, uint32_t *__restrict__ big_list,
                                                         unsigned int *big_count) {
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t t = (int64_t)blockIdx.x * 8 + w;
    if (t >= n_tiles) return;
    const unsigned long long b = ptr[t], e = ptr[t + 1];
    const int n = (int)(e - b);
    if (n <= 1) return;
    if (n > kSmallBin) {
        if (lane == 0) big_list[atomicAdd(big_count, 1u)] = (uint32_t)t;
        return;
    }
    if (n <= 32) warp_sort_bin<1>(idx, b, n, lane);
    else if (n <= 64) warp_sort_bin<2>(idx, b, n, lane);
    else if (n <= 128) warp_sort_bin<4>(idx, b, n, lane);
    else if (n <= 256) warp_sort_bin<8>(idx, b, n, lane);
    else if (n <= 512) warp_sort_bin<16>(idx, b, n, lane);
    else warp_sort_bin<32>(idx, b, n, lane);
}

// Large bins: one CTA per queued tile; 4096-entry chunks sorted in shared memory, then merge
// passes (each element's output rank = own index + lower_bound in the partner run; indices are
// unique) ping-ponging between idx and idx2.
constexpr int kChunk = 4096;
__global__ void __launch_bounds__(512) sort_large_kernel(const unsigned long long *__restrict__ ptr,
                                                         uint32_t *idx, uint32_t *idx2,
                                                         const uint32_t *__restrict__ big_list,
                                                         const unsigned int *__restrict__ big_count) {
    __shared__ uint32_t s[kChunk];
    const unsigned nb = *big_count;
    for (unsigned bi = blockIdx.x; bi < nb; bi += gridDim.x) {
        const int64_t t = big_list[bi];
        const unsigned long long b = ptr[t];
        const int64_t n = (int64_t)(ptr[t + 1] - b);
        uint32_t *src = idx + b, *dst = idx2 + b;
        for (int64_t c0 = 0; c0 < n; c0 += kChunk) {
            const int cn = (int)((n - c0) < kChunk ? (n - c0) : kChunk);
            int m = 2;
            while (m < cn) m <<= 1;
            for (int i = threadIdx.x; i < m; i += blockDim.x) s[i] = i < cn ? src[c0 + i] : 0xffffffffu;
            __syncthreads();
            for (int k = 2; k <= m; k <<= 1)
                for (int jj = k >> 1; jj > 0; jj >>= 1) {
                    for (int i = threadIdx.x; i < m; i += blockDim.x) {
                        const int l = i ^ jj;
                        if (l > i) {
                            const uint32_t x = s[i], y = s[l];
                            const bool up = (i & k) == 0;
                            if ((x > y) == up) { s[i] = y; s[l] = x; }
                        }
                    }
                    __syncthreads();
                }
            for (int i = threadIdx.x; i < cn; i += blockDim.x) src[c0 + i] = s[i];
            __syncthreads();
        }
        for (int64_t wdt = kChunk; wdt < n; wdt <<= 1) {
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
                const int64_t run = i / wdt, r0 = run * wdt, own = i - r0;
                const bool left = (run & 1) == 0;
                const int64_t p0 = left ? r0 + wdt : r0 - wdt;           // partner run start
                const int64_t p1 = min(p0 + wdt, n);
                const int64_t out0 = left ? r0 : p0;                      // merged block start
                const uint32_t x = src[i];
                int64_t lo = p0, hi = p0 < n ? p1 : p0;
                while (lo < hi) {
                    const int64_t mid = (lo + hi) >> 1;
                    if (src[mid] < x) lo = mid + 1; else hi = mid;
                }
                dst[out0 + own + (lo - p0)] = x;
            }
            __syncthreads();
            uint32_t *tmp = src; src = dst; dst = tmp;
        }
        if (src != idx + b)
            for (int64_t i = threadIdx.x; i < n; i += blockDim.x) idx[b + i] = src[i];
        __syncthreads();
    }
}

__global__ void finish_kernel(BinHeader *bh, const unsigned long long *ptr, int64_t n_tiles) {
    bh->total_entries = ptr[n_tiles];
    if (ptr[n_tiles] > (unsigned long long)bh->capacity) bh->status = 1;
}

// ---- Eq.(2) accumulation count and per-row work (diagnostics / band balancing, not the hot path) ----
// One warp per point: the lanes walk the point's canonical kept list (16-byte entries, X | Y << 14 |
// l << 28) and count the targets (s + X - H, s + Y - H) inside [0, n_h) x [row0, row1), s the point's
// shift (R-A8 standard: s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l); R-A20 exact: i with the class bits
// cleared) -- the exact number of Eq.(2) accumulations of the band.  With row_diff != NULL the
// point's full-hologram count is also spread uniformly over its reach rows [iy - Ek, iy + Ek] of a
// difference array (the work model of the balanced row bands).
__global__ void __launch_bounds__(256) count_acc_kernel(const float4 *__restrict__ pts, BinArgs A,
                                                        const KDesc *__restrict__ kd, const DDesc *__restrict__ dd,
                                                        const int32_t *__restrict__ gptr,
                                                        const uint4 *__restrict__ ent, int L,
                                                        unsigned long long *__restrict__ count,
                                                        double *__restrict__ row_diff) {
    const int lane = threadIdx.x & 31;
    const int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    if (j >= A.n) return;
    int ix = 0, iy = 0, iz = 0;
    if (!convert_point(pts[j], A, ix, iy, iz)) return;
    const int t = table_of(ix, iy, iz, A.cls_bits);
    const int H = kd[t].H;
    const int e0 = gptr[dd[t].group_base], e1 = gptr[dd[t].group_base + dd[t].n_groups];
    const int cm = (1 << A.cls_bits) - 1;
    unsigned long long band = 0, full = 0;
    for (int e = e0 + lane; e < e1; e += 32) {
        const uint32_t w = ent[e].x;
        const int X = (int)(w & 0x3fffu), Y = (int)((w >> 14) & 0x3fffu), l = (int)(w >> 28);
        const int h = 1 << (l - 1);
        const long long sx = A.cls_bits ? (ix & ~cm) : floor_div((long long)ix + h, 1LL << l) << l;
        const long long sy = A.cls_bits ? (iy & ~cm) : floor_div((long long)iy + h, 1LL << l) << l;
        const long long Xh = sx + X - H, Yh = sy + Y - H;
        if (Xh >= 0 && Xh < A.n_h && Yh >= 0 && Yh < A.n_h) {
            full++;
            if (Yh >= A.row0 && Yh < A.row1) band++;
        }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
        band += __shfl_xor_sync(0xffffffffu, band, o);
        full += __shfl_xor_sync(0xffffffffu, full, o);
    }
    if (lane == 0) {
        if (band) atomicAdd(count, band);
        if (row_diff && full) {
            const int ek = kd[t].Ek;
            const long long y0 = max(0LL, (long long)iy - ek), y1 = min((long long)A.n_h - 1, (long long)iy + ek);
            if (y1 >= y0) {
                const double wrow = (double)full / (double)(y1 - y0 + 1);
                atomicAdd(&row_diff[y0], wrow);
                atomicAdd(&row_diff[y1 + 1], -wrow);
            }
        }
    }
}

// In-place inclusive scan of n doubles by one CTA (the per-row work array: n = N_h <= 2^17).
__global__ void __launch_bounds__(1024) scan_rows_kernel(double *__restrict__ a, int64_t n) {
    __shared__ double part[1024];
    const int64_t per = (n + 1023) / 1024;
    const int64_t b = threadIdx.x * per, e = min(n, b + per);
    double s = 0.0;
    for (int64_t i = b; i < e; i++) s += a[i];
    part[threadIdx.x] = s;
    __syncthreads();
    for (int o = 1; o < 1024; o <<= 1) {
        const double v = threadIdx.x >= o ? part[threadIdx.x - o] : 0.0;
        __syncthreads();
        part[threadIdx.x] += v;
        __syncthreads();
    }
    double c = threadIdx.x ? part[threadIdx.x - 1] : 0.0;
    for (int64_t i = b; i < e; i++) {
        c += a[i];
        a[i] = c;
    }
}

}  // namespace

cudaError_t launch_count_acc(const TableHeader &h, const void *d_tables, const float4 *pts, int64_t n, double pitch,
                             int64_t n_h, double z_min, double dz, int n_depth, int cls_bits, int L, int64_t row0,
                             int64_t row1, unsigned long long *d_count, double *d_row_work, cudaStream_t s) {
    const char *tb = static_cast<const char *>(d_tables);
    cudaError_t e;
    BinArgs A;
    A.n = n; A.n_h = n_h; A.row0 = row0; A.row1 = row1;
    A.T = h.tile; A.tiles_x = 0; A.tiles_y = 0; A.n_depth = n_depth; A.cls_bits = cls_bits; A.psf = 0;
    A.pitch = pitch; A.z_min = z_min; A.dz = dz;
    if ((e = cudaMemsetAsync(d_count, 0, sizeof(unsigned long long), s)) != cudaSuccess) return e;
    if (d_row_work && (e = cudaMemsetAsync(d_row_work, 0, sizeof(double) * (size_t)(n_h + 1), s)) != cudaSuccess)
        return e;
    if (n > 0) {
        count_launches(1);
        count_acc_kernel<<<(unsigned)((n * 32 + 255) / 256), 256, 0, s>>>(
            pts, A, reinterpret_cast<const KDesc *>(tb + h.kdesc_off), reinterpret_cast<const DDesc *>(tb + h.ddesc_off),
            reinterpret_cast<const int32_t *>(tb + h.ptr_off), reinterpret_cast<const uint4 *>(tb + h.ent_off), L,
            d_count, d_row_work);
    }
    if (d_row_work) {
        count_launches(1);
        scan_rows_kernel<<<1, 1024, 0, s>>>(d_row_work, n_h);
    }
    return cudaGetLastError();
}

cudaError_t launch_bin(const BinHeader &h, void *d_bins, const KDesc *kd, const float4 *pts, double pitch,
                       int64_t n_h, double z_min, double dz, int n_depth, int cls_bits, int psf, cudaStream_t s) {
    char *base = reinterpret_cast<char *>(d_bins);
    BinHeader *bh = reinterpret_cast<BinHeader *>(base);
    int4 *pconv = reinterpret_cast<int4 *>(base + h.pts_off);
    unsigned long long *ptr = reinterpret_cast<unsigned long long *>(base + h.ptr_off);
    uint32_t *cnt = reinterpret_cast<uint32_t *>(base + h.cnt_off);
    uint32_t *idx = reinterpret_cast<uint32_t *>(base + h.idx_off);
    uint32_t *idx2 = reinterpret_cast<uint32_t *>(base + h.idx2_off);
    void *scan_scratch = base + h.scan_off;
    // the big-bin queue lives after the scan scratch
    uint32_t *big_list = reinterpret_cast<uint32_t *>(base + h.scan_off + scan_scratch_bytes(h.n_tiles + 1));
    unsigned int *big_count = reinterpret_cast<unsigned int *>(big_list + h.n_tiles);

    BinArgs A;
    A.n = h.n_points; A.n_h = n_h; A.row0 = h.row0; A.row1 = h.row1;
    A.T = h.T; A.tiles_x = h.tiles_x; A.tiles_y = h.tiles_y; A.n_depth = n_depth; A.cls_bits = cls_bits;
    A.psf = psf;
    A.pitch = pitch; A.z_min = z_min; A.dz = dz;
    cudaError_t e;
    if ((e = cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (size_t)(h.n_tiles + 1), s)) != cudaSuccess) return e;
    if ((e = cudaMemsetAsync(big_count, 0, sizeof(unsigned int), s)) != cudaSuccess) return e;
    const unsigned pb = (unsigned)((h.n_points + 255) / 256);
    if (h.n_points > 0) {
        count_launches(1);
        convert_count_kernel<<<pb, 256, 0, s>>>(pts, A, kd, pconv, cnt, bh);
    }
    if ((e = launch_scan_u32_to_u64(cnt, ptr, h.n_tiles + 1, scan_scratch, s)) != cudaSuccess) return e;
    const int cursor = h.capacity < (int64_t)0xffffffffLL;   // every bin position fits the 32-bit cursor
    if (cursor) {
        count_launches(1);
        init_cursor_kernel<<<(unsigned)((h.n_tiles + 1 + 255) / 256), 256, 0, s>>>(ptr, cnt, h.n_tiles + 1);
    } else if ((e = cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (size_t)(h.n_tiles + 1), s)) != cudaSuccess) {
        return e;
    }
    if (h.n_points > 0) {
        count_launches(1);
        scatter_kernel<<<pb, 256, 0, s>>>(A, kd, pconv, ptr, cnt, idx, cursor);
    }
    count_launches(1);
    sort_small_kernel<<<(unsigned)((h.n_tiles + 7) / 8), 256, 0, s>>>(h.n_tiles, ptr, idx, big_list, big_count);
    count_launches(1);
    sort_large_kernel<<<148 * 2, 512, 0, s>>>(ptr, idx, idx2, big_list, big_count);
    count_launches(1);
    finish_kernel<<<1, 1, 0, s>>>(bh, ptr, h.n_tiles);
    return cudaGetLastError();
}

}  // namespace wasabi
