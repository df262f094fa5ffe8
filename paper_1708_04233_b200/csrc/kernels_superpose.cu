// kernels_superpose.cu -- step 2b of WASABI, Eq.(2):
//   psi(m, n) = sum_j a_j sum_k c_{z_j,k} delta(m - alpha x_j, n - alpha y_j)
// with alpha = 2^-l for a level-l coefficient (reading R-A8: target X = s_l(ix) + dX,
// s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l)), in the interleaved in-place Haar layout (R-A6).
//
// Design (DESIGN.md §5 K4): one CTA = one warp owns one T x T tile of psi in shared memory; it
// walks the tile's bin (points in ascending order) and, per point, the kept coefficients whose
// target falls in the tile.  Those are found through the per-level band index of the LUT: for
// level l the tile window is a W x W rectangle (W = T/2^l blocks) of the depth's table, covered
// by at most 5 bands; each band gives one contiguous, X-exact entry range.  Lane r of the warp
// computes range r, the ranges are compacted and scanned, and the warp streams the flattened
// entries 32 at a time (one point per chunk, so all targets in a chunk are distinct: no atomics,
// no races).  psi is written once, coalesced.  Accumulation order per pixel is fixed (point
// order), hence bitwise deterministic and independent of the band split.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace wasabi {
namespace {

struct SupArgs {
    int T, S, L, tiles_x;
    int64_t row0, n_h;
};

__global__ void __launch_bounds__(32) superpose_kernel(const void *__restrict__ d_bins,
                                                       const void *__restrict__ d_tables, SupArgs A,
                                                       float2 *__restrict__ psi) {
    extern __shared__ float2 tile[];  // T x S
    __shared__ int4 rng[32];
    const char *bb = reinterpret_cast<const char *>(d_bins);
    const BinHeader *bh = reinterpret_cast<const BinHeader *>(bb);
    const int4 *__restrict__ pconv = reinterpret_cast<const int4 *>(bb + bh->pts_off);
    const unsigned long long *__restrict__ bptr = reinterpret_cast<const unsigned long long *>(bb + bh->ptr_off);
    const uint32_t *__restrict__ bidx = reinterpret_cast<const uint32_t *>(bb + bh->idx_off);
    const char *tb = reinterpret_cast<const char *>(d_tables);
    const TableHeader *th = reinterpret_cast<const TableHeader *>(tb);
    const KDesc *__restrict__ kd = reinterpret_cast<const KDesc *>(tb + th->kdesc_off);
    const int32_t *__restrict__ tptr = reinterpret_cast<const int32_t *>(tb + th->ptr_off);
    const float2 *__restrict__ tval = reinterpret_cast<const float2 *>(tb + th->val_off);
    const uint32_t *__restrict__ tpos = reinterpret_cast<const uint32_t *>(tb + th->pos_off);

    const int lane = threadIdx.x;
    const int T = A.T, S = A.S;
    const int64_t t = blockIdx.x;
    const int tx = (int)(t % A.tiles_x), ty = (int)(t / A.tiles_x);
    const int tile_x0 = tx * T;
    const int tile_y0 = (int)(A.row0 + (int64_t)ty * T);

    for (int i = lane; i < T * S; i += 32) tile[i] = make_float2(0.f, 0.f);

    // lane -> (level, band slot k) of the per-point range table
    int my_l = 0, my_k = 0;
    {
        int base = 0;
        for (int l = 1; l <= A.L; l++) {
            const int W = T >> l, hb = band_blocks(T, l);
            const int m = (hb == 1) ? W : W / hb + 1;
            if (lane >= base && lane < base + m) { my_l = l; my_k = lane - base; }
            base += m;
        }
    }
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const unsigned lanemask_le = lanemask_lt | (1u << lane);
    __syncwarp();

    const unsigned long long b0 = bptr[t], b1 = bptr[t + 1];
    for (unsigned long long pb = b0; pb < b1; pb += 32) {
        const int np = (int)min(32ull, b1 - pb);
        int4 q = make_int4(0, 0, 0, 0);
        if (lane < np) q = pconv[bidx[pb + lane]];
        for (int kk = 0; kk < np; kk++) {
            const int ix = __shfl_sync(0xffffffffu, q.x, kk);
            const int iy = __shfl_sync(0xffffffffu, q.y, kk);
            const int iz = __shfl_sync(0xffffffffu, q.z, kk);
            const float a = __int_as_float(__shfl_sync(0xffffffffu, q.w, kk));
            // ---- this lane's entry range
            int beg = 0, cnt = 0, base = 0, packed = 0;
            if (my_l > 0) {
                const int l = my_l;
                const int H = kd[iz].H;
                const int half = 1 << (l - 1);
                const int sx = (ix + half) >> l, sy = (iy + half) >> l;  // arithmetic shift = floor
                const int Hb = H >> l, nb = (2 * H) >> l, W = T >> l, hb = band_blocks(T, l);
                const int xb0 = (tile_x0 >> l) - sx + Hb, yb0 = (tile_y0 >> l) - sy + Hb;
                const int xb0c = max(xb0, 0), xb1c = min(xb0 + W, nb);
                const int yb0c = max(yb0, 0), yb1c = min(yb0 + W, nb);
                if (xb0c < xb1c && yb0c < yb1c) {
                    const int band = yb0c / hb + my_k;
                    if (band * hb < yb1c) {
                        const int row = kd[iz].ptr_base[l - 1] + band * (nb + 1);
                        beg = tptr[row + xb0c];
                        cnt = tptr[row + xb1c] - beg;
                        const int ulo = max(0, 2 * (yb0c - band * hb));
                        const int uhi = min(2 * hb, 2 * (yb1c - band * hb));
                        base = (((band * hb) << l) - H + (sy << l) - tile_y0) * S + ((sx << l) - H - tile_x0);
                        packed = (l - 1) | (ulo << 8) | (uhi << 16);
                    }
                }
            }
            // ---- compact non-empty ranges to lanes 0..nr-1, exclusive scan of counts
            const unsigned bal = __ballot_sync(0xffffffffu, cnt > 0);
            const int nr = __popc(bal);
            if (cnt > 0) rng[__popc(bal & lanemask_lt)] = make_int4(beg, base, packed, cnt);
            __syncwarp();
            int4 R = make_int4(0, 0, 0, 0);
            if (lane < nr) R = rng[lane];
            __syncwarp();
            int incl = R.w;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            const int total = __shfl_sync(0xffffffffu, incl, 31);
            const int excl = incl - R.w;
            // ---- stream the flattened entries, 32 per step
            for (int c0 = 0; c0 < total; c0 += 32) {
                const bool live = lane < nr;
                unsigned m = (live && excl > c0 && excl < c0 + 32) ? (1u << (excl - c0)) : 0u;
                m = __reduce_or_sync(0xffffffffu, m);
                const int rb = __popc(__ballot_sync(0xffffffffu, live && excl <= c0)) - 1;
                const int r = rb + __popc(m & lanemask_le);
                const int rbeg = __shfl_sync(0xffffffffu, R.x, r);
                const int rbase = __shfl_sync(0xffffffffu, R.y, r);
                const int rpk = __shfl_sync(0xffffffffu, R.z, r);
                const int rex = __shfl_sync(0xffffffffu, excl, r);
                const int e = c0 + lane;
                if (e < total) {
                    const int i = rbeg + (e - rex);
                    const uint32_t w = __ldg(tpos + i);
                    const float2 v = __ldg(tval + i);
                    const int u = (int)(w >> 16);
                    if (u >= ((rpk >> 8) & 255) && u < (rpk >> 16)) {
                        const int addr = ((int)(w & 0xffffu) << (rpk & 7)) + rbase;
                        float2 o = tile[addr];
                        o.x = fmaf(a, v.x, o.x);
                        o.y = fmaf(a, v.y, o.y);
                        tile[addr] = o;
                    }
                }
                __syncwarp();
            }
        }
    }
    __syncwarp();
    float2 *out = psi + (int64_t)(tile_y0 - A.row0) * A.n_h + tile_x0;
    for (int y = 0; y < T; y++)
        for (int x = lane; x < T; x += 32) out[(int64_t)y * A.n_h + x] = tile[y * S + x];
}

}  // namespace

cudaError_t launch_superpose_v1(const void *d_bins, const void *d_tables, int T, int S, int L, int tiles_x,
                                int tiles_y, int64_t row0, int64_t n_h, float2 *psi, cudaStream_t s) {
    const int smem = T * S * (int)sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(superpose_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    SupArgs A;
    A.T = T; A.S = S; A.L = L; A.tiles_x = tiles_x; A.row0 = row0; A.n_h = n_h;
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    if (n_tiles > 0) {
        count_launches(1);
        superpose_kernel<<<(unsigned)n_tiles, 32, smem, s>>>(d_bins, d_tables, A, psi);
    }
    return cudaGetLastError();
}

}  // namespace wasabi
