// kernels_superpose.cu -- step 2b of WASABI, Eq.(2):
//   psi(m, n) = sum_j a_j sum_k c_{z_j,k} delta(m - alpha x_j, n - alpha y_j)
// with alpha = 2^-l for a level-l coefficient (reading R-A8: target X = s_l(ix) + dX,
// s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l)), in the interleaved in-place Haar layout (R-A6).
//
// Design (DESIGN.md §5 K4).  One CTA owns one T x T tile of psi in shared memory and walks the
// tile's bin (points in ascending order).  Its two warps own pixel-disjoint level classes of the
// interleaved layout (warp 0: levels {1} U {4..L}; warp 1: levels {2, 3}; each position belongs
// to exactly one level), so they accumulate concurrently without atomics or barriers.  For a
// point, the kept coefficients of a level whose targets fall in the tile are found through the
// LUT's per-level band index: the tile window is W x W blocks (W = T/2^l), covered by <= 5 bands,
// each one contiguous, X-exact entry range ("slot").  Per batch of kB points a warp
//   phase A  computes the slots of two points per step (16-lane segments), compacts the non-empty
//            ranges and scans their counts -> per-point range records in shared memory;
//   phase C  streams the flattened entries 32 at a time (a chunk never mixes points, so all targets
//            of a chunk are distinct), with a kD-deep register ring prefetching the entry loads.
// psi is written once, coalesced.  Per-pixel accumulation order is fixed (point order): bitwise
// deterministic and independent of the band split.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"

namespace wasabi {
namespace {

struct SupArgs {
    int T, S, L, tiles_x;
    int64_t row0, n_h;
};

constexpr int kB = 16;      // points per batch
constexpr int kD = 8;       // prefetch depth (chunks)
constexpr int kSeg = 16;    // range slots per point and class
constexpr int kEmpty = 0x3fffffff;

// level class of warp w: w = 0 -> {1} U {4..L}, w = 1 -> {2, 3}
__device__ __forceinline__ bool in_class(int w, int l) { return w == 0 ? (l == 1 || l >= 4) : (l == 2 || l == 3); }

__global__ void __launch_bounds__(64) superpose_kernel(const void *__restrict__ d_bins,
                                                       const void *__restrict__ d_tables, SupArgs A,
                                                       float2 *__restrict__ psi) {
    extern __shared__ float2 tile[];            // T x S
    __shared__ int4 rec_s[2][kB][kSeg];         // (eoff, base, packed, -)
    __shared__ int ex_s[2][kB][kSeg];           // exclusive prefix of the compacted ranges
    __shared__ int tot_s[2][kB];
    __shared__ float a_s[2][kB];
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

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int T = A.T, S = A.S;
    const int64_t t = blockIdx.x;
    const int tile_x0 = (int)(t % A.tiles_x) * T;
    const int tile_y0 = (int)(A.row0 + (t / A.tiles_x) * (int64_t)T);

    for (int i = threadIdx.x; i < T * S; i += 64) tile[i] = make_float2(0.f, 0.f);

    // this lane's range slot: segment seg (point parity), slot -> (level, band k) within the class
    const int seg = lane >> 4, slot = lane & 15;
    int my_l = 0, my_k = 0;
    {
        int base = 0;
        for (int l = 1; l <= A.L; l++) {
            if (!in_class(wid, l)) continue;
            const int W = T >> l, hb = band_blocks(T, l);
            const int m = (hb == 1) ? W : W / hb + 1;
            if (slot >= base && slot < base + m) { my_l = l; my_k = slot - base; }
            base += m;
        }
    }
    const int my_half = my_l > 0 ? 1 << (my_l - 1) : 0;
    const int my_hb = my_l > 0 ? band_blocks(T, my_l) : 1;
    const int my_W = my_l > 0 ? T >> my_l : 0;
    const int my_tx = my_l > 0 ? tile_x0 >> my_l : 0;
    const int my_ty = my_l > 0 ? tile_y0 >> my_l : 0;
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const unsigned lanemask_le = lanemask_lt | (1u << lane);
    const unsigned segmask_lt = ((1u << slot) - 1u) << (seg * 16);
    int4(*rec)[kSeg] = rec_s[wid];
    int(*exs)[kSeg] = ex_s[wid];
    int *tots = tot_s[wid];
    float *as = a_s[wid];
    __syncthreads();

    const unsigned long long b0 = bptr[t], b1 = bptr[t + 1];
    for (unsigned long long pb = b0; pb < b1; pb += kB) {
        const int np = (int)min((unsigned long long)kB, b1 - pb);
        int4 q = make_int4(0, 0, 0, 0);
        if (lane < np) q = __ldg(pconv + __ldg(bidx + pb + lane));
        // ------------------------------------------------ phase A: two points per step
        for (int k0 = 0; k0 < np; k0 += 2) {
            const int k = k0 + seg;
            const int ix = __shfl_sync(0xffffffffu, q.x, k & 31);
            const int iy = __shfl_sync(0xffffffffu, q.y, k & 31);
            const int iz = __shfl_sync(0xffffffffu, q.z, k & 31);
            const int aw = __shfl_sync(0xffffffffu, q.w, k & 31);
            int beg = 0, cnt = 0, base = 0, packed = 0;
            if (my_l > 0 && k < np) {
                const int l = my_l;
                const int H = __ldg(&kd[iz].H);
                const int pbase = __ldg(&kd[iz].ptr_base[l - 1]);
                const int sx = (ix + my_half) >> l, sy = (iy + my_half) >> l;  // floor
                const int Hb = H >> l, nb = (2 * H) >> l;
                const int xb0 = my_tx - sx + Hb, yb0 = my_ty - sy + Hb;
                const int xb0c = max(xb0, 0), xb1c = min(xb0 + my_W, nb);
                const int yb0c = max(yb0, 0), yb1c = min(yb0 + my_W, nb);
                const int band = yb0c / my_hb + my_k;
                if (xb0c < xb1c && yb0c < yb1c && band * my_hb < yb1c) {
                    const int row = pbase + band * (nb + 1);
                    beg = __ldg(tptr + row + xb0c);
                    cnt = __ldg(tptr + row + xb1c) - beg;
                    const int ulo = max(0, 2 * (yb0c - band * my_hb));
                    const int uhi = min(2 * my_hb, 2 * (yb1c - band * my_hb));
                    base = (((band * my_hb) << l) - H + (sy << l) - tile_y0) * S + ((sx << l) - H - tile_x0);
                    packed = (l - 1) | (ulo << 8) | (uhi << 16);
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, cnt > 0);
            int incl = cnt;
#pragma unroll
            for (int o = 1; o < 16; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, incl, o, 16);
                if (slot >= o) incl += y;
            }
            const int excl = incl - cnt;
            const int nr = __popc((bal >> (seg * 16)) & 0xffffu);
            if (k < np) {
                if (cnt > 0) {
                    const int p = __popc(bal & segmask_lt);
                    rec[k][p] = make_int4(beg - excl, base, packed, 0);
                    exs[k][p] = excl;
                }
                if (slot >= nr) exs[k][slot] = kEmpty;
                if (slot == 15) { tots[k] = incl; as[k] = __int_as_float(aw); }
            }
        }
        __syncwarp();
        // ------------------------------------------------ phase C: chunk stream with prefetch
        int kp = 0, cp = 0;                 // prefetch cursor: point, chunk start
        int totp = tots[0];
        float ap = as[0];
        while (totp == 0 && ++kp < np) { totp = tots[kp]; ap = as[kp]; }
        uint32_t rw[kD];
        float rx[kD], ry[kD], ra[kD];
        int rb[kD], rp[kD];
        // prefetch the chunk at the (warp-uniform) cursor into ring slot s
#define WASABI_PREFETCH(s)                                                                  \
        do {                                                                                \
            rp[s] = -1;                                                                     \
            if (kp < np) {                                                                  \
                const int exv = lane < 16 ? exs[kp][lane] : kEmpty;                         \
                unsigned m = ((unsigned)(exv - cp - 1) < 31u) ? (1u << (exv - cp)) : 0u;    \
                m = __reduce_or_sync(0xffffffffu, m);                                       \
                const int rr = __popc(__ballot_sync(0xffffffffu, exv <= cp)) - 1 +          \
                               __popc(m & lanemask_le);                                     \
                const int e = cp + lane;                                                    \
                if (e < totp) {                                                             \
                    const int4 R = rec[kp][rr & 15];                                        \
                    const int i = e + R.x;                                                  \
                    rw[s] = __ldg(tpos + i);                                                \
                    const float2 v = __ldg(tval + i);                                       \
                    rx[s] = v.x; ry[s] = v.y; ra[s] = ap;                                   \
                    rb[s] = R.y; rp[s] = R.z;                                               \
                }                                                                           \
                cp += 32;                                                                   \
                if (cp >= totp) {                                                           \
                    cp = 0;                                                                 \
                    while (++kp < np) {                                                     \
                        totp = tots[kp];                                                    \
                        ap = as[kp];                                                        \
                        if (totp > 0) break;                                                \
                    }                                                                       \
                }                                                                           \
            }                                                                               \
        } while (0)
        // accumulate ring slot s into the tile (all targets of one chunk are distinct)
#define WASABI_CONSUME(s)                                                                   \
        do {                                                                                \
            if (rp[s] >= 0) {                                                               \
                const int u = (int)(rw[s] >> 16);                                           \
                if (u >= ((rp[s] >> 8) & 255) && u < (rp[s] >> 16)) {                      \
                    const int addr = ((int)(rw[s] & 0xffffu) << (rp[s] & 7)) + rb[s];       \
                    float2 o = tile[addr];                                                  \
                    o.x = fmaf(ra[s], rx[s], o.x);                                          \
                    o.y = fmaf(ra[s], ry[s], o.y);                                          \
                    tile[addr] = o;                                                         \
                }                                                                           \
            }                                                                               \
            __syncwarp();                                                                   \
        } while (0)
#pragma unroll
        for (int s = 0; s < kD; s++) WASABI_PREFETCH(s);
        while (true) {
            const bool exhausted = kp >= np;   // warp-uniform
#pragma unroll
            for (int s = 0; s < kD; s++) {
                WASABI_CONSUME(s);
                WASABI_PREFETCH(s);
            }
            if (exhausted) break;
        }
#undef WASABI_PREFETCH
#undef WASABI_CONSUME
        __syncwarp();
    }
    __syncthreads();
    float2 *out = psi + (int64_t)(tile_y0 - A.row0) * A.n_h + tile_x0;
    for (int y = wid; y < T; y += 2)
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
        superpose_kernel<<<(unsigned)n_tiles, 64, smem, s>>>(d_bins, d_tables, A, psi);
    }
    return cudaGetLastError();
}

}  // namespace wasabi
