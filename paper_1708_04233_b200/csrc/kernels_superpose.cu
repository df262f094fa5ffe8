// kernels_superpose.cu -- step 2b of WASABI, Eq.(2):
//   psi(m, n) = sum_j a_j sum_k c_{z_j,k} delta(m - alpha x_j, n - alpha y_j)
// with alpha = 2^-l for a level-l coefficient (reading R-A8: target X = s_l(ix) + dX,
// s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l)), in the interleaved in-place Haar layout (R-A6).
//
// Design (DESIGN.md §5 K4).  One CTA = one warp owns one T x T tile of psi in shared memory and
// walks the tile's bin (points in ascending order).  For a point, the kept coefficients of level l
// whose targets fall in the tile are found through the LUT's per-level band index: the tile window
// is W x W blocks (W = T/2^l), covered by <= 5 bands, each one contiguous, X-exact entry range
// ("slot"; <= 32 slots per point).  Per batch of kPB points:
//   ranges   lane s computes slot s of each point (two independent points per step for ILP),
//            compacts the non-empty ranges and scans their counts -> 8-byte range records
//            (entry offset, smem base of the point's level) in shared memory;
//   stream   the warp streams the flattened entries 32 at a time (a chunk never mixes points, so
//            all targets of a chunk are distinct: no atomics, no races).  The current point's range
//            prefixes live in registers (lane r holds range r); lane -> range uses one REDUX.OR
//            marker + two POPCs; a kD-deep register ring prefetches the entry loads.
// LUT entries are 16-byte records (pos = X | Y << 14 | level << 28, re, im, Y*S + X - pos):
// target = pos + word3 + base (one IADD3; every word of the 128-bit load is used).
// Rows outside the tile (band rounding) are rejected by one unsigned compare of the smem address
// (X ranges are exact).  psi is written once, coalesced.  Per-pixel accumulation order is fixed
// (point order): bitwise deterministic and independent of the band split.
#include <cuda_runtime.h>
#include <cstdint>

#include "internal.h"
#include "device_common.cuh"

namespace wasabi {
namespace {

struct SupArgs {
    int T, S, L, tiles_x;
    int64_t row0, n_h;
};

constexpr int kPB = 8;                 // points per range batch
constexpr int kD = 4;                  // prefetch depth (chunks)
constexpr int kEmpty = 0x3fffffff;
constexpr int kBadBase = 0x3fffffff;   // base of padding lanes: address always >= T*S

__device__ __forceinline__ float2 lds2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts2(uint32_t a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

// level class c: c = 0 -> {1} U {4..L}, c = 1 -> {2, 3} (pixel-disjoint in the interleaved layout)
__device__ __forceinline__ bool in_class(int c, int l) { return c == 0 ? (l == 1 || l >= 4) : (l == 2 || l == 3); }

// Warp w owns (level class c = w & 1) x (tile row half h = w >> 1): pixel-disjoint, so the four
// warps of a CTA accumulate into the shared tile concurrently.  SEGW lanes per point: each range
// step handles 32/SEGW points.
template <int SEGW>
__global__ void __launch_bounds__(128, 6) superpose_kernel(const void *__restrict__ d_bins,
                                                           const void *__restrict__ d_tables, SupArgs A,
                                                           float2 *__restrict__ psi, int fused, QArgs qa,
                                                           uint8_t *__restrict__ bits) {
    constexpr int PPS = 32 / SEGW;            // points per range step
    constexpr int kH = kPB / PPS;             // range steps per batch
    extern __shared__ float2 tile[];          // T x S (+4 scratch)
    __shared__ int2 rec_all[4][kPB][SEGW];    // (entry offset = beg - excl, base | shift << 23)
    __shared__ int ex_all[4][kPB][SEGW];      // exclusive prefix (kEmpty past the last range)
    __shared__ int tot_all[4][kPB];
    __shared__ float a_all[4][kPB];
    const char *bb = reinterpret_cast<const char *>(d_bins);
    const BinHeader *bh = reinterpret_cast<const BinHeader *>(bb);
    const int4 *__restrict__ pconv = reinterpret_cast<const int4 *>(bb + bh->pts_off);
    const unsigned long long *__restrict__ bptr = reinterpret_cast<const unsigned long long *>(bb + bh->ptr_off);
    const uint32_t *__restrict__ bidx = reinterpret_cast<const uint32_t *>(bb + bh->idx_off);
    const char *tb = reinterpret_cast<const char *>(d_tables);
    const TableHeader *th = reinterpret_cast<const TableHeader *>(tb);
    const KDesc *__restrict__ kd = reinterpret_cast<const KDesc *>(tb + th->kdesc_off);
    const int32_t *__restrict__ tptr = reinterpret_cast<const int32_t *>(tb + th->ptr_off);
    const uint4 *__restrict__ tent = reinterpret_cast<const uint4 *>(tb + th->ent_off);

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cls = wid & 1, half = wid >> 1;
    const int T = A.T, S = A.S, TS = T * S, Th = T / 2;
    const int64_t t = blockIdx.x;
    const int tile_x0 = (int)(t % A.tiles_x) * T;
    const int tile_y0 = (int)(A.row0 + (t / A.tiles_x) * (int64_t)T);
    const int sub_y0 = tile_y0 + half * Th;          // this warp's rows [sub_y0, sub_y0 + Th)
    const int sub_lo = half * Th * S;                // its smem address range [sub_lo, sub_lo + Th*S)
    const unsigned lanemask_lt = (1u << lane) - 1u;
    const unsigned lanemask_le = lanemask_lt | (1u << lane);
    const uint32_t tile_sa = (uint32_t)__cvta_generic_to_shared(tile);
    const uint32_t dummy_sa = tile_sa + 8u * (uint32_t)(TS + wid);
    int2(*rec_s)[SEGW] = rec_all[wid];
    int(*ex_s)[SEGW] = ex_all[wid];
    int *tot_s = tot_all[wid];
    float *a_s = a_all[wid];

    for (int i = threadIdx.x; i < TS; i += 128) tile[i] = make_float2(0.f, 0.f);

    // lane = (segment seg: which point of a step, slot) -> (level, band slot k) of this class
    const int seg = lane / SEGW, slot = lane % SEGW;
    int my_l = 0, my_k = 0;
    {
        int base = 0;
        for (int l = 1; l <= A.L; l++) {
            if (!in_class(cls, l)) continue;
            const int hb = band_blocks(T, l);
            const int yb_lo = sub_y0 >> l, yb_hi = ((sub_y0 + Th - 1) >> l) + 1;
            const int Wy = yb_hi - yb_lo;
            const int m = (hb == 1) ? Wy : (Wy + hb - 1) / hb + 1;
            if (slot >= base && slot < base + m) { my_l = l; my_k = slot - base; }
            base += m;
        }
    }
    const bool has_slot = my_l > 0;
    const int l_ = has_slot ? my_l : 1;
    const int my_half = 1 << (l_ - 1);
    const int my_hb = band_blocks(T, l_);
    const int my_lhb = 31 - __clz(my_hb);
    const int my_Wx = T >> l_;
    const int my_tx = tile_x0 >> l_;
    const int my_ty = sub_y0 >> l_;
    const int my_Wy = (((sub_y0 + Th - 1) >> l_) + 1) - my_ty;
    const unsigned seg_bits = SEGW == 32 ? 0xffffffffu : ((1u << SEGW) - 1u);
    const unsigned seg_lt = ((1u << slot) - 1u) << (seg * SEGW);
    __syncthreads();

    const unsigned long long b0 = bptr[t], b1 = bptr[t + 1];
    unsigned long long pb = b0;      // next point of the bin to load
    int np = 0;                      // non-empty points in the current batch
    int4 q = make_int4(0, 0, 0, 0);

    auto load_batch = [&]() {
        np = 0;
        while (np == 0 && pb < b1) {
            const int nq = (int)min((unsigned long long)kPB, b1 - pb);
            q = make_int4(0, 0, 0, 0);
            if (lane < nq) q = __ldg(pconv + __ldg(bidx + pb + lane));
            pb += nq;
            int ix[kH], iy[kH], H[kH], pbs[kH];
#pragma unroll
            for (int h = 0; h < kH; h++) {
                const int k = PPS * h + seg;
                ix[h] = __shfl_sync(0xffffffffu, q.x, k);
                iy[h] = __shfl_sync(0xffffffffu, q.y, k);
                const int iz = __shfl_sync(0xffffffffu, q.z, k);
                H[h] = 0; pbs[h] = 0;
                if (k < nq && has_slot) { H[h] = __ldg(&kd[iz].H); pbs[h] = __ldg(&kd[iz].ptr_base[l_ - 1]); }
            }
            int beg[kH], end[kH], bse[kH];
#pragma unroll
            for (int h = 0; h < kH; h++) {
                const int k = PPS * h + seg;
                const int sx = (ix[h] + my_half) >> l_, sy = (iy[h] + my_half) >> l_;   // floor
                const int Hb = H[h] >> l_, nb = (2 * H[h]) >> l_;
                const int xb0 = my_tx - sx + Hb, yb0 = my_ty - sy + Hb;
                const int xb0c = max(xb0, 0), xb1c = min(xb0 + my_Wx, nb);
                const int yb0c = max(yb0, 0), yb1c = min(yb0 + my_Wy, nb);
                const int band = (yb0c >> my_lhb) + my_k;
                const bool ok = k < nq && has_slot && xb0c < xb1c && yb0c < yb1c && band * my_hb < yb1c;
                const int row = pbs[h] + band * (nb + 1);
                beg[h] = 0; end[h] = 0;
                if (ok) { beg[h] = __ldg(tptr + row + xb0c); end[h] = __ldg(tptr + row + xb1c); }
                bse[h] = ((sy << l_) - H[h] - tile_y0) * S + ((sx << l_) - H[h] - tile_x0);
            }
#pragma unroll
            for (int h = 0; h < kH; h++) {
                const int c = end[h] - beg[h];
                const unsigned bal = __ballot_sync(0xffffffffu, c > 0);
                if (bal == 0u) continue;
                int incl = c;
#pragma unroll
                for (int o = 1; o < SEGW; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, incl, o, SEGW);
                    if (slot >= o) incl += y;
                }
                const int excl = incl - c;
                // compacted index of my segment's point among the non-empty points of this step
                const unsigned nonempty_segs = [&] {
                    unsigned m = 0;
#pragma unroll
                    for (int g = 0; g < PPS; g++) m |= ((bal >> (g * SEGW)) & seg_bits) ? (1u << g) : 0u;
                    return m;
                }();
                const unsigned mine = (bal >> (seg * SEGW)) & seg_bits;
                const int idx = np + __popc(nonempty_segs & ((1u << seg) - 1u));
                if (mine) {
                    if (c > 0) {
                        const int p = __popc(bal & seg_lt);
                        rec_s[idx][p] = make_int2(beg[h] - excl, bse[h]);
                        ex_s[idx][p] = excl;
                    }
                    if (slot >= __popc(mine)) ex_s[idx][slot] = kEmpty;
                    if (slot == SEGW - 1) tot_s[idx] = incl;
                }
                const float aw = __int_as_float(__shfl_sync(0xffffffffu, q.w, PPS * h + seg));
                if (mine && slot == 0) a_s[idx] = aw;
                np += __popc(nonempty_segs);
            }
        }
        __syncwarp();
    };

    // prefetch cursor (warp-uniform except exv)
    int kp = 0, cp = 0, totp = 0, exv = kEmpty;
    float ap = 0.f;
    load_batch();
    if (np > 0) { totp = tot_s[0]; exv = lane < SEGW ? ex_s[0][lane] : kEmpty; ap = a_s[0]; }
    bool done = np == 0;

    uint32_t rw[kD], rz[kD];
    float rx[kD], ry[kD], ra[kD];
    int rb[kD];
#pragma unroll
    for (int s = 0; s < kD; s++) { rw[s] = 0; rz[s] = 0; rx[s] = 0.f; ry[s] = 0.f; ra[s] = 0.f; }
#define WASABI_PREFETCH(s)                                                                  \
    do {                                                                                    \
        rb[s] = kBadBase;                                                                   \
        if (kp < np) {                                                                      \
            unsigned m = ((unsigned)(exv - cp - 1) < 31u) ? (1u << (exv - cp)) : 0u;        \
            m = __reduce_or_sync(0xffffffffu, m);                                           \
            const int rr = __popc(__ballot_sync(0xffffffffu, exv <= cp)) - 1 +              \
                           __popc(m & lanemask_le);                                         \
            const int e = cp + lane;                                                        \
            const int2 d = rec_s[kp][rr & (SEGW - 1)];                                      \
            if (e < totp) {                                                                 \
                const uint4 en = __ldg(tent + e + d.x);                                     \
                rw[s] = en.x; rx[s] = __uint_as_float(en.y); ry[s] = __uint_as_float(en.z); rz[s] = en.w; \
                rb[s] = d.y; ra[s] = ap;                                                    \
            }                                                                               \
            cp += 32;                                                                       \
            if (cp >= totp) {                                                               \
                cp = 0;                                                                     \
                if (++kp < np) {                                                            \
                    totp = tot_s[kp]; exv = lane < SEGW ? ex_s[kp][lane] : kEmpty; ap = a_s[kp]; \
                }                                                                           \
            }                                                                               \
        }                                                                                   \
    } while (0)
#define WASABI_CONSUME(s)                                                                   \
    do {                                                                                    \
        const int addr = (int)(rw[s] + rz[s]) + rb[s];                                       \
        const uint32_t sa = (unsigned)(addr - sub_lo) < (unsigned)(Th * S)                  \
                                ? tile_sa + 8u * (uint32_t)addr : dummy_sa;                 \
        float2 o = lds2(sa);                                                                \
        o.x = fmaf(ra[s], rx[s], o.x);                                                      \
        o.y = fmaf(ra[s], ry[s], o.y);                                                      \
        sts2(sa, o);                                                                        \
    } while (0)
#pragma unroll
    for (int s = 0; s < kD; s++) WASABI_PREFETCH(s);
    while (true) {
#pragma unroll
        for (int s = 0; s < kD; s++) {
            WASABI_CONSUME(s);
            WASABI_PREFETCH(s);
        }
        if (done) break;
        if (kp >= np) {
            load_batch();
            kp = 0; cp = 0;
            if (np > 0) { totp = tot_s[0]; exv = lane < SEGW ? ex_s[0][lane] : kEmpty; ap = a_s[0]; }
            else done = true;     // one more round drains the ring
        }
    }
#undef WASABI_PREFETCH
#undef WASABI_CONSUME
    __syncthreads();
    if (fused) {
        // steps 3 (+4) in place: psi never leaves shared memory
        inverse_haar_tile(tile, T, S, A.L, threadIdx.x, 128);
        if (bits) {
            const int bpr = T / 8;
            for (int bi = threadIdx.x; bi < T * bpr; bi += 128) {
                const int row = bi / bpr, xb = bi % bpr;
                const int64_t Y = tile_y0 + row;
                unsigned byte = 0;
#pragma unroll
                for (int i = 0; i < 8; i++) {
                    const int x = xb * 8 + i;
                    const float I = interference(tile[row * S + x], tile_x0 + x, Y, qa);
                    byte |= (I >= 0.0f ? 1u : 0u) << (7 - i);
                }
                bits[(Y - A.row0) * (A.n_h / 8) + tile_x0 / 8 + xb] = (uint8_t)byte;
            }
        }
        if (!psi) return;
    }
    float2 *out = psi + (int64_t)(tile_y0 - A.row0) * A.n_h + tile_x0;
    for (int y = wid; y < T; y += 4)
        for (int x = lane; x < T; x += 32) out[(int64_t)y * A.n_h + x] = tile[y * S + x];
}

}  // namespace

cudaError_t launch_superpose(const void *d_bins, const void *d_tables, int T, int S, int L, int tiles_x, int tiles_y,
                             int64_t row0, int64_t n_h, float2 *psi, int fused, const double *print4, double pitch,
                             uint8_t *bits, cudaStream_t s) {
    const int smem = (T * S + 4) * (int)sizeof(float2);
    // range slots per (class, row half) and point: <= 8 for T = 64, <= 16 for T = 128
    auto kern = T <= 64 ? superpose_kernel<8> : superpose_kernel<16>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    SupArgs A;
    A.T = T; A.S = S; A.L = L; A.tiles_x = tiles_x; A.row0 = row0; A.n_h = n_h;
    const int64_t n_tiles = (int64_t)tiles_x * tiles_y;
    if (n_tiles > 0) {
        count_launches(1);
        kern<<<(unsigned)n_tiles, 128, smem, s>>>(d_bins, d_tables, A, psi, fused,
                                                  make_qargs(print4, pitch, n_h), bits);
    }
    return cudaGetLastError();
}

}  // namespace wasabi
