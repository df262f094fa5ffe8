// kernels_superpose.cu -- step 2b of WASABI, Eq.(2):
//   psi(m, n) = sum_j a_j sum_k c_{z_j,k} delta(m - alpha x_j, n - alpha y_j)
// with alpha = 2^-l for a level-l coefficient (reading R-A8: target X = s_l(ix) + dX,
// s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l)), in the interleaved in-place Haar layout (R-A6).
//
// Design (DESIGN.md §6 "Superpose").  One CTA owns one T x T tile of psi in shared memory and
// walks the tile's bin (points in ascending order).  Warp w owns the pixels of level class
// c = w & 1 ({1, 3, 6} or {2, 4, 5}; {1} or {2, 3} for L <= 3; every level has its own pixels) in the 32-row strip
// w >> 1, so the warps of a CTA accumulate concurrently without atomics.  For a point and a level
// of its class, the kept coefficients landing in the strip are ONE contiguous range of the window
// LUT (internal.h: per-variant 32-row bands, column-group pointers), so a batch of 32 points
// (lane = point) computes all its ranges with two pointer loads per (point, level), and the warp
// then streams each range 32 entries per chunk: lane i of chunk c reads entry beg + 32 c + i
// (float2 value + uint16 position) and does one read-modify-write in shared memory.  A chunk never
// mixes points, so its targets are distinct; chunks run in point order for each level, so every
// pixel (which belongs to exactly one level) accumulates in point order: bitwise deterministic
// and independent of the band split (R-A11).  A kD-deep register ring keeps the loads of the next
// chunks in flight across range and level boundaries of a batch (idle lanes address the warp's
// dummy cell).  Column overrun of the level-1/2 column groups lands in kWinMargin
// margin columns of the shared tile (never read).  Shared accesses go through an XOR bank swizzle
// (swz below), tiles run in groups of 28 tile rows (L2 reuse of the window LUT), and the next
// batch's point records are prefetched during the ring.  The kernel sits between the L1TEX/LSU data
// pipe (~80%: scattered 8-byte shared-memory read-modify-writes, LUT and pointer loads, shuffles)
// and instruction issue / load latency.
#include <cuda_runtime.h>
#include <cstdint>
#include <type_traits>

#include "internal.h"
#include "device_common.cuh"

namespace wasabi {
namespace {

struct SupArgs {
    int L, cls_bits, tiles_x;
    int64_t row0, n_h;
    int64_t tile0;   // first tile (row-major in the bins' band) of this launch
    int tile_rows;   // tile rows of this launch
};

#ifndef WASABI_KD
#define WASABI_KD 6
#endif
#ifndef WASABI_MINB
#define WASABI_MINB 5
#endif
#ifndef WASABI_PF
#define WASABI_PF 0   // bulk L2 prefetch of each batch's ranges: measured slower with the ring at full C4
#endif

constexpr int kD = WASABI_KD;          // register ring depth (chunks in flight per warp)

#ifndef WASABI_GROUP
#define WASABI_GROUP 28
#endif
// Tile order: groups of kGroup tile rows, column-major inside a group, so that the CTAs resident
// at one time cover a compact, about square 2-D region (28 x ~26 tiles at 740 resident CTAs) instead of a
// full-width tile row: its points span fewer depth tables, and more of the window-LUT reads hit
// L2 (0 = row-major).
constexpr int kGroup = WASABI_GROUP;

#ifndef WASABI_L1NA
#define WASABI_L1NA 0
#endif
// Window-LUT loads: read once per use (14% L1 hit rate), so optionally not allocated in L1.
__device__ __forceinline__ float2 ldg_stream(const float2 *p) {
#if WASABI_L1NA
    float2 v;
    asm volatile("ld.global.nc.L1::no_allocate.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}
__device__ __forceinline__ int ldg_stream(const uint16_t *p) {
#if WASABI_L1NA
    unsigned short v;
    asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(p));
    return v;
#else
    return __ldg(p);
#endif
}

// Bulk prefetch of [p, p + bytes) into L2 (16-byte granules): one instruction per range, so the
// later chunks of a range hit L2 instead of waiting on DRAM.
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
constexpr unsigned kFull = 0xffffffffu;
// Opaque copies for the ring slots' per-chunk base and amplitude: without them the compiler sees that
// most slots hold the same c_sa / c_a and keeps a rotating queue of copies (7-8 MOVs per ring slot,
// 29 -> 23 SASS instructions per slot; fused C4 75.4 -> 73.8 ms, psi identical).
__device__ __forceinline__ uint32_t opq(uint32_t x) { uint32_t y; asm volatile("mov.b32 %0, %1;" : "=r"(y) : "r"(x)); return y; }
__device__ __forceinline__ float opqf(float x) { float y; asm volatile("mov.b32 %0, %1;" : "=f"(y) : "f"(x)); return y; }

#ifndef WASABI_SWZ
#define WASABI_SWZ 1
#endif
// Shared-tile bank swizzle.  A level-l coefficient sits at a pixel whose X and Y are multiples of
// 2^(l-1) (R-A6), so in a linear tile the cells of a level-2 chunk fall on even bank pairs and
// those of a level-3 chunk on a quarter of them: ~6.2 wavefronts per 32-lane LDS.64 against an
// ideal 2 (ncu, v19; tools/bank_model.py reproduces it).  The byte address a of a cell is replaced
// by a ^ ((a >> 5) & 0x38): address bits 3..5 (the cell inside its 64-byte block) XOR address
// bits 8..10, a permutation inside each aligned 8-cell block.  With rows of stride S = T + 8 cells
// starting on 64-byte boundaries (tile base 64-byte aligned), margin blocks stay margin blocks; the
// model predicts ~3.5 wavefronts per chunk.
__device__ __forceinline__ uint32_t swz(uint32_t a) {
#if WASABI_SWZ
#ifndef WASABI_SWZ_SHIFT
#define WASABI_SWZ_SHIFT 5
#endif
    return a ^ ((a >> WASABI_SWZ_SHIFT) & 0x38u);
#else
    return a;
#endif
}

__device__ __forceinline__ float4 lds4(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts4(uint32_t a, float4 v) {
    asm volatile("st.shared.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w) : "memory");
}
__device__ __forceinline__ float2 lds2(uint32_t a) {
    float2 v;
    asm volatile("ld.shared.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void sts2(uint32_t a, float2 v) {
    asm volatile("st.shared.v2.f32 [%0], {%1, %2};" ::"r"(a), "f"(v.x), "f"(v.y) : "memory");
}

#ifndef WASABI_DEBUG_BOUNDS
#define WASABI_DEBUG_BOUNDS 0   // 1: trap on a shared access outside the tile or a LUT index outside the arrays
#endif
#ifndef WASABI_BULKZERO
#define WASABI_BULKZERO 1
#endif
#if WASABI_BULKZERO
__device__ float4 g_zero[128 * (128 + kWinMargin + 2) / 2 + 16];   // zeros (static storage) for the tile fill
#endif
#ifndef WASABI_L1Q
#define WASABI_L1Q 1
#endif
#ifndef WASABI_STCS
#define WASABI_STCS 1
#endif
// levels of class c, slot j: superpose_class_level (internal.h), c = 0 -> {1, 3, 6}, c = 1 -> {2, 4, 5} (L <= 3: {1} / {2, 3});
// the table descriptor carries, per class, H and the window-pointer rows of those levels (KDesc.cls4)

// Steps 3 (+4) of a T x T psi tile held in shared memory (swizzled cells, swz), shared by the scatter
// and gather superposition kernels: fused -> the R-A6 inverse butterflies level by level in place, the
// print bits (print_byte) and u (psi pointer, may be NULL); unfused -> psi written as is.
template <int T, int NT>
__device__ __forceinline__ void tile_epilogue(float2 *tile, uint32_t tile_sa, int L, int fused, const QArgs &qa,
                                              uint8_t *__restrict__ bits, float2 *__restrict__ psi, int64_t row0,
                                              int64_t n_h, int tile_x0, int tile_y0) {
    constexpr int M = kWinMargin, S = T + M;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    auto cell = [&](int r, int x) -> float2 & {
        return tile[(swz(tile_sa + 8u * (uint32_t)(M + r * S + x)) - tile_sa) >> 3];
    };
    if (fused) {
        // steps 3 (+4) in place: psi never leaves shared memory; the
        // R-A6 butterflies level by level from L (inv_butterfly, device_common.cuh), swizzled cells
        for (int l = L; l >= 1; l--) {
            const int st = 1 << (l - 1), nq = T >> l;
#if WASABI_L1Q
            if (l == 1) {   // a level-1 quad's rows are aligned 16-byte cell pairs (swapped for odd keys)
                for (int qd = threadIdx.x; qd < nq * nq; qd += NT) {
                    const int bx = (qd % nq) << 1, by = (qd / nq) << 1;
                    const uint32_t a0 = swz(tile_sa + 8u * (uint32_t)(M + by * S + bx));
                    const uint32_t a1 = swz(tile_sa + 8u * (uint32_t)(M + (by + 1) * S + bx));
                    const float4 w0 = lds4(a0 & ~15u), w1 = lds4(a1 & ~15u);
                    float2 q[4];
                    q[0] = (a0 & 8u) ? make_float2(w0.z, w0.w) : make_float2(w0.x, w0.y);
                    q[1] = (a0 & 8u) ? make_float2(w0.x, w0.y) : make_float2(w0.z, w0.w);
                    q[2] = (a1 & 8u) ? make_float2(w1.z, w1.w) : make_float2(w1.x, w1.y);
                    q[3] = (a1 & 8u) ? make_float2(w1.x, w1.y) : make_float2(w1.z, w1.w);
                    inv_butterfly(&q[0], &q[1], &q[2], &q[3]);
                    sts4(a0 & ~15u, (a0 & 8u) ? make_float4(q[1].x, q[1].y, q[0].x, q[0].y)
                                              : make_float4(q[0].x, q[0].y, q[1].x, q[1].y));
                    sts4(a1 & ~15u, (a1 & 8u) ? make_float4(q[3].x, q[3].y, q[2].x, q[2].y)
                                              : make_float4(q[2].x, q[2].y, q[3].x, q[3].y));
                }
                __syncthreads();
                continue;
            }
#endif
            for (int qd = threadIdx.x; qd < nq * nq; qd += NT) {
                const int bx = (qd % nq) << l, by = (qd / nq) << l;
                inv_butterfly(&cell(by, bx), &cell(by, bx + st), &cell(by + st, bx), &cell(by + st, bx + st));
            }
            __syncthreads();
        }
        if (bits) {
            constexpr int bpr = T / 8;
            auto bytes = [&](auto series) {   // the series test hoisted out of the byte loop
                for (int bi = threadIdx.x; bi < T * bpr; bi += NT) {
                    const int row = bi / bpr, xb = bi % bpr;
                    const int64_t Y = tile_y0 + row;
                    float2 v[8];
#pragma unroll
                    for (int i = 0; i < 8; i++) v[i] = cell(row, xb * 8 + i);
                    const unsigned byte = print_byte_t<decltype(series)::value>(v, tile_x0 + xb * 8, ref_row(Y, qa), qa);
                    bits[(Y - row0) * (n_h / 8) + tile_x0 / 8 + xb] = (uint8_t)byte;
                }
            };
            if (qa.series) bytes(std::true_type{}); else bytes(std::false_type{});
        }
        if (!psi) return;
    }
    float2 *out = psi + (int64_t)(tile_y0 - row0) * n_h + tile_x0;
#pragma unroll 4
    for (int y = wid; y < T; y += NT / 32) {
        float2 v[T / 32];                     // loads of a row first, then its coalesced stores
#pragma unroll
        for (int i = 0; i < T / 32; i++) v[i] = cell(y, lane + 32 * i);
#pragma unroll
        for (int i = 0; i < T / 32; i++) {
#if WASABI_STCS   // write-once output: evict-first in L2, so it does not displace the window LUT
            __stcs(out + (int64_t)y * n_h + lane + 32 * i, v[i]);
#else
            out[(int64_t)y * n_h + lane + 32 * i] = v[i];
#endif
        }
    }
}

template <int T, bool EX>
__global__ void __launch_bounds__(2 * T, T == 64 ? WASABI_MINB : 1) superpose_kernel(const void *__restrict__ d_bins,
                                                                           const void *__restrict__ d_tables,
                                                                           SupArgs A, float2 *__restrict__ psi,
                                                                           int fused, QArgs qa,
                                                                           uint8_t *__restrict__ bits) {
    constexpr int M = kWinMargin, S = T + M, NT = 2 * T;
    constexpr int kData = M + T * S + M;      // margin-padded tile; a block of per-warp dummy cells follows
    static_assert(S % 8 == 0 && M % 8 == 0 && NT / 32 <= 8, "swizzle blocks");
    extern __shared__ float2 tile[];
    const char *bb = reinterpret_cast<const char *>(d_bins);
    const BinHeader *bh = reinterpret_cast<const BinHeader *>(bb);
    const int4 *__restrict__ pconv = reinterpret_cast<const int4 *>(bb + bh->pts_off);
    const unsigned long long *__restrict__ bptr = reinterpret_cast<const unsigned long long *>(bb + bh->ptr_off);
    const uint32_t *__restrict__ bidx = reinterpret_cast<const uint32_t *>(bb + bh->idx_off);
    const char *tb = reinterpret_cast<const char *>(d_tables);
    const TableHeader *th = reinterpret_cast<const TableHeader *>(tb);
    const KDesc *__restrict__ kd = reinterpret_cast<const KDesc *>(tb + th->kdesc_off);
    const int32_t *__restrict__ vptr = reinterpret_cast<const int32_t *>(tb + th->vptr_off);
    const float2 *__restrict__ vval = reinterpret_cast<const float2 *>(tb + th->vval_off);
    const uint16_t *__restrict__ vpos = reinterpret_cast<const uint16_t *>(tb + th->vpos_off);

    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int cls = wid & 1, strip = wid >> 1;
    int64_t t;
    if (kGroup > 0) {
        const int64_t per_group = (int64_t)kGroup * A.tiles_x;
        const int64_t g = blockIdx.x / per_group, rem = blockIdx.x - g * per_group;
        const int gh = (int)min((int64_t)kGroup, A.tile_rows - g * kGroup);
        t = A.tile0 + (g * kGroup + rem % gh) * A.tiles_x + rem / gh;
    } else {
        t = A.tile0 + blockIdx.x;
    }
    const int tile_x0 = (int)(t % A.tiles_x) * T;
    const int tile_y0 = (int)(A.row0 + (t / A.tiles_x) * (int64_t)T);
    const int strip_y0 = tile_y0 + kWinRows * strip;
    const int strip_base = M + kWinRows * strip * S;   // smem index of (strip row 0, column 0)
    const int dummy = kData + wid;
    const uint32_t tile_sa = (uint32_t)__cvta_generic_to_shared(tile);
    if (tile_sa & 63u) __trap();              // the swizzle permutes 64-byte blocks of the tile
    // pixel (r, x) of the tile: cell M + r S + x, swizzled
    auto cell = [&](int r, int x) -> float2 & {
        return tile[(swz(tile_sa + 8u * (uint32_t)(M + r * S + x)) - tile_sa) >> 3];
    };

    // the tile's bin pointers first: their load chain (bin -> point -> descriptor -> window pointers ->
    // first chunks) overlaps the zero fill, whose completion is awaited only before the first
    // shared-memory access of the ring
    const unsigned long long b1 = bptr[t + 1];
    unsigned long long pb = bptr[t];
#if WASABI_BULKZERO
    // zero the tile + dummy block by one bulk async copy from a zero buffer (the copy engine, not the
    // LSU); the mbarrier sits after the dummy block
    {
        const uint32_t mbar = tile_sa + 8u * (uint32_t)(kData + 8);
        constexpr uint32_t zbytes = 8u * (uint32_t)(kData + 8);
        static_assert(zbytes % 16 == 0 && zbytes <= sizeof(g_zero), "bulk zero fill");
        if (threadIdx.x == 0) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mbar) : "memory");
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(zbytes) : "memory");
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(tile_sa), "l"(g_zero), "r"(zbytes), "r"(mbar) : "memory");
        }
        __syncthreads();   // the mbarrier is initialised; the wait is deferred to just before the ring
    }
#else
    for (int i = threadIdx.x; i < kData + 8; i += NT) tile[i] = make_float2(0.f, 0.f);
    __syncthreads();
#endif

    const int lv0 = superpose_class_level(cls, 0, A.L), lv1 = superpose_class_level(cls, 1, A.L);
    const int lv2 = superpose_class_level(cls, 2, A.L);

    // batch state: lane = point; per level slot j its range: first entry beg and pk = (smem base << 16)
    // | length; the CURRENT batch (beg, pk, a_l) and the NEXT one (nbeg, npk, na), loaded while the
    // current batch's chunks stream (software-pipelined batches, WASABI_PIPE)
    float a_l = 0.f, na = 0.f;
    constexpr int kSlots = 3;                         // level slots per warp
    int beg[3] = {0, 0, 0}, pk[3] = {0, 0, 0}, nbeg[3] = {0, 0, 0}, npk[3] = {0, 0, 0};
    const int cb = EX ? A.L : 0;               // offset-class bits (R-A20) or 0
    const int cmask = (1 << cb) - 1;
    auto range = [&](int l, int ix, int iy, int H, int side, int vrow, bool ok, int &b, int &p) {
        b = 0; p = 0;
        if (l == 0) return;
        const int h = 1 << (l - 1);
        // R-A8 level shift, or the 2^L-aligned shift of the offset-class tables (R-A20)
        const int sx = EX ? ix & ~cmask : ((ix + h) >> l) << l;
        const int sy = EX ? iy & ~cmask : ((iy + h) >> l) << l;
        const int o = strip_y0 - sy + H;                 // window rows [o, o + 32)
        const int xs = tile_x0 - sx + H;                 // window columns [xs, xs + T)
        ok = ok && o > -kWinRows && o < side && xs > -T && xs < side;
        const int lq = win_lq(l, cb), lg = win_lg(l);
        const int v = (o & (kWinRows - 1)) >> lq;
        const int k = (o - (v << lq) + kWinRows) >> 5;
        const int ncol = win_cols(side, l);
        const int xa = max(xs >> lg, 0), xb = min((xs + T + (1 << lg) - 1) >> lg, ncol);
        int n = 0;
        if (ok && xa < xb) {
            const int row = vrow + (v * win_bands(side) + k) * (ncol + 1);
            b = __ldg(vptr + row + xa);
            n = __ldg(vptr + row + xb) - b;
        }
        p = (int)(((uint32_t)(strip_base - xs) << 16) | (uint32_t)n);   // |base| < 2^15, length < 2^16
    };
    // the point records of the next batch are loaded one batch ahead and its bin indices two
    // batches ahead (the loads overlap the ring): two dependent round trips off the batch phase
    // (batches are 32 points but the last)
    uint32_t nidx = pb + 32 + lane < b1 ? __ldg(bidx + pb + 32 + lane) : 0u;
    int4 qn = pb + lane < b1 ? __ldg(pconv + __ldg(bidx + pb + lane)) : make_int4(0, 0, 0, 0);
    // the next batch with any work from pb on into (ob, op, oa); false: none left
    auto fetch = [&](int *ob, int *op, float &oa) -> bool {
        while (pb < b1) {
            const int nq = (int)min((unsigned long long)32, b1 - pb);
            const bool ok = lane < nq;
            const int4 q = qn;
            qn = pb + nq + lane < b1 ? __ldg(pconv + nidx) : make_int4(0, 0, 0, 0);
            nidx = pb + nq + 32 + lane < b1 ? __ldg(bidx + pb + nq + 32 + lane) : 0u;
            int4 hv = make_int4(0, 0, 0, 0);    // (H, window-pointer rows of the class's three levels)
            if (ok) hv = __ldg(reinterpret_cast<const int4 *>(kd[table_of(q.x, q.y, q.z, cb)].cls4[cls]));
            pb += nq;
            oa = __int_as_float(q.w);
            const int side = 2 * hv.x + (EX ? 1 << A.L : 0);
            range(lv0, q.x, q.y, hv.x, side, hv.y, ok, ob[0], op[0]);
            range(lv1, q.x, q.y, hv.x, side, hv.z, ok, ob[1], op[1]);
            range(lv2, q.x, q.y, hv.x, side, hv.w, ok, ob[2], op[2]);
            bool any = false;
#pragma unroll
            for (int j = 0; j < kSlots; j++) any |= __any_sync(kFull, (op[j] & 0xffff) != 0);
            if (any) return true;
        }
        return false;
    };

    // range generator (warp-uniform): level slot gj, remaining points gm, current range
    int gj = 0, c_beg = 0, c_end = 0;
    uint32_t c_sa = tile_sa;
    unsigned gm = 0u;
    float c_a = 0.f;
    int have = 0, nhave = 0, refill = 0;   // ints, not bools: bools get byte-packed (PRMT per update)
    int s_beg = 0, s_pk = 0;                 // this lane's range for slot gj: first entry, (base << 16) | length
    auto select_slot = [&]() {
        s_beg = gj == 0 ? beg[0] : gj == 1 ? beg[1] : beg[2];
        s_pk = gj == 0 ? pk[0] : gj == 1 ? pk[1] : pk[2];
        gm = __ballot_sync(kFull, (s_pk & 0xffff) != 0);
    };
    auto next_range = [&]() {
        while (gm == 0u) {
            if (++gj >= kSlots) {    // batch exhausted: continue with the prefetched next batch, if any
                if (!nhave) {
                    have = 0;
                    c_beg = c_end = 0;    // an empty range: the remaining ring slots idle
                    return;
                }
#pragma unroll
                for (int j = 0; j < kSlots; j++) { beg[j] = nbeg[j]; pk[j] = npk[j]; }
                a_l = na;
                nhave = 0;
                refill = 1;        // the ring loop fetches the batch after it
                gj = 0;
            }
            select_slot();
        }
        const int p = __ffs(gm) - 1;
        gm &= gm - 1u;
        c_beg = __shfl_sync(kFull, s_beg, p);
        const int q = __shfl_sync(kFull, s_pk, p);   // 3 shuffles per range: they use the L1TEX data pipe
        c_end = c_beg + (q & 0xffff);
        c_sa = tile_sa + 8u * (uint32_t)(q >> 16);
        c_a = __shfl_sync(kFull, a_l, p);
        have = 1;
    };
    if (fetch(beg, pk, a_l)) {
        nhave = fetch(nbeg, npk, na);
        gj = 0;
        select_slot();
        next_range();
    }

    // kD-deep register ring of chunks, continuous across range, level and batch boundaries
    // (slot: value, position, smem byte base of the range or of the dummy cell, a_j)
    const uint32_t dummy_sa = tile_sa + 8u * (uint32_t)dummy;
    float2 rv[kD];
    int rp[kD];
    uint32_t rb[kD];
    float ra[kD];
#pragma unroll
    for (int u = 0; u < kD; u++) rv[u] = make_float2(0.f, 0.f);
#define WASABI_PREFETCH(u)                                                          \
    do {                                                                            \
        const int e = c_beg + lane;                                                 \
        const bool v = e < c_end;                                                   \
        if (WASABI_DEBUG_BOUNDS && v && (e < 0 || (int64_t)e >= th->vent_cap + 32)) __trap();   \
        rp[u] = 0;                                                                  \
        if (v) {                                                                    \
            rv[u] = ldg_stream(vval + e);                                           \
            rp[u] = ldg_stream(vpos + e);                                           \
        }                                                                           \
        rb[u] = opq(v ? c_sa : dummy_sa);                                           \
        ra[u] = opqf(c_a);                                                          \
        c_beg += 32;                                                                \
        if (c_beg >= c_end) next_range();                                           \
    } while (0)
#if WASABI_DEBUG_BOUNDS   // every shared access inside the CTA's tile + dummy block
#define WASABI_CHECK_SA(sa) do { if ((sa) - tile_sa >= 8u * (uint32_t)(kData + 8)) __trap(); } while (0)
#else
#define WASABI_CHECK_SA(sa) do { } while (0)
#endif
#define WASABI_CONSUME(u)                                                           \
    do {                                                                            \
        const uint32_t sa = swz(rb[u] + 8u * (uint32_t)rp[u]);                      \
        WASABI_CHECK_SA(sa);                                                        \
        float2 o = lds2(sa);                                                        \
        o.x = fmaf(ra[u], rv[u].x, o.x);                                            \
        o.y = fmaf(ra[u], rv[u].y, o.y);                                            \
        sts2(sa, o);                                                                \
    } while (0)
    // Batches are software-pipelined: when the range generator exhausts a batch it continues with the
    // prefetched next one (a register swap) and flags a refill; the ring loop then leaves its unrolled
    // body with the chunks of the new batch in flight, fetches the batch after it (the window-pointer
    // loads overlap those chunks) and re-enters without draining.  The batch code stays inlined once
    // (fetch, outside the ring body).  The ring drains only at the tile's last batch.
    const int had = have;   // the prefetches may exhaust a small tile (have = 0): its chunks still get consumed
    if (had) {
#pragma unroll
        for (int u = 0; u < kD; u++) WASABI_PREFETCH(u);
    }
#if WASABI_BULKZERO
    {
        const uint32_t mbar = tile_sa + 8u * (uint32_t)(kData + 8);
        asm volatile("{\n .reg .pred p;\n WZ_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n"
                     " @!p bra WZ_%=;\n}" ::"r"(mbar) : "memory");
    }
#endif
    if (had) {
        while (true) {
            bool more = true;
            while (more) {
                more = (have & ~refill) != 0;
#pragma unroll
                for (int u = 0; u < kD; u++) {
                    WASABI_CONSUME(u);
                    WASABI_PREFETCH(u);
                }
            }
            if (!refill) break;                  // drained: no batch left
            refill = 0;
            nhave = fetch(nbeg, npk, na);
        }
    }
#undef WASABI_PREFETCH
#undef WASABI_CONSUME
    __syncthreads();
    tile_epilogue<T, NT>(tile, tile_sa, A.L, fused, qa, bits, psi, A.row0, A.n_h, tile_x0, tile_y0);
}

template <int T, bool EX>
cudaError_t launch_t(const void *d_bins, const void *d_tables, const SupArgs &A, int64_t n_tiles, float2 *psi,
                     int fused, const QArgs &qa, uint8_t *bits, cudaStream_t s) {
    constexpr int M = kWinMargin, S = T + M;
    const int smem = (M + T * S + M + 8 + (WASABI_BULKZERO ? 1 : 0)) * (int)sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(superpose_kernel<T, EX>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (n_tiles > 0) {
        count_launches(1);
        superpose_kernel<T, EX><<<(unsigned)n_tiles, 2 * T, smem, s>>>(d_bins, d_tables, A, psi, fused, qa, bits);
    }
    return cudaGetLastError();
}

// ---- dense gather superposition (gather-mode tables; wasabi.h WASABI_FLAG_GATHER) ----
// Eq.(2) per PIXEL instead of per kept coefficient: a level-l pixel of the tile (R-A6) receives
// a_j table_j(pixel - s_l + H_j) from every point j of the tile's bin, in bin order, from the point's
// dense wavelet table (kept value or 0; R-A8 shifts, or the 2^L-aligned shift of the offset-class
// tables, R-A20).  Unkept coefficients add an exact 0 and positions outside the table nothing, so psi
// is bit-identical to the scatter kernel's.  The dense tables are in Mallat order (internal.h
// mallat_index), where a level-l shift is an integer translation of the level's three subband planes:
// in the tile's own Mallat view (level 1: 3 planes x 32 x 32 cells, level 2: 3 x 16 x 16, levels >= 3
// and LL: 256 cells) every warp load is a contiguous run of one table plane row.  One CTA per 64 x 64
// tile, 256 threads, psi in registers: thread (warp w, lane) owns 12 level-1 cells (plane b = k / 4,
// plane row w + 8 (k % 4), column lane), 3 level-2 cells (plane k, row 2w + lane / 16, column lane % 16)
// and one cell of levels >= 3 / LL (cell tid in level order); then psi goes to the shared tile in the
// interleaved layout and through the scatter kernel's epilogue.
struct GatherArgs {
    int L, cls_bits, tiles_x, tile_rows;
    int64_t row0, n_h, tile0;
};
struct GatherPoint {          // one point of a batch, per tile
    const float2 *tp;         // its dense table
    float a;
    int s;                    // table side
    int off[kMaxLevels + 1];  // Mallat plane-stack offset of level l (1..L), LL at [L]
    int2 o[kMaxLevels];       // table plane coordinates of the tile's plane origin, per level
    int in1;                  // the tile's level-1 window (32 x 32 per plane) lies inside the table
    int pad;
};
constexpr int kGatherBatch = 64;
constexpr int kGatherChunk = 1024;   // bin points sorted by depth at a time (keys: depth << 10 | index)

__global__ void __launch_bounds__(256, 3) gather_kernel(const void *__restrict__ d_bins,
                                                        const void *__restrict__ d_tables, GatherArgs A,
                                                        float2 *__restrict__ psi, int fused, QArgs qa,
                                                        uint8_t *__restrict__ bits) {
    constexpr int T = 64, NT = 256;
    extern __shared__ float2 tile[];
    __shared__ GatherPoint gp[kGatherBatch];
    const char *bb = reinterpret_cast<const char *>(d_bins);
    const BinHeader *bh = reinterpret_cast<const BinHeader *>(bb);
    const int4 *__restrict__ pconv = reinterpret_cast<const int4 *>(bb + bh->pts_off);
    const unsigned long long *__restrict__ bptr = reinterpret_cast<const unsigned long long *>(bb + bh->ptr_off);
    const uint32_t *__restrict__ bidx = reinterpret_cast<const uint32_t *>(bb + bh->idx_off);
    const char *tb = reinterpret_cast<const char *>(d_tables);
    const TableHeader *th = reinterpret_cast<const TableHeader *>(tb);
    const KDesc *__restrict__ kd = reinterpret_cast<const KDesc *>(tb + th->kdesc_off);
    const DDesc *__restrict__ dd = reinterpret_cast<const DDesc *>(tb + th->ddesc_off);
    const float2 *__restrict__ dense = reinterpret_cast<const float2 *>(tb + th->dense_off);

    int64_t t;
    {   // the scatter kernel's tile order (groups of kGroup tile rows, column-major inside a group)
        const int64_t per_group = (int64_t)kGroup * A.tiles_x;
        const int64_t g = blockIdx.x / per_group, rem = blockIdx.x - g * per_group;
        const int gh = (int)min((int64_t)kGroup, A.tile_rows - g * kGroup);
        t = A.tile0 + (g * kGroup + rem % gh) * A.tiles_x + rem / gh;
    }
    const int tile_x0 = (int)(t % A.tiles_x) * T;
    const int tile_y0 = (int)(A.row0 + (t / A.tiles_x) * (int64_t)T);
    const uint32_t tile_sa = (uint32_t)__cvta_generic_to_shared(tile);
    const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
    const int L = A.L;
    // this thread's cell of levels >= 3 / LL: level lc (L + 1 = LL), subband bc, plane cell (ic, jc)
    int lc = L + 1, bc = 0, ic, jc;
    {
        int c = tid;
        for (int l = 3; l <= L; l++) {
            const int q = T >> l, n = 3 * q * q;
            if (c < n) { lc = l; bc = c / (q * q); c -= bc * q * q; break; }
            c -= n;
        }
        const int q = T >> (lc <= L ? lc : L);
        ic = c % q; jc = c / q;
    }
    const int lcs = lc <= L ? lc : L;            // LL moves with level L (R-A6, R-A8)
    float2 h1[12], h2[3], hc;
#pragma unroll
    for (int k = 0; k < 12; k++) h1[k] = make_float2(0.f, 0.f);
#pragma unroll
    for (int k = 0; k < 3; k++) h2[k] = make_float2(0.f, 0.f);
    hc = make_float2(0.f, 0.f);
    const int cm = (1 << A.cls_bits) - 1;
    const unsigned long long b0 = bptr[t], b1 = bptr[t + 1];
    // depth-major order (reading R-A22): the bin is taken in chunks of up to kGatherChunk points (in
    // bin order), each chunk sorted by (depth level, position in the bin); the CTAs resident at one
    // time then read the dense tables of a few depths at a time (L2 reuse) instead of all of them
    __shared__ uint32_t skey[kGatherChunk];
    for (unsigned long long cbeg = b0; cbeg < b1; cbeg += kGatherChunk) {
    const int nc = (int)min((unsigned long long)kGatherChunk, b1 - cbeg);
    int sz = 64;
    while (sz < nc) sz <<= 1;
    __syncthreads();
    for (int i = tid; i < sz; i += NT)
        skey[i] = i < nc ? ((uint32_t)pconv[bidx[cbeg + i]].z << 10) | (uint32_t)i : 0xffffffffu;
    for (int k = 2; k <= sz; k <<= 1) {          // bitonic sort, ascending (keys are distinct)
        for (int jj = k >> 1; jj > 0; jj >>= 1) {
            __syncthreads();
            for (int i = tid; i < sz; i += NT) {
                const int ij = i ^ jj;
                if (ij > i) {
                    const uint32_t x = skey[i], y = skey[ij];
                    if ((x > y) == ((i & k) == 0)) { skey[i] = y; skey[ij] = x; }
                }
            }
        }
    }
    for (int pb = 0; pb < nc; pb += kGatherBatch) {
        const int np = min(kGatherBatch, nc - pb);
        __syncthreads();
        if (tid < np) {
            const int4 q = pconv[bidx[cbeg + (skey[pb + tid] & 1023u)]];
            const int tb_ = table_of(q.x, q.y, q.z, A.cls_bits);
            const int H = kd[tb_].H;
            GatherPoint P;
            P.tp = dense + dd[tb_].coef_off;
            P.s = kd[tb_].side;
            P.a = __int_as_float(q.w);
            int off = 0;
#pragma unroll
            for (int l = 1; l <= kMaxLevels; l++) {
                const int h = 1 << (l - 1), sl = P.s >> l;
                const int sx = A.cls_bits ? (q.x & ~cm) : ((q.x + h) >> l) << l;
                const int sy = A.cls_bits ? (q.y & ~cm) : ((q.y + h) >> l) << l;
                // exact: every term is a multiple of 2^l
                P.o[l - 1] = make_int2((tile_x0 - sx + H) >> l, (tile_y0 - sy + H) >> l);
                P.off[l - 1] = off;
                if (l <= L) off += 3 * sl * sl;
            }
            {
                const int s1 = P.s >> 1;
                P.in1 = P.o[0].x >= 0 && P.o[0].x + T / 2 <= s1 && P.o[0].y >= 0 && P.o[0].y + T / 2 <= s1;
            }
            P.off[kMaxLevels] = off;   // LL right after level L (set in the loop above when L < 6)
            gp[tid] = P;
        }
        __syncthreads();
        for (int j = 0; j < np; j++) {
            const GatherPoint &G = gp[j];
            const float a = G.a;
            const int s = G.s;
            const float2 *__restrict__ tp = G.tp;
            {   // level 1: 12 rows of 32 cells per warp (32-bit offsets from the table pointer)
                const int s1 = s >> 1, d8 = 8 * s1, P1 = s1 * s1;
                const int2 o = G.o[0];
                const int ox = o.x + lane, oy = o.y + w;
                const float2 *__restrict__ p = tp + (oy * s1 + ox);
                if (G.in1) {        // the whole 32 x 32 window inside the table: no checks
#pragma unroll
                    for (int k = 0; k < 12; k++) {
                        const float2 v = __ldg(p + ((k >> 2) * P1 + (k & 3) * d8));
                        h1[k].x = fmaf(a, v.x, h1[k].x);
                        h1[k].y = fmaf(a, v.y, h1[k].y);
                    }
                } else {
                    const bool cok = (unsigned)ox < (unsigned)s1;
#pragma unroll
                    for (int k = 0; k < 12; k++) {
                        if (cok && (unsigned)(oy + 8 * (k & 3)) < (unsigned)s1) {
                            const float2 v = __ldg(p + ((k >> 2) * P1 + (k & 3) * d8));
                            h1[k].x = fmaf(a, v.x, h1[k].x);
                            h1[k].y = fmaf(a, v.y, h1[k].y);
                        }
                    }
                }
            }
            {   // level 2: one row of 16 cells per half-warp, three planes
                const int s2 = s >> 2;
                const int2 o = G.o[1];
                const int ox = o.x + (lane & 15), oy = o.y + 2 * w + (lane >> 4);
                if ((unsigned)ox < (unsigned)s2 && (unsigned)oy < (unsigned)s2) {
                    const float2 *__restrict__ p = tp + (G.off[1] + oy * s2 + ox);
                    const int P2 = s2 * s2;
#pragma unroll
                    for (int k = 0; k < 3; k++) {
                        const float2 v = __ldg(p + k * P2);
                        h2[k].x = fmaf(a, v.x, h2[k].x);
                        h2[k].y = fmaf(a, v.y, h2[k].y);
                    }
                }
            }
            {   // levels >= 3 / LL: one cell
                const int sc = s >> lcs;
                const int2 o = G.o[lcs - 1];
                const int ox = o.x + ic, oy = o.y + jc;
                if ((unsigned)ox < (unsigned)sc && (unsigned)oy < (unsigned)sc) {
                    const float2 v = __ldg(tp + (G.off[lc - 1] + bc * sc * sc + oy * sc + ox));
                    hc.x = fmaf(a, v.x, hc.x);
                    hc.y = fmaf(a, v.y, hc.y);
                }
            }
        }
    }
    }
    // psi of the tile into the (swizzled) shared tile in the interleaved layout, then the epilogue
    constexpr int M = kWinMargin, S = T + M;
    auto cell = [&](int r, int x) -> float2 & {
        return tile[(swz(tile_sa + 8u * (uint32_t)(M + r * S + x)) - tile_sa) >> 3];
    };
#pragma unroll
    for (int k = 0; k < 12; k++) {   // level 1, subband b: pixel (2i + (b != 1), 2j + (b >= 1))
        const int b = k >> 2, jr = w + 8 * (k & 3);
        cell(2 * jr + (b >= 1), 2 * lane + (b != 1)) = h1[k];
    }
#pragma unroll
    for (int k = 0; k < 3; k++) {    // level 2: (4i + 2 (b != 1), 4j + 2 (b >= 1))
        const int jr = 2 * w + (lane >> 4), ir = lane & 15;
        cell(4 * jr + 2 * (k >= 1), 4 * ir + 2 * (k != 1)) = h2[k];
    }
    {
        const int hh = lc <= L ? 1 << (lc - 1) : 0;
        cell((jc << lcs) + (bc >= 1 ? hh : 0), (ic << lcs) + (bc != 1 ? hh : 0)) = hc;
    }
    __syncthreads();
    tile_epilogue<T, NT>(tile, tile_sa, L, fused, qa, bits, psi, A.row0, A.n_h, tile_x0, tile_y0);
}

}  // namespace

cudaError_t launch_gather(const void *d_bins, const void *d_tables, int L, int cls_bits, int tiles_x, int tiles_y,
                          int64_t row0, int64_t n_h, float2 *psi, int fused, const double *print4, double pitch,
                          uint8_t *bits, cudaStream_t s, int tile_row0, int tile_row1) {
    constexpr int T = 64, M = kWinMargin, S = T + M;
    if (L < 2) return cudaErrorInvalidValue;
    if (tile_row1 < 0) tile_row1 = tiles_y;
    GatherArgs A;
    A.L = L; A.cls_bits = cls_bits; A.tiles_x = tiles_x; A.row0 = row0; A.n_h = n_h;
    A.tile0 = (int64_t)tile_row0 * tiles_x;
    A.tile_rows = tile_row1 - tile_row0;
    const int64_t n_tiles = (int64_t)tiles_x * (tile_row1 - tile_row0);
    const QArgs qa = make_qargs(print4, pitch, n_h);
    const int smem = (M + T * S + M + 8) * (int)sizeof(float2);
    cudaError_t e = cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (e != cudaSuccess) return e;
    if (n_tiles > 0) {
        count_launches(1);
        gather_kernel<<<(unsigned)n_tiles, 256, smem, s>>>(d_bins, d_tables, A, psi, fused, qa, bits);
    }
    return cudaGetLastError();
}

cudaError_t launch_superpose(const void *d_bins, const void *d_tables, int T, int S, int L, int cls_bits, int tiles_x,
                             int tiles_y, int64_t row0, int64_t n_h, float2 *psi, int fused, const double *print4,
                             double pitch, uint8_t *bits, cudaStream_t s, int tile_row0, int tile_row1) {
    if (S != T + kWinMargin) return cudaErrorInvalidValue;
    if (tile_row1 < 0) tile_row1 = tiles_y;
    SupArgs A;
    A.L = L; A.cls_bits = cls_bits; A.tiles_x = tiles_x; A.row0 = row0; A.n_h = n_h;
    A.tile0 = (int64_t)tile_row0 * tiles_x;
    A.tile_rows = tile_row1 - tile_row0;
    const int64_t n_tiles = (int64_t)tiles_x * (tile_row1 - tile_row0);
    const QArgs qa = make_qargs(print4, pitch, n_h);
    if (cls_bits)
        return T <= 64 ? launch_t<64, true>(d_bins, d_tables, A, n_tiles, psi, fused, qa, bits, s)
                       : launch_t<128, true>(d_bins, d_tables, A, n_tiles, psi, fused, qa, bits, s);
    return T <= 64 ? launch_t<64, false>(d_bins, d_tables, A, n_tiles, psi, fused, qa, bits, s)
                   : launch_t<128, false>(d_bins, d_tables, A, n_tiles, psi, fused, qa, bits, s);
}

}  // namespace wasabi
