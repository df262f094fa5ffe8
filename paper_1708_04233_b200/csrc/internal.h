// internal.h -- device buffer layouts and kernel launchers of libwasabi (product side only).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace wasabi {

constexpr uint64_t kTableMagic = 0x3142545942415357ull;  // "WSABYTB1"
constexpr uint64_t kBinMagic = 0x314e494249425357ull;    // "WSBIBIN1"
constexpr int kMaxLevels = 6;
constexpr int kMaxTableSide = 16384;  // 2H limit: entry positions are packed as 14-bit X and Y

// LUT entry (16 bytes, 16-byte aligned so that any range of entries is a legal TMA bulk copy):
//   x = X | Y << 14 | level << 28   (table coordinates of the coefficient, level 1..L; LL is level L)
//   y, z = value (re, im) as float bits, w = 0
__host__ __device__ inline uint32_t pack_entry_pos(int X, int Y, int level) {
    return (uint32_t)X | ((uint32_t)Y << 14) | ((uint32_t)level << 28);
}

// Compact per-table data read by the hot kernels (112 bytes).
struct KDesc {
    int32_t H;                    // table half side (H, vbase: one 8-byte load in the hot kernel)
    int32_t vbase;                // window LUT pointer slots of this table start here (== vptr_base[0])
    int32_t E;                    // structural footprint bound ceil(R) + 3 2^(L-1) (buffer sizing)
    int32_t Ek;                   // kept reach, per axis (R-A19; computed by the table build)
    int32_t Q;                    // kept reach, squared distance (R-A19; computed by the table build)
    int32_t ptr_base[kMaxLevels]; // canonical LUT: level l (1..L) band pointer rows start at ptr_base[l-1]
    int32_t vptr_base[kMaxLevels];// window LUT: level l pointer rows start at vptr_base[l-1]
    int32_t side;                 // table side: 2H, or 2H + 2^L for offset-class tables (R-A20)
    int32_t Ed;                   // PSF-disc reach per axis, ceil(Rh), Rh = R(|z_d| + dz/2) + 1 (direct sums)
    int32_t Qd;                   // PSF-disc reach, squared distance ceil(Rh^2)
    int32_t cls4[2][4];           // superposition warp class c: {H, vptr_base of its level slots 0..2}
};                                // (one 16-byte load per point; superpose_class_level)
static_assert(sizeof(KDesc) % 16 == 0 && offsetof(KDesc, cls4) % 16 == 0, "KDesc: cls4[c] is one 16-byte load");

// Level of slot j (0..2) of superposition warp class c (every Haar level owns its own pixels, R-A6):
// c = 0 -> {1, 3, 6}, c = 1 -> {2, 4, 5} (L >= 4); 0 = none (levels beyond L).
// With L <= 3 the classes are {1} / {2, 3} (coif1 at level 3: superpose 4.09 -> 3.96 ms on a 4096-row
// C4 band; Haar at level 3 unchanged).
__host__ __device__ inline int superpose_class_level(int c, int j, int L) {
    if (L <= 3) {
        const int l3 = c == 0 ? (j == 0 ? 1 : 0) : (j < 2 ? j + 2 : 0);
        return l3 <= L ? l3 : 0;
    }
    const int l = c == 0 ? (j == 0 ? 1 : j == 1 ? 3 : j == 2 ? 6 : 0) : (j == 0 ? 2 : j < 3 ? j + 3 : 0);
    return l <= L ? l : 0;
}

// Offset-class tables (WASABI_FLAG_EXACT_SHIFT, reading R-A20): with cb = L class bits, depth d
// has 4^L tables t = (d << 2cb) | (cy << cb) | cx, (cx, cy) = (ix, iy) mod 2^L; every level of a
// point is shifted by the 2^L-aligned (ix - cx, iy - cy).  cb = 0: one table per depth.
__host__ __device__ inline int table_of(int ix, int iy, int iz, int cb) {
    const int m = (1 << cb) - 1;
    return (iz << (2 * cb)) | ((iy & m) << cb) | (ix & m);
}

// ---- window LUT (the superposition kernel's copy of the kept lists) ----
// A warp of the superposition kernel owns a 32-row strip of a T x T tile.  For a point and a
// level l its strip is the table window rows [o, o + 32), o = strip_y0 - s_l(iy) + H, columns
// [xs, xs + T), xs = tile_x0 - s_l(ix) + H.  o is a multiple of q_l = min(2^l, 32), so the
// level-l entries are stored once per "variant" v = (o mod 32) / q_l in bands of exactly 32
// rows [v q_l + 32 (k - 1), v q_l + 32 k): every strip window is exactly one band (no rows
// outside the window are streamed).  Inside a band entries are ordered by column group of
// G_l = max(8, 2^l) pixels with one int32 pointer per group boundary, so a window is one
// contiguous entry range; for l <= 2 it may include up to kWinMargin columns on either side,
// which land in the shared tile's margin columns (never read).
constexpr int kWinRows = 32;
#ifndef WASABI_WIN_MARGIN
#define WASABI_WIN_MARGIN 8
#endif
// >= 6 (level-1 column-group overrun); 8 so that the shared tile's rows (stride T + 8) start on
// 8-cell (64-byte) boundaries and the superposition kernel's bank swizzle (an XOR of address
// bits 3..5) keeps every margin cell inside a margin block
constexpr int kWinMargin = WASABI_WIN_MARGIN;
static_assert(kWinMargin >= 6 && kWinMargin % 8 == 0, "window margin: >= 6 and a multiple of 8");
// log2 q_l: window starts are multiples of min(2^l, 32); with offset-class tables (cb = L class
// bits, R-A20) every level is shifted by multiples of 2^L, so of min(2^max(l, L), 32)
__host__ __device__ inline int win_lq(int l, int cb) { const int m = l > cb ? l : cb; return m < 5 ? m : 5; }
__host__ __device__ inline int win_lg(int l) { return l < 3 ? 3 : l; }          // log2 G_l
__host__ __device__ inline int win_variants(int l, int cb) { return kWinRows >> win_lq(l, cb); }
__host__ __device__ inline int win_bands(int side) { return (side + kWinRows - 1) / kWinRows + 1; }
__host__ __device__ inline int win_cols(int side, int l) { return (side + (1 << win_lg(l)) - 1) >> win_lg(l); }
// pointer slots of level l of one table
// window-LUT positions are uint16 (Y - band start) * S + X: 31 (T + margin) + side - 1 must fit
static_assert(31 * (128 + kWinMargin) + kMaxTableSide - 1 <= 65535, "window-LUT positions overflow uint16");
__host__ __device__ inline int win_slots(int side, int l, int cb) {
    return win_variants(l, cb) * win_bands(side) * (win_cols(side, l) + 1);
}

// Dense wavelet tables of the gather superposition (WASABI_FLAG_GATHER), Mallat (subband-planar)
// order: table side s, s_l = s >> l; level l = 1..L, subband b = 0 (X & h, Y even at h), 1 (Y & h
// only), 2 (both), h = 2^(l-1), is the s_l x s_l plane at mallat_plane(s, l) + b s_l^2, cell (X >> l,
// Y >> l) row-major; LL (X, Y multiples of 2^L) is the plane at mallat_plane(s, L + 1).  A level-l
// shift by a multiple of 2^l (R-A8, R-A20) is then an integer translation of the level's planes.
__host__ __device__ inline int32_t mallat_plane(int s, int l) {
    int32_t off = 0;
    for (int k = 1; k < l; k++) off += 3 * (s >> k) * (s >> k);
    return off;
}
__host__ __device__ inline int64_t mallat_index(int X, int Y, int s, int L) {
    const int m = X | Y;
    for (int l = 1; l <= L; l++) {
        const int h = 1 << (l - 1);
        if (m & h) {
            const int sl = s >> l, b = ((Y & h) ? 1 : 0) + (((X & h) && (Y & h)) ? 1 : 0);
            return (int64_t)mallat_plane(s, l) + (int64_t)b * sl * sl + (int64_t)(Y >> l) * sl + (X >> l);
        }
    }
    const int sL = s >> L;
    return (int64_t)mallat_plane(s, L + 1) + (int64_t)(Y >> L) * sL + (X >> L);
}

// Per-depth data used by the table build and exports.
struct DDesc {
    double z, R;
    int64_t nnz, n_r;
    int64_t coef_off;   // element offset of this depth's (2H)^2 table in the build scratch
    int32_t side;       // 2H
    int32_t tiles;      // ceil(side / 64) tiles per side for K1
    int32_t cta_base;   // prefix of K1 CTAs (tiles^2)
    int32_t group_base; // prefix of (level, band, Xb) groups (== its ptr_base for level 1)
    int32_t n_groups;
    int32_t vgroup_base; // prefix of window-LUT pointer slots (== its vptr_base for level 1)
    int32_t cx, cy;      // PSF centre offset from (H, H): the offset class (R-A20), else 0
};

struct TableHeader {
    uint64_t magic;
    uint64_t param_hash;
    int32_t n_depth, levels, tile, S;  // n_depth = number of TABLES; S = smem row stride baked into positions
    int64_t total_entries;             // sum N_r,d
    int64_t total_ptrs;                // int32 pointer slots
    int64_t total_ctas;                // K1 grid
    int64_t kdesc_off, ddesc_off, ent_off, ptr_off, ctabase_off;  // byte offsets
    int64_t pad0;
    int64_t table_bytes;
    int64_t total_vptrs;               // window-LUT int32 pointer slots
    int64_t vent_cap;                  // window-LUT entry capacity (bound: 16 N_r per depth)
    int64_t vptr_off, vval_off, vpos_off;  // window LUT: pointers, float2 values, uint16 positions
    int32_t cls_bits, n_zlevels;       // offset-class bits cb (0 or L) and depth levels N_z
    int32_t wavelet, gather;           // 0 Haar, 1 coif1 (R-A21); 1: dense gather superposition
    int64_t dense_off;                 // dense wavelet tables (gather mode), byte offset
};
static_assert(sizeof(TableHeader) <= 256, "table header must fit the 256-byte slot");

struct BinHeader {
    uint64_t magic;
    uint64_t param_hash;
    int64_t n_points, row0, row1;
    int32_t T, tiles_x, tiles_y, pad0;
    int64_t n_tiles, capacity;
    int64_t pts_off, ptr_off, cnt_off, idx_off, idx2_off, scan_off;  // byte offsets
    int64_t bin_bytes;
    // device-written statistics
    unsigned long long n_valid, n_skipped, total_entries, status;
    int64_t pad[2];
};

// Band height (pixels) of the per-level pointer index: T/4, >= 2^l (hb_l = max(1, (T/4) >> l)).
__host__ __device__ inline int band_blocks(int T, int l) {
    int hb = (T / 4) >> l;
    return hb < 1 ? 1 : hb;
}

// Dense (untransformed) PSF table of one depth, for the direct-sum stamping kernel (32 bytes).
struct DenseDesc {
    double z, R;
    int64_t off;       // element offset of the (side x side) complex64 table
    int32_t side;      // 2H
    int32_t cta_base;  // prefix of 64x64 build CTAs
};

// ---- table geometry computed on host (L0) ----
struct LevelGeom {
    int nb, hb, nbands;   // blocks per row, band height (blocks), bands
};

// Number of kernels this library has launched (process-wide, relaxed atomic).
void count_launches(int n);

// ---- launchers ----
cudaError_t launch_psf_haar(const TableHeader &h, const void *d_tables, float2 *coef_val, uint32_t *coef_key,
                            double k, double pitch, int levels, int n_depth, cudaStream_t s);
cudaError_t launch_select(const TableHeader &h, const void *d_tables, const uint32_t *coef_key,
                          unsigned int *hist, unsigned long long *sel_state, int n_depth, cudaStream_t s);
cudaError_t launch_groups(const TableHeader &h, void *d_tables, const float2 *coef_val, const uint32_t *coef_key,
                          const unsigned long long *sel_state, int pass, cudaStream_t s);
// the window LUT per canonical entry (pass 0: count into the vptr slots; pass 1: place at cursor[])
cudaError_t launch_ventries(const TableHeader &h, void *d_tables, int pass, int32_t *cursor, cudaStream_t s);
// coiflet mode (R-A21): fp64 PSF + L-level coif1 analysis of every table (work/tmp: fp64 tables,
// d_pre: per level the (n_tables + 1) prefix of (lines x pairs) work items, h_pre_last: its totals)
cudaError_t launch_coif_tables(const TableHeader &h, const void *d_tables, double2 *work, double2 *tmp,
                               const int64_t *d_pre, const int64_t *h_pre_last, float2 *val, uint32_t *key,
                               int64_t n_coef, double k, double pitch, int L, cudaStream_t s);
// coif1 synthesis of a psi band (nrows x n_h) in place, levels L..1
cudaError_t launch_coif_inverse(float2 *psi, int64_t nrows, int64_t n_h, int L, cudaStream_t s);
cudaError_t launch_coif_fused(const float2 *psi, int64_t e0, int64_t e1, int64_t row0, int64_t row1, int64_t n_h,
                              int L, const double *print4, double pitch, float2 *u, uint8_t *bits, cudaStream_t s);
// gather mode: every kept canonical entry written into its table's dense copy (zeroed beforehand)
cudaError_t launch_dense_fill(const TableHeader &h, void *d_tables, cudaStream_t s);
cudaError_t launch_scan_i32(int32_t *data, int64_t n, void *scratch, cudaStream_t s);
cudaError_t launch_scan_u32_to_u64(const uint32_t *in, unsigned long long *out, int64_t n, void *scratch,
                                   cudaStream_t s);
size_t scan_scratch_bytes(int64_t n);

// psf = 1: bins by the whole PSF disc (Ed, Qd) instead of the kept coefficients' reach (direct sum)
cudaError_t launch_bin(const BinHeader &bh, void *d_bins, const KDesc *kd, const float4 *pts,
                       double pitch, int64_t n_h, double z_min, double dz, int n_depth, int cls_bits,
                       int psf, cudaStream_t s);

// Eq.(2) accumulation count of band [row0, row1) into *d_count (device u64) and, if d_row_work !=
// NULL (n_h + 1 doubles), the per-row work estimate of the balanced bands (inclusive prefix sums of
// a difference array, scanned: [Y] = work of row Y for Y < n_h).  h: the host copy of the table header.
cudaError_t launch_count_acc(const TableHeader &h, const void *d_tables, const float4 *pts, int64_t n, double pitch,
                             int64_t n_h, double z_min, double dz, int n_depth, int cls_bits, int L, int64_t row0,
                             int64_t row1, unsigned long long *d_count, double *d_row_work, cudaStream_t s);

// fused = 0: write psi; fused = 1: inverse Haar in shared memory, write u (psi pointer, may be NULL)
// and, if bits != NULL, the print bits (print4 = {xr, yr, zr, 1/lambda}).
// tile rows [tile_row0, tile_row1) of the bins' band (tile_row1 < 0: all)
cudaError_t launch_superpose(const void *d_bins, const void *d_tables, int T, int S, int L, int cls_bits, int tiles_x,
                             int tiles_y, int64_t row0, int64_t n_h, float2 *psi, int fused, const double *print4,
                             double pitch, uint8_t *bits, cudaStream_t s, int tile_row0 = 0, int tile_row1 = -1);
// dense gather superposition (gather-mode tables, T = 64): same outputs as launch_superpose
cudaError_t launch_gather(const void *d_bins, const void *d_tables, int L, int cls_bits, int tiles_x, int tiles_y,
                          int64_t row0, int64_t n_h, float2 *psi, int fused, const double *print4, double pitch,
                          uint8_t *bits, cudaStream_t s, int tile_row0 = 0, int tile_row1 = -1);
cudaError_t launch_write_blob(void *dst, const void *src, size_t bytes, cudaStream_t s);

cudaError_t launch_psf_dense(const DenseDesc *d_desc, int n_depth, float2 *out, double k, double pitch,
                             int64_t total_ctas, cudaStream_t s);
cudaError_t launch_stamp(const void *d_bins, const DenseDesc *d_desc, const float2 *dense, int tiles_x, int tiles_y,
                         int64_t row0, int64_t n_h, int T, float2 *u, cudaStream_t s);

// exact Eq.(1) (D1) of a band from the original points and PSF-disc bins
cudaError_t launch_exact(const void *d_bins, const float4 *pts, int tiles_x, int tiles_y, int64_t row0, int64_t n_h,
                         int T, double pitch, double tan_theta, double wavelength, float2 *u, cudaStream_t s);

cudaError_t launch_inverse(const float2 *psi, float2 *u, int64_t rows, int64_t n_h, int64_t row0, int levels,
                           const double *print4 /* xr, yr, zr, inv_lambda or NULL */, double pitch,
                           uint8_t *bits, cudaStream_t s);
cudaError_t launch_quantize(const float2 *u, int64_t rows, int64_t n_h, int64_t row0, const double *print4,
                            double pitch, uint8_t *bits, cudaStream_t s);

}  // namespace wasabi
