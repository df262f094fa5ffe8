/*
 * wasabi.h -- C ABI of the B200-native WASABI hot path (arXiv 1708.04233,
 * "Fast, large-scale hologram calculation in wavelet domain"; PAPER.md in the
 * reference).  Library: paper_1708_04233_b200/libwasabi.so (sm_100a kernels).
 *
 * The path (Sec. 1, :86-95 and :115-125):
 *   step 1  wasabi_build_psf_tables  per-depth PSF u_z = exp(ikr) circ(.),
 *           depth-discretised (:91), forward Haar FWT (:91, Haar per north_star instead of
 *           the paper's coiflets :106), top-N_r strong coefficients kept in a LUT (:92).
 *   step 2a wasabi_bin_points        object points (x, y, z, a) (Eq.(1), :70-75) converted to
 *           pixels/levels and binned to the T x T tiles their PSF footprint overlaps -- the
 *           paper's sub-hologram re-basing x'_j = x_j - s N_h (:115-122) applied per tile.
 *   step 2b wasabi_superpose         Eq.(2) (:108-113): psi(m,n) = sum_j a_j sum_k c_{z_j,k}
 *           delta(m - alpha x_j, n - alpha y_j), alpha = 2^-l per level (reading R-A8).
 *   step 3  wasabi_inverse_wt        inverse FWT of psi (:94, :123), optionally fused with
 *   step 4  wasabi_quantize          binary-amplitude print pattern against a spherical
 *           reference wave (:135, :137).
 * Readings of the paper where it is silent/garbled are listed in DESIGN.md §2 (R-xx).
 *
 * Conventions (all entry points):
 *  - Ownership: the CALLER allocates and frees every device buffer.  The library never
 *    allocates device memory (wasabi_hologram_host copies into a caller-provided workspace).
 *  - Streams: every compute call is asynchronous on `stream` (cudaStream_t; NULL = legacy
 *    default stream).  Size queries are host-only.  export/stats/check calls synchronise.
 *  - Errors: functions return wasabi_status; on a non-OK status wasabi_last_error() returns a
 *    thread-local message.  WASABI_EINVAL = parameter violation (message names it),
 *    WASABI_ENOSPC = buffer too small (message gives the required bytes), WASABI_ECUDA = a CUDA
 *    launch/API error, WASABI_ESTATE = a buffer built with other parameters.
 *  - Point-level problems never fail a call (non-finite coordinates, a <= 0, z more than half
 *    a level outside [z_min, z_max]): such points are skipped and counted (wasabi_bins_stats).
 *  - Pixel convention: hologram pixel (X, Y) is at ((X - N_h/2) p, (Y - N_h/2) p) metres
 *    (hologram-centred origin, reading R-A9).  Fields are row-major, Y slowest.
 *  - Complex fields are interleaved float32 (re, im) = "complex64", 8 bytes per pixel.
 *  - Bands: [row0, row1) is a band of hologram rows; row0 and row1 must be multiples of
 *    params.tile.  All band buffers hold only the band: (row1-row0) x N_h pixels.
 */
#ifndef WASABI_H
#define WASABI_H

#include <stddef.h>
#include <stdint.h>
#include <cuda_runtime_api.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    WASABI_OK = 0,
    WASABI_EINVAL = -1,
    WASABI_ENOSPC = -2,
    WASABI_ECUDA = -3,
    WASABI_ESTATE = -4
} wasabi_status;

/* Problem parameters -- the paper's problem statement (Eq.(1) inputs; depth
 * discretisation :91; wavelet levels :106) plus the GPU tile side. */
typedef struct {
    double wavelength_m;  /* lambda > 0; Nyquist: lambda < 2 * pitch, else EINVAL   */
    double pitch_m;       /* pixel pitch p > 0                                      */
    int64_t n_h;          /* square hologram side N_h; multiple of tile                            */
    int32_t n_depth;      /* N_z >= 1 depth levels                              */
    int32_t levels;       /* Haar levels L, 1..6                                                    */
    double z_min_m;       /* level centres z_d = z_min + d (z_max - z_min)/(N_z - 1) (R-A3)         */
    double z_max_m;       /* z_max >= z_min; N_z = 1 uses z_min only                                */
    double retention;     /* r in (0, 1]: N_r,d = min(nnz_d, ceil(r_ppm nnz_d / 1e6)), r_ppm =
                             llround(r 1e6) >= 1 (R-A4; the paper's N_r = pi (W/2)^2 gamma, :92)   */
    int32_t tile;         /* T: bin / superposition tile side; 64 or 128 (multiple of 2^L)        */
    uint32_t flags;       /* 0, WASABI_FLAG_EXACT_SHIFT or WASABI_FLAG_COIFLET (not both), optionally
                             | WASABI_FLAG_GATHER or WASABI_FLAG_SCATTER; other bits: EINVAL       */
} wasabi_params;

/* Exact off-grid shifts (reading R-A20; needs levels <= 4).  Instead of
 * one table per depth whose level-l coefficients are shifted by s_l = 2^l floor((i + 2^(l-1))/2^l)
 * (R-A8, exact only for 2^L-aligned points), every depth d gets 4^L "offset-class" tables
 * t = d 4^L + cy 2^L + cx, (cx, cy) = (ix, iy) mod 2^L, each the PSF centred at (H + cx, H + cy)
 * in a (2H + 2^L)^2 table, transformed and shrunk on its own; every coefficient of a point is
 * shifted by the 2^L-aligned (ix - cx, iy - cy).  At r = 1 the hologram then equals the
 * quantised direct sum for ANY integer position.  In this mode the `depth` argument of
 * wasabi_depth_geometry / wasabi_export_table / wasabi_export_reach is the table index t
 * (0 <= t < wasabi_table_count). */
#define WASABI_FLAG_EXACT_SHIFT 1u

/* Coiflets, the paper's wavelet ("coiflets as the wavelets at level 3"; SURVEY.md
 * §8(f) NEXT-2, reading R-A21; needs levels <= 4, not with EXACT_SHIFT).  The tables
 * use the coif1 filter bank (6 taps) on the interleaved layout with zero extension, padded so every
 * nonzero coefficient is kept in the table; the superposition is unchanged.  The inverse is not
 * block-local: u on rows [row0, row1) needs psi on the HALO band [max(0, row0 - H), min(n_h, row1 +
 * H)), H = wasabi_coif_halo_rows(params), so: wasabi_bin_points + wasabi_superpose on the halo band,
 * then wasabi_inverse_wt (d_psi = that halo band, transformed in place).  wasabi_superpose_inverse
 * (the fused Haar kernel) returns EINVAL in this mode; wasabi_hologram_host handles it. */
#define WASABI_FLAG_COIFLET 2u

/* Dense gather superposition (the r -> 100% regime).  Eq.(2) is a sum of
 * sparse kept coefficients; at high retention the kept set is nearly dense and a per-pixel GATHER from
 * a dense wavelet-domain table (kept value or 0; one side^2 complex64 table per PSF table, in Mallat
 * subband-planar order) beats the scatter of the kept list.  Each pixel of level l (R-A6) reads its
 * table at (pixel - s_l + H) for every point of its tile's bin, in depth-major order (reading R-A22:
 * chunks of up to 1024 bin points, each sorted by (depth level, bin position), so the CTAs resident
 * at one time read a few depths' tables at a time): psi equals the scatter path's up to the fp32
 * rounding of the reordered sum, and is itself bitwise independent of the band split.  Default
 * (neither flag): gather iff retention >= 0.25 (measured crossover at C5), tile == 64, levels >= 2 and not coiflets; the flags
 * force one path (GATHER needs tile 64, levels >= 2, Haar).  In gather mode the table buffer holds
 * the dense tables instead of the superposition's window LUT. */
#define WASABI_FLAG_GATHER 4u
#define WASABI_FLAG_SCATTER 8u

/* Rows of psi halo the coiflet inverse needs on each side of a band (= tile; 0 for Haar). */
int64_t wasabi_coif_halo_rows(const wasabi_params *params);

/* Spherical reference wave point (paper default (0, 0.030, -0.400) m). */
typedef struct {
    double x_r_m, y_r_m, z_r_m;
} wasabi_print_params;

/* Host-side geometry of one depth level (no device access). */
typedef struct {
    double z_m;           /* level depth z_d                                                       */
    double radius_px;     /* R_d = |z_d| tan(asin(lambda/2p)) / p (reading R-A2)      */
    int64_t half;         /* H_d: PSF table side is 2 H_d, centre at (H_d, H_d)                    */
    int64_t footprint;    /* E_d = ceil(R_d) + 3 2^(L-1): footprint half-size used for binning     */
    int64_t nnz;          /* structural nonzero wavelet coefficients (blocks touching the disc)   */
    int64_t n_r;          /* N_r,d kept coefficients                                               */
} wasabi_depth_info;

/* ---------------------------------------------------------------- step 1 */

/* Bytes of the table buffer (device, immutable after build) and of the build scratch. */
wasabi_status wasabi_psf_tables_bytes(const wasabi_params *params, size_t *table_bytes,
                                      size_t *scratch_bytes);

/* Step 1: for every depth level, PSF -> L-level forward Haar (fp64) -> keep the
 * N_r,d coefficients with the largest fp32(|c|^2), ties to the smaller table index (R-A13) ->
 * LUT.  d_tables (table_bytes) and d_scratch (scratch_bytes) are caller-owned device buffers;
 * d_tables is fully (re)written and self-describing; d_scratch may be reused after the stream
 * passes this call.  Alignment: 256 bytes. */
wasabi_status wasabi_build_psf_tables(const wasabi_params *params, void *d_tables, size_t table_bytes,
                                      void *d_scratch, size_t scratch_bytes, cudaStream_t stream);

/* Geometry of depth `depth` (host only; table index in WASABI_FLAG_EXACT_SHIFT mode). */
wasabi_status wasabi_depth_geometry(const wasabi_params *params, int32_t depth, wasabi_depth_info *out);

/* Number of PSF tables: n_depth, or n_depth 4^L with WASABI_FLAG_EXACT_SHIFT (host only). */
wasabi_status wasabi_table_count(const wasabi_params *params, int64_t *n_tables);

/* ---------------------------------------------------------------- step 2a */

/* Upper bound of the bin buffer for n points and band [row0, row1) (host only, no sync). */
wasabi_status wasabi_bin_points_bytes(const wasabi_params *params, int64_t n, int64_t row0, int64_t row1,
                                      size_t *bin_bytes);

/* Step 2a: convert points to (ix, iy, iz) in fp64 (R-A3, R-A9, R-A17) and
 * build, for every T x T tile of band [row0, row1), the list of points (ascending index,
 * R-A11) whose footprint (R-A19: the kept coefficients' reach ek, q of the point's depth, see
 * wasabi_export_reach) contains the tile.  The buffer bound uses the structural E >= ek.
 * d_points: n x 4 float32 (x, y, z, a) [m, m, m, -], 16-byte aligned, n >= 0.
 * d_bins: bin_bytes from wasabi_bin_points_bytes (or more); fully rewritten.
 * d_tables: built by wasabi_build_psf_tables with the same params. */
wasabi_status wasabi_bin_points(const wasabi_params *params, const void *d_tables, const float *d_points,
                                int64_t n, int64_t row0, int64_t row1, void *d_bins, size_t bin_bytes,
                                cudaStream_t stream);

/* ---------------------------------------------------------------- step 2b */

/* Step 2b, Eq.(2): psi for band [row0, row1) (must equal the bins' band) in
 * the interleaved in-place Haar layout (R-A6).  Coefficient (l, dX, dY, c) of point j lands at
 * X = s_l(ix_j) + dX, Y = s_l(iy_j) + dY with s_l(i) = 2^l floor((i + 2^(l-1)) / 2^l) (R-A8);
 * contributions outside the hologram or band are dropped (R-A12).  One CTA owns each tile in
 * shared memory, no global atomics; per-pixel accumulation order is fixed (deterministic).
 * d_psi: (row1 - row0) x n_h complex64, overwritten. */
wasabi_status wasabi_superpose(const wasabi_params *params, const void *d_tables, const void *d_bins,
                               int64_t row0, int64_t row1, float *d_psi, cudaStream_t stream);

/* Steps 2b + 3 (+ 4) fused (PAPER.md:93-94 run back to back): each tile's
 * psi is superposed, inverse-transformed and quantised in shared memory and never written to HBM.
 * Results are bit-identical to wasabi_superpose followed by wasabi_inverse_wt.
 * d_u: (row1 - row0) x n_h complex64 or NULL (print only); d_bits as in wasabi_quantize or NULL
 * (then `print` may be NULL). */
wasabi_status wasabi_superpose_inverse(const wasabi_params *params, const void *d_tables, const void *d_bins,
                                       int64_t row0, int64_t row1, const wasabi_print_params *print, float *d_u,
                                       uint8_t *d_bits, cudaStream_t stream);

/* ---------------------------------------------------------------- steps 3 (+4) */

/* Step 3: L-level inverse Haar, tile-local (band rows multiples of 2^L, so
 * no halo).  d_psi is only read in Haar mode (d_u may alias it: in place); it is overwritten in
 * coiflet mode (below).  d_u == NULL: u is not written (print only).
 * d_bits != NULL fuses step 4 (see wasabi_quantize) and requires `print`.
 * WASABI_FLAG_COIFLET: d_psi is the halo band [max(0, row0 - H), min(n_h, row1 + H)) x n_h
 * (H = wasabi_coif_halo_rows); coif1 synthesis with zero outside the band and the hologram.
 *  - d_u outside d_psi, or d_u == NULL with d_bits: FUSED -- each 64 x 64 tile of u is synthesised
 *    from its psi (plus a halo of 3 (2^L - 1) pixels, rounded up to 2^L) in shared memory and
 *    quantised there; d_psi is only read.
 *  - d_u == the matching rows of d_psi, or d_u == d_bits == NULL: the line passes run IN PLACE on
 *    the halo band and rows [row0, row1) of d_psi are u (then d_bits, if any, from them).
 *  Both give bit-identical u and bits. */
wasabi_status wasabi_inverse_wt(const wasabi_params *params, float *d_psi, float *d_u, int64_t row0,
                                int64_t row1, const wasabi_print_params *print, uint8_t *d_bits,
                                cudaStream_t stream);

/* Step 4: R = exp(+i k sqrt((x-x_r)^2 + (y-y_r)^2 + z_r^2)) with the phase
 * reduced in fp64 (R-A15), I = Re(u conj(R)), bit = (I >= 0) (R-A14).  d_bits: (row1-row0) x
 * n_h/8 bytes, pixel X -> byte X >> 3, bit 7 - (X & 7) (MSB first); 1 = transparent.  Per print
 * byte the distance takes one fp64 square root and a second-order series for the other 7 pixels
 * when the series error is below 1e-8 quarter cycles everywhere (checked from the parameters;
 * otherwise one square root per pixel); (cos, sin) of the fractional quarter cycle in fp32 (< 1e-7).
 * Every entry point binarises through the same code, so fused and unfused bits are identical. */
wasabi_status wasabi_quantize(const wasabi_params *params, const wasabi_print_params *print, const float *d_u,
                              int64_t row0, int64_t row1, uint8_t *d_bits, cudaStream_t stream);

/* ---------------------------------------------------------------- conventional baseline */

/* The conventional method the paper compares against (N-LUT), on the GPU:
 * the quantised direct sum of Eq.(1) by stamping the same (untransformed) PSF tables,
 * u(X, Y) = sum_j a_j f_{iz_j}(X - ix_j, Y - iy_j) -- WASABI without the shrinkage.  It is the
 * reference for the PSNR of the C5 sweep (reading R-A18) and the same-box speed-up baseline.
 * Dense tables: one (2H_d)^2 complex64 table per depth (caller-owned buffer). */
wasabi_status wasabi_psf_dense_bytes(const wasabi_params *params, size_t *bytes);
wasabi_status wasabi_build_psf_dense(const wasabi_params *params, void *d_dense, size_t bytes, cudaStream_t stream);
/* Bins for the direct sum: as wasabi_bin_points, but a point is listed in every tile its whole PSF disc
 * (R-A2: ceil(R) per axis, squared distance ceil(R^2)) reaches, not only the tiles its kept coefficients
 * reach (R-A19) -- the conventional method stamps the unshrunk PSF.  Standard parameters only (no
 * EXACT_SHIFT / COIFLET: EINVAL).  Same buffer size query (wasabi_bin_points_bytes). */
wasabi_status wasabi_bin_points_psf(const wasabi_params *params, const void *d_tables, const float *d_points,
                                    int64_t n, int64_t row0, int64_t row1, void *d_bins, size_t bin_bytes,
                                    cudaStream_t stream);
/* d_bins from wasabi_bin_points_psf (or wasabi_bin_points: then only the kept coefficients' reach is
 * covered) for the same band; d_u: (row1 - row0) x n_h complex64, overwritten. */
wasabi_status wasabi_direct_sum(const wasabi_params *params, const void *d_dense, const void *d_bins, int64_t row0,
                                int64_t row1, float *d_u, cudaStream_t stream);

/* The EXACT Eq.(1) on the GPU -- "D1": u(X, Y) = sum_j a_j exp(i k r_j) with the continuous
 * (x_j, y_j, z_j) (no position or depth quantisation), r_j = sqrt((x - x_j)^2 + (y - y_j)^2 + z_j^2), over
 * the diffraction-limited window rho < |z_j| tan(asin(lambda/2p)) (+ the rho = 0 pixel; R-A2 at the
 * point's own depth).  The window test and r_j in fp64 (the oracle's operation sequence), the phase as the
 * fp64 quarter-cycle count 4 r_j / lambda with (cos, sin) of its fraction in fp32 (< 1e-7), fp32
 * accumulation in point order.  The PSNR reference of the C5 sweep (R-A18).  d_points: the original
 * n x 4 float32 points; d_bins from wasabi_bin_points_psf for the same band and points (its reach
 * covers a point anywhere within half a depth level of its level, i.e. every point the bins accept;
 * points the bins skip -- R-A17 -- do not contribute).  d_u: (row1 - row0) x n_h complex64, overwritten. */
wasabi_status wasabi_direct_exact(const wasabi_params *params, const float *d_points, int64_t n, const void *d_bins,
                                  int64_t row0, int64_t row1, float *d_u, cudaStream_t stream);

/* ---------------------------------------------------------------- work accounting (not the hot path) */

/* The exact number of Eq.(2) accumulations whose target lies in the hologram
 * and in rows [row0, row1): sum over valid points j of the kept coefficients (l, X, Y) of the point's
 * table with (s_l(ix_j) + X - H, s_l(iy_j) + Y - H) inside (R-A8; R-A20 shifts in exact mode) --
 * the work a band's superposition does (4 fp32 flops each).  d_scratch: >= 8 bytes of device
 * memory.  SYNCHRONOUS (one 8-byte device->host read); one warp per point walks its kept list. */
wasabi_status wasabi_count_accumulations(const wasabi_params *params, const void *d_tables, const float *d_points,
                                        int64_t n, int64_t row0, int64_t row1, void *d_scratch, int64_t *h_count,
                                        cudaStream_t stream);

/* Per-row work estimate for work-balanced row bands (PAPER.md:115-125 sub-holograms):
 * every valid point's in-hologram accumulation count, spread uniformly over its reach rows
 * [iy - Ek, iy + Ek] (R-A19) and clipped to the hologram.  d_row_work: n_h + 1 doubles (device);
 * on completion d_row_work[Y] (Y < n_h) is the estimated work of row Y (entry n_h is scratch).
 * d_scratch >= 8 bytes.  Asynchronous. */
wasabi_status wasabi_row_work(const wasabi_params *params, const void *d_tables, const float *d_points, int64_t n,
                              double *d_row_work, void *d_scratch, cudaStream_t stream);

/* ---------------------------------------------------------------- whole path, host buffers */

/* Device workspace for wasabi_hologram_host (tables + scratch + points + bins + field). */
wasabi_status wasabi_hologram_workspace_bytes(const wasabi_params *params, int64_t n, int64_t row0,
                                              int64_t row1, size_t *workspace_bytes);

/* Whole hot path from HOST buffers: H2D copy of h_points (n x 4 float32), steps 1-4 for band
 * [row0, row1) (steps 2b-4 through wasabi_superpose_inverse), D2H copy of the bits (h_bits, (row1-row0) x n_h/8 bytes) and, if h_u != NULL,
 * of u ((row1-row0) x n_h complex64).  Host buffers should be pinned for asynchronous copies.
 * WASABI_FLAG_COIFLET: psi on the halo band (wasabi_superpose), then wasabi_inverse_wt -- fused tiles
 * when h_u == NULL (print only), the in-place line passes when u is wanted (u = the band rows of psi).
 * Returns after enqueueing; the caller synchronises `stream` before reading h_bits / h_u. */
wasabi_status wasabi_hologram_host(const wasabi_params *params, const wasabi_print_params *print,
                                   const float *h_points, int64_t n, int64_t row0, int64_t row1,
                                   void *d_workspace, size_t workspace_bytes, uint8_t *h_bits, float *h_u,
                                   cudaStream_t stream);

/* ---------------------------------------------------------------- diagnostics (synchronous) */

/* Verify that d_tables was built with these params (header magic + parameter hash). */
wasabi_status wasabi_tables_check(const wasabi_params *params, const void *d_tables);

/* Export the kept coefficients of one depth in canonical (level, Y, X) order (R-A5): level l
 * (LL counts as level L), dX = X - H_d, dY = Y - H_d, value (re, im) float32.  Host arrays of
 * capacity cap; *n_out = N_r,d (ENOSPC if cap is smaller). */
wasabi_status wasabi_export_table(const wasabi_params *params, const void *d_tables, int32_t depth,
                                  int32_t *h_level, int32_t *h_dx, int32_t *h_dy, float *h_val, int64_t cap,
                                  int64_t *n_out);

/* Export the footprint reach of one depth computed by the table build (reading R-A19): over the
 * kept coefficients (level l, dX, dY) with h = 2^(l-1), *h_ek = max(max(|dX|, |dY|) + h) and
 * *h_q = max((|dX| + h)^2 + (|dY| + h)^2).  Step 2a lists a point in a tile iff the tile meets
 * [ix +- ek] x [iy +- ek] and its pixel nearest to (ix, iy) is within squared distance q.
 * Synchronous device->host read. */
wasabi_status wasabi_export_reach(const wasabi_params *params, const void *d_tables, int32_t depth, int32_t *h_ek,
                                  int32_t *h_q);

/* Export bins: h_tile_ptr (n_tiles + 1, tiles row-major within the band) and h_point_idx
 * (cap entries); *n_out = total entries (ENOSPC if cap is smaller). */
wasabi_status wasabi_export_bins(const wasabi_params *params, const void *d_bins, int64_t *h_tile_ptr,
                                 int32_t *h_point_idx, int64_t cap, int64_t *n_out);

/* Bin statistics: out[0] valid points, out[1] skipped points, out[2] bin entries, out[3] bin
 * capacity, out[4] row0, out[5] row1, out[6] number of tiles, out[7] status (0 = ok). */
wasabi_status wasabi_bins_stats(const void *d_bins, int64_t out[8]);

/* Thread-local message for the last non-OK status of this thread ("" if none). */
const char *wasabi_last_error(void);

/* Number of CUDA kernels this library has launched in this process (diagnostic counter). */
unsigned long long wasabi_kernel_launches(void);

/* Library version string. */
const char *wasabi_version(void);

#ifdef __cplusplus
}
#endif

#endif /* WASABI_H */
