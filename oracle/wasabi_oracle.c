/*
 * wasabi_oracle.c -- plain, slow, fp64 CPU oracle for the WASABI hot path of
 * arXiv 1708.04233 ("Fast, large-scale hologram calculation in wavelet domain").
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library.  It shares no code,
 * header, table or constant with the CUDA path (paper_1708_04233_b200/csrc).
 * Build: gcc -O2 -ffp-contract=off -fPIC -shared (no fast-math, no FMA contraction).
 *
 * Every function follows the paper (PAPER.md line numbers, section, equation)
 * in the paper's order, with the readings listed in DESIGN.md §2 ("R-xx") where
 * the paper is silent, ambiguous or garbled:
 *   R-A1  Haar (orthonormal, 1/2 per 2-D level) instead of coiflets (north_star)
 *   R-A2  PSF window radius rho_max = |z| tan(asin(lambda/2p)), S = {dx^2+dy^2 < R^2} U {(0,0)}
 *   R-A3  depth levels z_d = z_min + d (z_max-z_min)/(N_z-1), nearest, ties to lower
 *   R-A4  N_r,d = min(nnz_d, ceil(r_ppm nnz_d / 1e6)), nnz_d structural
 *   R-A5  one joint ranking over all levels and subbands incl. LL, by |c|
 *   R-A6  interleaved in-place Haar layout (Fig. 2(a) missing)
 *   R-A8  per-level shift s_l = 2^l floor((ix + 2^(l-1)) / 2^l) ("alpha")
 *   R-A9  ix = floor(x/p + 1/2) + N_h/2 (hologram-centred origin)
 *   R-A11 bins in ascending point order; accumulation point-major, entry canonical order
 *   R-A12 coefficients outside the hologram / band / window are dropped
 *   R-A13 rank key kappa = fp32_RN(re^2+im^2), ties to the smaller linear index
 *   R-A14 bit = Re(u conj(R)) >= 0
 *   R-A15 R = exp(+i k sqrt((x-xr)^2+(y-yr)^2+zr^2))
 *   R-A17 a <= 0, non-finite, or z beyond half a level outside the range: skipped
 *
 * Parity pins (tests/test_oracle_*.py) pin every function here to closed forms,
 * invariants, brute force, or the paper's printed parameters; see DESIGN.md §4.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_PI 3.14159265358979323846

typedef struct {
    double wavelength;   /* lambda [m] (Eq.(1)) */
    double pitch;        /* p [m], hologram sampling pitch */
    int64_t n_h;         /* N_h, hologram side in pixels */
    int32_t n_depth;     /* N_z */
    int32_t levels;      /* L, wavelet levels (Haar here) */
    double z_min, z_max; /* depth range [m] */
    double retention;    /* r in (0,1] (north_star "top-r%") */
    int32_t exact;       /* 1: exact off-grid shifts via offset-class tables */
    int32_t wavelet;     /* 0: Haar (R-A1); 1: coif1, the paper's coiflets (NEXT-2, R-A21) */
} orc_params;

/* R-A20 (NEXT-4): with exact = 1 every depth has 4^L tables, one per sub-position class
 * (cx, cy) = (ix mod 2^L, iy mod 2^L); table t = d 4^L + cy 2^L + cx holds the PSF centred at
 * (H + cx, H + cy) in a (2H + 2^L)^2 table, and a point's coefficients of every level are shifted
 * by the 2^L-aligned s = (ix - cx, iy - cy), so WASABI at r = 100% equals the quantised direct sum
 * for any integer position.  exact = 0: one table per depth (t = d), centre (H, H), side 2H. */
static int orc_cls_bits(const orc_params *P) { return P->exact ? P->levels : 0; }
int64_t orc_n_tables(const orc_params *P) { return (int64_t)P->n_depth << (2 * orc_cls_bits(P)); }
static int orc_table_depth(const orc_params *P, int64_t t) { return (int)(t >> (2 * orc_cls_bits(P))); }
static int64_t orc_table_cx(const orc_params *P, int64_t t) { return t & (((int64_t)1 << orc_cls_bits(P)) - 1); }
static int64_t orc_table_cy(const orc_params *P, int64_t t) {
    return (t >> orc_cls_bits(P)) & (((int64_t)1 << orc_cls_bits(P)) - 1);
}

/* ---------------------------------------------------------------- geometry */

/* PAPER.md:90 PSF radius.  R-A2: maximum diffraction angle sin(theta) = lambda/(2p). */
static double orc_tan_theta(const orc_params *P) {
    double sigma = P->wavelength / (2.0 * P->pitch);
    return sigma / sqrt(1.0 - sigma * sigma);
}

/* PAPER.md:91 depth discretisation; R-A3: inclusive endpoints. */
static double orc_level_z(const orc_params *P, int d) {
    if (P->n_depth <= 1) return P->z_min;
    double dz = (P->z_max - P->z_min) / (double)(P->n_depth - 1);
    return P->z_min + (double)d * dz;
}

/* R_d in pixels (R-A2). */
static double orc_radius_px(const orc_params *P, double z) {
    return fabs(z) * orc_tan_theta(P) / P->pitch;
}

/* Table half side H_d = 2^L (floor(R/2^L) + 1): table side 2H holds the disc and is 2^L aligned.
 * Coiflets (R-A21): the coefficients of a disc spread up to 3 (2^L - 1) px beyond it, so the table
 * is padded: H = 2^L (floor((R + 3 2^L)/2^L) + 1) holds every nonzero coefficient exactly. */
static int64_t orc_half(const orc_params *P, double R) {
    int64_t B = (int64_t)1 << P->levels;
    double pad = P->wavelet == 1 ? 3.0 * (double)B : 0.0;
    return B * ((int64_t)floor((R + pad) / (double)B) + 1);
}

/* S_d membership: circ(c) = 1 iff c < 1, centre always kept (R-A17). */
static int orc_in_support(int64_t dx, int64_t dy, double R) {
    if (dx == 0 && dy == 0) return 1;
    return (double)(dx * dx + dy * dy) < R * R;
}

/* Structural nnz_d (R-A4): number of coefficient positions whose support block touches S_d.
 * Brute force over the mask: level-l detail coefficients (3 per 2^l block) and level-L
 * scaling coefficients (1 per 2^L block). */
static int64_t orc_nnz_fb(const orc_params *P, int64_t side, int64_t Cx, int64_t Cy, double R);
static int64_t orc_nnz_c(const orc_params *P, int64_t side, int64_t Cx, int64_t Cy, double R) {
    if (P->wavelet == 1) return orc_nnz_fb(P, side, Cx, Cy, R);
    int64_t nnz = 0;
    unsigned char *m = (unsigned char *)calloc((size_t)(side * side), 1);
    for (int64_t Y = 0; Y < side; Y++)
        for (int64_t X = 0; X < side; X++) m[Y * side + X] = (unsigned char)orc_in_support(X - Cx, Y - Cy, R);
    for (int l = 1; l <= P->levels; l++) {
        int64_t b = (int64_t)1 << l;
        for (int64_t Y0 = 0; Y0 < side; Y0 += b)
            for (int64_t X0 = 0; X0 < side; X0 += b) {
                int touch = 0;
                for (int64_t y = Y0; y < Y0 + b && !touch; y++)
                    for (int64_t x = X0; x < X0 + b; x++)
                        if (m[y * side + x]) { touch = 1; break; }
                if (touch) nnz += (l == P->levels) ? 4 : 3;
            }
    }
    free(m);
    return nnz;
}
static int64_t orc_nnz(const orc_params *P, int64_t H, double R) { return orc_nnz_c(P, 2 * H, H, H, R); }

/* Footprint E (reading R-A19's structural bound): a kept coefficient of a point lies within E px
 * per axis: ceil(R) + 3 2^(L-1) for Haar; coiflet tables spread 3 2^L further (R-A21). */
static int64_t orc_footprint(const orc_params *P, double R) {
    return (int64_t)ceil(R) + (P->wavelet == 1 ? 7 : 3) * ((int64_t)1 << (P->levels - 1));
}

/* Table t geometry (R-A20): depth, H, side, PSF centre (Cx, Cy). */
static void orc_table_geom(const orc_params *P, int64_t t, int *d, double *R, int64_t *H, int64_t *side,
                           int64_t *Cx, int64_t *Cy) {
    *d = orc_table_depth(P, t);
    *R = orc_radius_px(P, orc_level_z(P, *d));
    *H = orc_half(P, *R);
    *side = 2 * *H + (P->exact ? ((int64_t)1 << P->levels) : 0);
    *Cx = *H + orc_table_cx(P, t);
    *Cy = *H + orc_table_cy(P, t);
}


/* R-A4: N_r,d = min(nnz, ceil(r_ppm * nnz / 1e6)), r_ppm = llround(r * 1e6). */
static int64_t orc_n_r(const orc_params *P, int64_t nnz) {
    int64_t r_ppm = llround(P->retention * 1e6);
    int64_t n = (r_ppm * nnz + 999999) / 1000000;
    return n < nnz ? n : nnz;
}

/* Geometry of table t: hsn = {H, side, nnz, N_r}. */
int orc_table_info(const orc_params *P, int64_t t, int64_t *hsn) {
    int d; double R; int64_t H, side, Cx, Cy;
    orc_table_geom(P, t, &d, &R, &H, &side, &Cx, &Cy);
    int64_t c = orc_nnz_c(P, side, Cx, Cy, R);
    hsn[0] = H; hsn[1] = side; hsn[2] = c; hsn[3] = orc_n_r(P, c);
    return 0;
}

/* Per-depth geometry.  E_d = ceil(R_d) + 3*2^(L-1) is the footprint half-size (bins). */
int orc_geometry(const orc_params *P, double *z, double *R, int64_t *H, int64_t *E, int64_t *nnz,
                 int64_t *n_r) {
    for (int d = 0; d < P->n_depth; d++) {
        double zd = orc_level_z(P, d);
        double Rd = orc_radius_px(P, zd);
        int64_t Hd = orc_half(P, Rd);
        if (z) z[d] = zd;
        if (R) R[d] = Rd;
        if (H) H[d] = Hd;
        if (E) E[d] = orc_footprint(P, Rd);
        if (nnz || n_r) {
            int64_t c = orc_nnz(P, Hd, Rd);
            if (nnz) nnz[d] = c;
            if (n_r) n_r[d] = orc_n_r(P, c);
        }
    }
    return 0;
}

/* Geometry of one depth: zr = {z_d, R_d}, hen = {H_d, E_d, nnz_d, N_r,d}. */
int orc_depth_info(const orc_params *P, int d, double *zr, int64_t *hen) {
    double zd = orc_level_z(P, d), Rd = orc_radius_px(P, zd);
    int64_t Hd = orc_half(P, Rd), c = orc_nnz(P, Hd, Rd);
    zr[0] = zd; zr[1] = Rd;
    hen[0] = Hd; hen[1] = orc_footprint(P, Rd);
    hen[2] = c; hen[3] = orc_n_r(P, c);
    return 0;
}

/* ---------------------------------------------------------------- PSF (step 1) */

/* u_z = exp(i k r) circ(.), unit amplitude (Eq.(1) carries only a_j).
 * Table t (R-A20): side 2H (+ 2^L in exact mode), centre (Cx, Cy); f interleaved (re, im) row-major. */
int orc_psf_table(const orc_params *P, int64_t t, double *f) {
    int d; double R; int64_t H, side, Cx, Cy;
    orc_table_geom(P, t, &d, &R, &H, &side, &Cx, &Cy);
    double z = orc_level_z(P, d);
    double k = 2.0 * ORC_PI / P->wavelength;
    for (int64_t Y = 0; Y < side; Y++)
        for (int64_t X = 0; X < side; X++) {
            int64_t dx = X - Cx, dy = Y - Cy;
            double *o = f + 2 * (Y * side + X);
            if (!orc_in_support(dx, dy, R)) { o[0] = 0.0; o[1] = 0.0; continue; }
            double xp = (double)dx * P->pitch, yp = (double)dy * P->pitch;
            double r = sqrt((xp * xp + yp * yp) + z * z);   /* r_hj */
            double ph = k * r;
            o[0] = cos(ph);
            o[1] = sin(ph);
        }
    return 0;
}

/* ---------------------------------------------------------------- filter banks (R-A21) */

/* R-A21: "we used coiflets as the wavelets at level 3".
 * The order is not given; coif1 (the shortest coiflet, 6 taps) in closed form (Daubechies'
 * K = 1 coiflet):  h0 = sqrt(2)/32 [1-s, 5+s, 14+2s, 14-2s, 1-s, -3+s], s = sqrt(7), with
 * h1[k] = (-1)^k h0[5-k].  Convention on the infinite grid (zero extension):
 *   analysis  a[m] = sum_k h0[k] x[2m + k - off],  d[m] = sum_k h1[k] x[2m + k - off]
 *   synthesis x[n] = sum_m h0[n - 2m + off] a[m] + h1[n - 2m + off] d[m]
 * with off = 2 for coif1 (the filter's first moment about k = 2 vanishes, so a[m] samples
 * x near 2m) and off = 0 for Haar (h0 = [1, 1]/sqrt2, h1 = [1, -1]/sqrt2), which reproduces the
 * R-A6 butterflies.  Interleaved layout (R-A6): a level-l step works on the samples at multiples of
 * 2^(l-1); a[m] goes to sample 2m (position 2^l m), d[m] to sample 2m + 1. */
typedef struct { int taps, off; double h0[6], h1[6]; } orc_fb;

static void orc_filters(int wavelet, orc_fb *F) {
    memset(F, 0, sizeof *F);
    if (wavelet == 1) {
        double s7 = sqrt(7.0), c = sqrt(2.0) / 32.0;
        double v[6] = {1.0 - s7, 5.0 + s7, 14.0 + 2.0 * s7, 14.0 - 2.0 * s7, 1.0 - s7, -3.0 + s7};
        F->taps = 6; F->off = 2;
        for (int k = 0; k < 6; k++) F->h0[k] = v[k] * c;
    } else {
        F->taps = 2; F->off = 0;
        F->h0[0] = F->h0[1] = 1.0 / sqrt(2.0);
    }
    for (int k = 0; k < F->taps; k++) F->h1[k] = ((k & 1) ? -1.0 : 1.0) * F->h0[F->taps - 1 - k];
}

/* Filters of a wavelet (for the filter pins): h0, h1 (6 each, zero padded), returns taps; off out. */
int orc_filter_bank(int wavelet, double *h0, double *h1, int *off) {
    orc_fb F;
    orc_filters(wavelet, &F);
    for (int k = 0; k < 6; k++) { h0[k] = F.h0[k]; h1[k] = F.h1[k]; }
    *off = F.off;
    return F.taps;
}

/* One analysis (dir = +1) or synthesis (dir = -1) step along a line of N complex samples, sample n at
 * f + 2 n st; N even.  Zero extension beyond [0, N).  Sums in tap order k = 0..taps-1. */
static void orc_fb_line(const orc_fb *F, double *f, int64_t st, int64_t N, int dir, double *tmp) {
    for (int64_t n = 0; n < N; n++) { tmp[2 * n] = f[2 * n * st]; tmp[2 * n + 1] = f[2 * n * st + 1]; }
    if (dir > 0) {
        for (int64_t m = 0; m < N / 2; m++)
            for (int c = 0; c < 2; c++) {
                double a = 0.0, d = 0.0;
                for (int k = 0; k < F->taps; k++) {
                    int64_t i = 2 * m + k - F->off;
                    if (i < 0 || i >= N) continue;
                    a += F->h0[k] * tmp[2 * i + c];
                    d += F->h1[k] * tmp[2 * i + c];
                }
                f[2 * (2 * m) * st + c] = a;
                f[2 * (2 * m + 1) * st + c] = d;
            }
    } else {
        for (int64_t n = 0; n < N; n++)
            for (int c = 0; c < 2; c++) {
                double x = 0.0;
                /* k = n - 2m + off in [0, taps): m from (n + off)/2 down to (n + off - taps + 1)/2 */
                int64_t m_hi = (n + F->off) / 2, m_lo = m_hi - F->taps / 2 - 1;
                for (int64_t m = m_lo; m <= m_hi; m++) {
                    int64_t k = n - 2 * m + F->off;
                    if (m < 0 || m >= N / 2 || k < 0 || k >= F->taps) continue;
                    x += F->h0[k] * tmp[2 * (2 * m) + c];
                    x += F->h1[k] * tmp[2 * (2 * m + 1) + c];
                }
                f[2 * n * st + c] = x;
            }
    }
}

/* L-level 2-D forward (rows, then columns, per level) / inverse (columns, then rows, levels L..1)
 * of a rows x cols interleaved complex array (row stride `stride`), zero extension. */
void orc_fb_fwd(int wavelet, double *f, int64_t rows, int64_t cols, int64_t stride, int L) {
    orc_fb F;
    orc_filters(wavelet, &F);
    double *tmp = (double *)malloc(sizeof(double) * 2 * (size_t)(rows > cols ? rows : cols));
    for (int l = 1; l <= L; l++) {
        int64_t s = (int64_t)1 << (l - 1);
        for (int64_t Y = 0; Y < rows; Y += s) orc_fb_line(&F, f + 2 * (Y * stride), s, cols / s, +1, tmp);
        for (int64_t X = 0; X < cols; X += s) orc_fb_line(&F, f + 2 * X, s * stride, rows / s, +1, tmp);
    }
    free(tmp);
}

void orc_fb_inv(int wavelet, double *f, int64_t rows, int64_t cols, int64_t stride, int L) {
    orc_fb F;
    orc_filters(wavelet, &F);
    double *tmp = (double *)malloc(sizeof(double) * 2 * (size_t)(rows > cols ? rows : cols));
    for (int l = L; l >= 1; l--) {
        int64_t s = (int64_t)1 << (l - 1);
        for (int64_t X = 0; X < cols; X += s) orc_fb_line(&F, f + 2 * X, s * stride, rows / s, -1, tmp);
        for (int64_t Y = 0; Y < rows; Y += s) orc_fb_line(&F, f + 2 * (Y * stride), s, cols / s, -1, tmp);
    }
    free(tmp);
}

/* ---------------------------------------------------------------- Haar (steps 1, 3) */

/* Forward FWT, R-A1/R-A6: level l = 1..L on every 2^l-aligned block, in place:
 *   LL=((a+b)+(c+d))/2 at (X0,Y0), HL=((a-b)+(c-d))/2 at (X0+s,Y0),
 *   LH=((a+b)-(c+d))/2 at (X0,Y0+s), HH=((a-b)-(c-d))/2 at (X0+s,Y0+s), s = 2^(l-1).
 * f interleaved complex, row-major with row stride `stride` complex elements. */
void orc_haar_fwd(double *f, int64_t rows, int64_t cols, int64_t stride, int L) {
    for (int l = 1; l <= L; l++) {
        int64_t b = (int64_t)1 << l, s = b >> 1;
        for (int64_t Y0 = 0; Y0 < rows; Y0 += b)
            for (int64_t X0 = 0; X0 < cols; X0 += b)
                for (int c = 0; c < 2; c++) {
                    double *pa = f + 2 * (Y0 * stride + X0) + c;
                    double *pb = f + 2 * (Y0 * stride + X0 + s) + c;
                    double *pc = f + 2 * ((Y0 + s) * stride + X0) + c;
                    double *pd = f + 2 * ((Y0 + s) * stride + X0 + s) + c;
                    double a = *pa, bb = *pb, cc = *pc, dd = *pd;
                    *pa = ((a + bb) + (cc + dd)) / 2.0;
                    *pb = ((a - bb) + (cc - dd)) / 2.0;
                    *pc = ((a + bb) - (cc + dd)) / 2.0;
                    *pd = ((a - bb) - (cc - dd)) / 2.0;
                }
    }
}

/* Inverse FWT (PAPER.md:94 step 3, :123): l = L..1,
 *   a=((LL+HL)+(LH+HH))/2, b=((LL-HL)+(LH-HH))/2, c=((LL+HL)-(LH+HH))/2, d=((LL-HL)-(LH-HH))/2. */
void orc_haar_inv(double *f, int64_t rows, int64_t cols, int64_t stride, int L) {
    for (int l = L; l >= 1; l--) {
        int64_t b = (int64_t)1 << l, s = b >> 1;
        for (int64_t Y0 = 0; Y0 < rows; Y0 += b)
            for (int64_t X0 = 0; X0 < cols; X0 += b)
                for (int c = 0; c < 2; c++) {
                    double *pa = f + 2 * (Y0 * stride + X0) + c;
                    double *pb = f + 2 * (Y0 * stride + X0 + s) + c;
                    double *pc = f + 2 * ((Y0 + s) * stride + X0) + c;
                    double *pd = f + 2 * ((Y0 + s) * stride + X0 + s) + c;
                    double LL = *pa, HL = *pb, LH = *pc, HH = *pd;
                    *pa = ((LL + HL) + (LH + HH)) / 2.0;
                    *pb = ((LL - HL) + (LH - HH)) / 2.0;
                    *pc = ((LL + HL) - (LH + HH)) / 2.0;
                    *pd = ((LL - HL) - (LH - HH)) / 2.0;
                }
    }
}

/* Level of an interleaved position (R-A6): t = min(ctz X, ctz Y); t >= L -> LL (level L),
 * else level t+1.  Subband code: 0 LL, 1 HL, 2 LH, 3 HH. */
static void orc_classify(int64_t X, int64_t Y, int L, int *level, int *band) {
    int t = 0;
    while (t < L && ((X >> t) & 1) == 0 && ((Y >> t) & 1) == 0) t++;
    if (t >= L) { *level = L; *band = 0; return; }
    *level = t + 1;
    *band = (int)(((X >> t) & 1) | (((Y >> t) & 1) << 1));
}

/* ---------------------------------------------------------------- selection (step 1) */

typedef struct { float kappa; int64_t lin; } orc_key;

static int orc_key_cmp(const void *a, const void *b) {
    const orc_key *x = (const orc_key *)a, *y = (const orc_key *)b;
    if (x->kappa > y->kappa) return -1;       /* larger magnitude first */
    if (x->kappa < y->kappa) return 1;
    return (x->lin < y->lin) ? -1 : (x->lin > y->lin);   /* R-A13 tie-break */
}

typedef struct { int level; int64_t X, Y; } orc_pos;
static int orc_canon_cmp(const void *a, const void *b) {
    const orc_pos *x = (const orc_pos *)a, *y = (const orc_pos *)b;
    if (x->level != y->level) return x->level - y->level;
    if (x->Y != y->Y) return (x->Y < y->Y) ? -1 : 1;
    return (x->X < y->X) ? -1 : (x->X > y->X);
}

/* Full transformed table of depth d (for invariant tests).  coef: (2H)^2 interleaved complex. */
int orc_table_coeffs(const orc_params *P, int64_t t, double *coef) {
    int d; double R; int64_t H, side, Cx, Cy;
    orc_table_geom(P, t, &d, &R, &H, &side, &Cx, &Cy);
    orc_psf_table(P, t, coef);
    if (P->wavelet == 1) orc_fb_fwd(1, coef, side, side, side, P->levels);   /* coif1, R-A21 */
    else orc_haar_fwd(coef, side, side, side, P->levels);
    return 0;
}

/* Structural nnz of a filter-bank transform (R-A21; with Haar filters it equals the block count):
 * the coefficient of level l at index (m, n) = (X >> l, Y >> l) depends on the input rectangle
 * [2^l m - off (2^l - 1), 2^l m + (taps - 1 - off)(2^l - 1)] (same in Y); it can be nonzero iff the
 * rectangle meets S_d, i.e. iff the rectangle's lattice point nearest to the centre is in S_d. */
static int64_t orc_nnz_fb(const orc_params *P, int64_t side, int64_t Cx, int64_t Cy, double R) {
    orc_fb F;
    orc_filters(P->wavelet, &F);
    int64_t nnz = 0;
    for (int64_t Y = 0; Y < side; Y++)
        for (int64_t X = 0; X < side; X++) {
            int lv, bd;
            orc_classify(X, Y, P->levels, &lv, &bd);
            int64_t b = (int64_t)1 << lv, mx = X >> lv, my = Y >> lv;
            int64_t x0 = b * mx - F.off * (b - 1), x1 = b * mx + (F.taps - 1 - F.off) * (b - 1);
            int64_t y0 = b * my - F.off * (b - 1), y1 = b * my + (F.taps - 1 - F.off) * (b - 1);
            int64_t nx = Cx < x0 ? x0 : (Cx > x1 ? x1 : Cx), ny = Cy < y0 ? y0 : (Cy > y1 ? y1 : Cy);
            if (orc_in_support(nx - Cx, ny - Cy, R)) nnz++;
        }
    return nnz;
}

/* Structural nnz by the filter-bank footprint rule for any wavelet (pin: Haar == block count). */
int64_t orc_nnz_footprint(const orc_params *P, int64_t t) {
    int d; double R; int64_t H, side, Cx, Cy;
    orc_table_geom(P, t, &d, &R, &H, &side, &Cx, &Cy);
    return orc_nnz_fb(P, side, Cx, Cy, R);
}

/* PAPER.md:92 "select N_r strong coefficients among the wavelet-domain PSF and store them in
 * the LUT".  Full sort of all side^2 positions of table t by (kappa desc, linear index asc)
 * (R-A13, R-A5), first N_r kept, then re-sorted canonically by (level, Y, X).  Outputs level,
 * dx = X - H, dy = Y - H (offsets from the 2^L-aligned table centre (H, H)), fp64 value (re, im).
 * Returns the count (N_r) or -1 if cap is too small. */
int64_t orc_select(const orc_params *P, int64_t t, int32_t *level, int32_t *dx, int32_t *dy, double *val,
                   int64_t cap) {
    int d; double R; int64_t H, side, Cx, Cy;
    orc_table_geom(P, t, &d, &R, &H, &side, &Cx, &Cy);
    int64_t n = side * side;
    int64_t nr = orc_n_r(P, orc_nnz_c(P, side, Cx, Cy, R));
    if (nr > cap) return -1;
    double *c = (double *)malloc(sizeof(double) * 2 * (size_t)n);
    orc_table_coeffs(P, t, c);
    orc_key *keys = (orc_key *)malloc(sizeof(orc_key) * (size_t)n);
    for (int64_t i = 0; i < n; i++) {
        double re = c[2 * i], im = c[2 * i + 1];
        double m2 = re * re + im * im;
        keys[i].kappa = (float)m2;         /* fp32 round-to-nearest of the fp64 |c|^2 */
        keys[i].lin = i;                   /* Y * side + X */
    }
    qsort(keys, (size_t)n, sizeof(orc_key), orc_key_cmp);
    orc_pos *sel = (orc_pos *)malloc(sizeof(orc_pos) * (size_t)(nr > 0 ? nr : 1));
    for (int64_t i = 0; i < nr; i++) {
        int lv, bd;
        sel[i].X = keys[i].lin % side;
        sel[i].Y = keys[i].lin / side;
        orc_classify(sel[i].X, sel[i].Y, P->levels, &lv, &bd);
        sel[i].level = lv;
    }
    qsort(sel, (size_t)nr, sizeof(orc_pos), orc_canon_cmp);
    for (int64_t i = 0; i < nr; i++) {
        int64_t X = sel[i].X, Y = sel[i].Y;
        level[i] = sel[i].level;
        dx[i] = (int32_t)(X - H);
        dy[i] = (int32_t)(Y - H);
        val[2 * i] = c[2 * (Y * side + X)];
        val[2 * i + 1] = c[2 * (Y * side + X) + 1];
    }
    free(sel);
    free(keys);
    free(c);
    return nr;
}

/* ---------------------------------------------------------------- LUT cache */

typedef struct {
    int built;
    int64_t n, H;
    int32_t *level, *dx, *dy;
    double *val;
} orc_depth_list;

typedef struct {
    orc_params P;
    orc_depth_list *lists;
} orc_lut;

void *orc_lut_new(const orc_params *P) {
    orc_lut *t = (orc_lut *)calloc(1, sizeof(orc_lut));
    t->P = *P;
    t->lists = (orc_depth_list *)calloc((size_t)orc_n_tables(P), sizeof(orc_depth_list));
    return t;
}

void orc_lut_free(void *h) {
    orc_lut *t = (orc_lut *)h;
    if (!t) return;
    for (int64_t d = 0; d < orc_n_tables(&t->P); d++) {
        free(t->lists[d].level); free(t->lists[d].dx); free(t->lists[d].dy); free(t->lists[d].val);
    }
    free(t->lists);
    free(t);
}

static orc_depth_list *orc_lut_get(orc_lut *t, int64_t d) {
    orc_depth_list *L = &t->lists[d];
    if (L->built) return L;
    const orc_params *P = &t->P;
    int dd; double R; int64_t side, Cx, Cy;
    orc_table_geom(P, d, &dd, &R, &L->H, &side, &Cx, &Cy);
    int64_t cap = orc_n_r(P, orc_nnz_c(P, side, Cx, Cy, R));
    L->level = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap + 1));
    L->dx = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap + 1));
    L->dy = (int32_t *)malloc(sizeof(int32_t) * (size_t)(cap + 1));
    L->val = (double *)malloc(sizeof(double) * 2 * (size_t)(cap + 1));
    L->n = orc_select(P, d, L->level, L->dx, L->dy, L->val, cap);
    L->built = 1;
    return L;
}

/* Build (force) the list of depth d in the cache; returns N_r,d. */
int64_t orc_lut_build_depth(void *h, int64_t d) { return orc_lut_get((orc_lut *)h, d)->n; }

/* Table of a point (R-A20): t = iz in the standard mode, iz 4^L + (iy mod 2^L) 2^L + (ix mod 2^L)
 * in the exact mode. */
static int64_t orc_point_table(const orc_params *P, int64_t ix, int64_t iy, int iz) {
    int b = orc_cls_bits(P);
    int64_t m = ((int64_t)1 << b) - 1;
    return ((int64_t)iz << (2 * b)) | ((iy & m) << b) | (ix & m);
}

/* Coefficient shift of a point (R-A8 standard, R-A20 exact): level-l target = s + (dX, dY). */
static int64_t orc_shift(const orc_params *P, int64_t i, int l) {
    if (P->exact) {
        int64_t B = (int64_t)1 << P->levels;
        return i - (i & (B - 1));
    }
    int64_t b = (int64_t)1 << l;
    int64_t q = (i + (b >> 1)) / b;
    if (((i + (b >> 1)) % b != 0) && (i + (b >> 1) < 0)) q--;
    return b * q;
}

/* Exported for the R-A8 pins (tests/test_oracle_shift.py): the level-l coefficient shift of
 * pixel index i (orc_shift). */
int64_t orc_level_shift(const orc_params *P, int64_t i, int l) { return orc_shift(P, i, l); }

/* Reach of table d's kept list (reading R-A19; exact mode R-A20: no rounding term).  A level-l entry (dX, dY) of a point at (ix, iy)
 * lands at (s_l(ix) + dX, s_l(iy) + dY) (R-A8), and s_l(i) - i lies in (-2^(l-1), 2^(l-1)], so
 * with h = 2^(l-1) the target is within |dX| + h of ix and |dY| + h of iy.  Over the kept list:
 *   ek = max max(|dX|, |dY|) + h        (square bound)
 *   q  = max (|dX| + h)^2 + (|dY| + h)^2  (squared-distance bound)
 * The LL entries carry level L. */
void orc_lut_reach(void *h, int64_t d, int64_t *ek, int64_t *q) {
    orc_lut *t = (orc_lut *)h;
    orc_depth_list *L = orc_lut_get(t, d);
    int64_t e = 0, qq = 0;
    int64_t cx = orc_table_cx(&t->P, d), cy = orc_table_cy(&t->P, d);
    for (int64_t k = 0; k < L->n; k++) {
        int64_t ax, ay;
        if (t->P.exact) {   /* R-A20: the offset from the point is exactly (dX - cx, dY - cy) */
            ax = llabs((long long)(L->dx[k] - cx)); ay = llabs((long long)(L->dy[k] - cy));
        } else {
            int64_t hl = (int64_t)1 << (L->level[k] - 1);
            ax = llabs((long long)L->dx[k]) + hl; ay = llabs((long long)L->dy[k]) + hl;
        }
        if (ax > e) e = ax;
        if (ay > e) e = ay;
        if (ax * ax + ay * ay > qq) qq = ax * ax + ay * ay;
    }
    *ek = e;
    *q = qq;
}

/* ---------------------------------------------------------------- points (step 2a) */

/* R-A9 / R-A3 / R-A17: point -> (ix, iy, iz), valid flag.  pts is (n, 4) fp64 (x, y, z, a). */
static int orc_point(const orc_params *P, const double *pt, int64_t *ix, int64_t *iy, int *iz) {
    double x = pt[0], y = pt[1], z = pt[2], a = pt[3];
    if (!isfinite(x) || !isfinite(y) || !isfinite(z) || !isfinite(a) || !(a > 0.0)) return 0;
    double u = x / P->pitch, v = y / P->pitch;
    if (!(fabs(u) <= 1073741824.0) || !(fabs(v) <= 1073741824.0)) return 0;
    *ix = (int64_t)floor(u + 0.5) + P->n_h / 2;
    *iy = (int64_t)floor(v + 0.5) + P->n_h / 2;
    if (P->n_depth <= 1) { *iz = 0; return 1; }
    double dz = (P->z_max - P->z_min) / (double)(P->n_depth - 1);
    double t = (z - P->z_min) / dz;
    if (t < -0.5 || t > (double)(P->n_depth - 1) + 0.5) return 0;
    int64_t q = (int64_t)ceil(t - 0.5);          /* nearest level, ties to the lower index */
    if (q < 0) q = 0;
    if (q > P->n_depth - 1) q = P->n_depth - 1;
    *iz = (int)q;
    return 1;
}

int orc_points(const orc_params *P, const double *pts, int64_t n, int64_t *ix, int64_t *iy, int32_t *iz,
               int8_t *valid) {
    for (int64_t j = 0; j < n; j++) {
        int64_t a = 0, b = 0;
        int c = 0;
        valid[j] = (int8_t)orc_point(P, pts + 4 * j, &a, &b, &c);
        ix[j] = a; iy[j] = b; iz[j] = c;
    }
    return 0;
}

/* ---------------------------------------------------------------- bins (step 2a) */

/* Footprint membership (R-A12, R-A19): tile [X0, X1] x [Y0, Y1] is in the footprint of a point at
 * (ix, iy) of depth d iff it meets the square [ix - ek_d, ix + ek_d] x [iy - ek_d, iy + ek_d] and
 * its pixel nearest to (ix, iy) lies within squared distance q_d (orc_lut_reach). */
static int orc_tile_in_footprint(int64_t ix, int64_t iy, int64_t ek, int64_t q, int64_t X0, int64_t X1,
                                 int64_t Y0, int64_t Y1) {
    if (ix + ek < X0 || ix - ek > X1 || iy + ek < Y0 || iy - ek > Y1) return 0;
    int64_t ddx = 0, ddy = 0;
    if (ix < X0) ddx = X0 - ix;
    if (ix > X1) ddx = ix - X1;
    if (iy < Y0) ddy = Y0 - iy;
    if (iy > Y1) ddy = iy - Y1;
    return ddx * ddx + ddy * ddy <= q;
}

/* PAPER.md:115-122 sub-hologram re-basing, applied per T x T tile (R-A12): point j is in
 * bin(tx,ty) iff the tile is in its footprint (orc_tile_in_footprint with the reach ek[t], q[t]
 * of its table t = orc_point_table) and lies in rows [row0, row1).  Brute force over all tiles of the band, points
 * ascending.  tile_ptr has n_tiles+1 entries (tiles row-major within the band).  Returns total
 * entries, or -(needed) if cap is too small (idx untouched beyond cap). */
int64_t orc_bins(const orc_params *P, int64_t T, const double *pts, int64_t n, int64_t row0, int64_t row1,
                 const int64_t *ek, const int64_t *q, int64_t *tile_ptr, int32_t *idx, int64_t cap) {
    int64_t tiles_x = P->n_h / T, tiles_y = (row1 - row0) / T;
    int64_t *pp = (int64_t *)malloc(sizeof(int64_t) * 3 * (size_t)(n > 0 ? n : 1));
    int8_t *ok = (int8_t *)malloc((size_t)(n > 0 ? n : 1));
    for (int64_t j = 0; j < n; j++) {
        int64_t ix, iy;
        int iz;
        ok[j] = (int8_t)orc_point(P, pts + 4 * j, &ix, &iy, &iz);
        pp[3 * j + 0] = ix; pp[3 * j + 1] = iy; pp[3 * j + 2] = iz;
    }
    int64_t total = 0;
    for (int64_t ty = 0; ty < tiles_y; ty++)
        for (int64_t tx = 0; tx < tiles_x; tx++) {
            int64_t t = ty * tiles_x + tx;
            int64_t X0 = tx * T, X1 = X0 + T - 1, Y0 = row0 + ty * T, Y1 = Y0 + T - 1;
            tile_ptr[t] = total;
            for (int64_t j = 0; j < n; j++) {
                if (!ok[j]) continue;
                int64_t d = orc_point_table(P, pp[3 * j], pp[3 * j + 1], (int)pp[3 * j + 2]);
                if (!orc_tile_in_footprint(pp[3 * j], pp[3 * j + 1], ek[d], q[d], X0, X1, Y0, Y1)) continue;
                if (total < cap) idx[total] = (int32_t)j;
                total++;
            }
        }
    tile_ptr[tiles_x * tiles_y] = total;
    free(ok); free(pp);
    return total <= cap ? total : -total;
}

/* One bin by the same definition (for sampled parity at full size): points ascending whose
 * footprint contains tile [X0, X0+T) x [Y0, Y0+T) (absolute hologram rows).  Returns the count. */
int64_t orc_bin_tile(const orc_params *P, int64_t T, const double *pts, int64_t n, int64_t X0, int64_t Y0,
                     const int64_t *ek, const int64_t *q, int32_t *idx, int64_t cap) {
    int64_t total = 0;
    for (int64_t j = 0; j < n; j++) {
        int64_t ix, iy;
        int iz;
        if (!orc_point(P, pts + 4 * j, &ix, &iy, &iz)) continue;
        int64_t d = orc_point_table(P, ix, iy, iz);
        if (!orc_tile_in_footprint(ix, iy, ek[d], q[d], X0, X0 + T - 1, Y0, Y0 + T - 1)) continue;
        if (total < cap) idx[total] = (int32_t)j;
        total++;
    }
    return total;
}

/* ---------------------------------------------------------------- WASABI (steps 2b, 3) */

/* Eq.(2), with the sub-hologram re-basing of PAPER.md:121-122 replaced by a
 * window [x0, x0+w) x [y0, y0+h) of the full hologram (R-A12: coefficients outside the window or
 * outside [0, N_h)^2 are dropped).  psi(m, n) = sum_j a_j sum_k c_{z_j,k} delta(...) with the
 * level shift s_l = 2^l floor((ix + 2^(l-1)) / 2^l) (R-A8).  psi: h x w interleaved complex,
 * overwritten.  Points ascending, list entries in canonical order (R-A11).  Exact mode (R-A20):
 * the point's class table, every level shifted by s = (ix - cx, iy - cy).
 * Returns the number of in-window accumulations. */
int64_t orc_wasabi_window(void *lut, const double *pts, int64_t n, int64_t x0, int64_t y0, int64_t w,
                          int64_t h, double *psi) {
    orc_lut *t = (orc_lut *)lut;
    const orc_params *P = &t->P;
    memset(psi, 0, sizeof(double) * 2 * (size_t)(w * h));
    int64_t count = 0;
    for (int64_t j = 0; j < n; j++) {
        int64_t ix, iy;
        int iz;
        if (!orc_point(P, pts + 4 * j, &ix, &iy, &iz)) continue;
        double R = orc_radius_px(P, orc_level_z(P, iz));
        int64_t E = orc_footprint(P, R);
        if (ix + E < x0 || ix - E >= x0 + w || iy + E < y0 || iy - E >= y0 + h) continue;
        orc_depth_list *L = orc_lut_get(t, orc_point_table(P, ix, iy, iz));
        double a = pts[4 * j + 3];
        for (int64_t k = 0; k < L->n; k++) {
            int l = L->level[k];
            int64_t sx = orc_shift(P, ix, l), sy = orc_shift(P, iy, l);
            int64_t X = sx + L->dx[k], Y = sy + L->dy[k];
            if (X < 0 || X >= P->n_h || Y < 0 || Y >= P->n_h) continue;
            if (X < x0 || X >= x0 + w || Y < y0 || Y >= y0 + h) continue;
            double *o = psi + 2 * ((Y - y0) * w + (X - x0));
            o[0] += a * L->val[2 * k];
            o[1] += a * L->val[2 * k + 1];
            count++;
        }
    }
    return count;
}

/* Steps 2b + 3 on a window (x0, y0, w, h multiples of 2^L): psi by Eq.(2) (orc_wasabi_window) and
 * u = inverse FWT.  Haar: blocks are 2^L-local, so the window's own psi suffices.
 * Coiflets (R-A21): u at the window needs psi up to 3 (2^L - 1) px beyond it, so psi is formed on
 * the window grown by 64 px per side (clipped to the hologram: coefficients outside [0, N_h)^2 are
 * dropped, R-A12) and inverted with zero extension; u and psi are returned on the window. */
int64_t orc_hologram_window(void *lut, const double *pts, int64_t n, int64_t x0, int64_t y0, int64_t w,
                            int64_t h, double *u, double *psi) {
    orc_lut *t = (orc_lut *)lut;
    const orc_params *P = &t->P;
    int64_t g = P->wavelet == 1 ? 64 : 0;
    int64_t ex0 = x0 - g < 0 ? 0 : x0 - g, ey0 = y0 - g < 0 ? 0 : y0 - g;
    int64_t ex1 = x0 + w + g > P->n_h ? P->n_h : x0 + w + g, ey1 = y0 + h + g > P->n_h ? P->n_h : y0 + h + g;
    int64_t ew = ex1 - ex0, eh = ey1 - ey0;
    double *pe = (double *)malloc(sizeof(double) * 2 * (size_t)(ew * eh));
    int64_t cnt = orc_wasabi_window(lut, pts, n, ex0, ey0, ew, eh, pe);
    for (int64_t Y = 0; Y < h; Y++)
        memcpy(psi + 2 * (Y * w), pe + 2 * ((Y + y0 - ey0) * ew + (x0 - ex0)), sizeof(double) * 2 * (size_t)w);
    if (P->wavelet == 1) orc_fb_inv(1, pe, eh, ew, ew, P->levels);
    else orc_haar_inv(pe, eh, ew, ew, P->levels);
    for (int64_t Y = 0; Y < h; Y++)
        memcpy(u + 2 * (Y * w), pe + 2 * ((Y + y0 - ey0) * ew + (x0 - ex0)), sizeof(double) * 2 * (size_t)w);
    free(pe);
    return cnt;
}

/* ---------------------------------------------------------------- quantise (step 4) */

/* PAPER.md:135 (spherical reference at (x_r, y_r, z_r)) and :137 (binary amplitude), R-A14/A15.
 * u: h x w interleaved complex for hologram pixels [x0, x0+w) x [y0, y0+h).
 * bits: h x (w/8) bytes, pixel X -> byte (X - x0) >> 3, bit 7 - ((X - x0) & 7); 1 = I >= 0.
 * I_out (optional): the interference term I = Re(u conj(R)). */
int orc_quantize(const orc_params *P, double xr, double yr, double zr, const double *u, int64_t x0,
                 int64_t y0, int64_t w, int64_t h, uint8_t *bits, double *I_out) {
    double k = 2.0 * ORC_PI / P->wavelength;
    memset(bits, 0, (size_t)(h * (w / 8)));
    for (int64_t Y = y0; Y < y0 + h; Y++)
        for (int64_t X = x0; X < x0 + w; X++) {
            double x = (double)(X - P->n_h / 2) * P->pitch, y = (double)(Y - P->n_h / 2) * P->pitch;
            double ddx = x - xr, ddy = y - yr;
            double r = sqrt((ddx * ddx + ddy * ddy) + zr * zr);
            double ph = k * r;
            double Rr = cos(ph), Ri = sin(ph);
            const double *uu = u + 2 * ((Y - y0) * w + (X - x0));
            double I = uu[0] * Rr + uu[1] * Ri;     /* Re(u conj(R)) */
            if (I_out) I_out[(Y - y0) * w + (X - x0)] = I;
            if (I >= 0.0) bits[(Y - y0) * (w / 8) + ((X - x0) >> 3)] |= (uint8_t)(0x80u >> ((X - x0) & 7));
        }
    return 0;
}

/* ---------------------------------------------------------------- direct sums (Eq.(1)) */

/* D1: exact Eq.(1) on a window, continuous (x_j, y_j, z_j), with the
 * diffraction-limited window rho < |z_j| tan(theta) (+ the rho = 0 pixel), evaluated in
 * pixel units.  Per-pixel double loop (the O(N N_h^2) form of PAPER.md:76). */
int orc_direct_d1(const orc_params *P, const double *pts, int64_t n, int64_t x0, int64_t y0, int64_t w,
                  int64_t h, double *u) {
    double k = 2.0 * ORC_PI / P->wavelength, tn = orc_tan_theta(P);
    for (int64_t Y = y0; Y < y0 + h; Y++)
        for (int64_t X = x0; X < x0 + w; X++) {
            double sr = 0.0, si = 0.0;
            double xh = (double)(X - P->n_h / 2) * P->pitch, yh = (double)(Y - P->n_h / 2) * P->pitch;
            for (int64_t j = 0; j < n; j++) {
                const double *q = pts + 4 * j;
                if (!isfinite(q[0]) || !isfinite(q[1]) || !isfinite(q[2]) || !(q[3] > 0.0)) continue;
                double ex = (double)(X - P->n_h / 2) - q[0] / P->pitch;
                double ey = (double)(Y - P->n_h / 2) - q[1] / P->pitch;
                double rho2 = ex * ex + ey * ey;
                double Rj = fabs(q[2]) * tn / P->pitch;
                if (!(rho2 < Rj * Rj) && rho2 != 0.0) continue;
                double ddx = xh - q[0], ddy = yh - q[1];
                double r = sqrt((ddx * ddx + ddy * ddy) + q[2] * q[2]);
                sr += q[3] * cos(k * r);
                si += q[3] * sin(k * r);
            }
            u[2 * ((Y - y0) * w + (X - x0))] = sr;
            u[2 * ((Y - y0) * w + (X - x0)) + 1] = si;
        }
    return 0;
}

/* D2: quantised direct sum ("PSF stamping", the N-LUT-like form): snapped (ix, iy), level depth
 * z_iz and integer support S_iz, summed point by point. */
int orc_direct_d2(const orc_params *P, const double *pts, int64_t n, int64_t x0, int64_t y0, int64_t w,
                  int64_t h, double *u) {
    double k = 2.0 * ORC_PI / P->wavelength;
    memset(u, 0, sizeof(double) * 2 * (size_t)(w * h));
    for (int64_t j = 0; j < n; j++) {
        int64_t ix, iy;
        int iz;
        if (!orc_point(P, pts + 4 * j, &ix, &iy, &iz)) continue;
        double z = orc_level_z(P, iz), R = orc_radius_px(P, z);
        int64_t Rc = (int64_t)ceil(R) + 1;
        for (int64_t Y = iy - Rc; Y <= iy + Rc; Y++) {
            if (Y < y0 || Y >= y0 + h) continue;
            for (int64_t X = ix - Rc; X <= ix + Rc; X++) {
                if (X < x0 || X >= x0 + w) continue;
                int64_t dx = X - ix, dy = Y - iy;
                if (!orc_in_support(dx, dy, R)) continue;
                double xp = (double)dx * P->pitch, yp = (double)dy * P->pitch;
                double r = sqrt((xp * xp + yp * yp) + z * z);
                double *o = u + 2 * ((Y - y0) * w + (X - x0));
                o[0] += pts[4 * j + 3] * cos(k * r);
                o[1] += pts[4 * j + 3] * sin(k * r);
            }
        }
    }
    return 0;
}
