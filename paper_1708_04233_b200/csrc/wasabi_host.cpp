// wasabi_host.cpp -- the C ABI (include/wasabi.h): parameter validation, host-side geometry (L0),
// device buffer layouts, and the kernel launch sequence of every step.  No device memory is
// allocated here; every buffer belongs to the caller.
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <algorithm>
#include <string>
#include <vector>

#include "wasabi.h"
#include "internal.h"

#include <atomic>
#include <memory>
#include <mutex>

using namespace wasabi;

namespace wasabi {
static std::atomic<unsigned long long> g_launches{0};
void count_launches(int n) { g_launches.fetch_add((unsigned long long)n, std::memory_order_relaxed); }
}  // namespace wasabi

namespace {

thread_local std::string g_err;

wasabi_status fail(wasabi_status s, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return s;
}

wasabi_status cuda_fail(cudaError_t e, const char *what) {
    return fail(WASABI_ECUDA, "%s: %s (%s)", what, cudaGetErrorName(e), cudaGetErrorString(e));
}

#define CK(expr, what)                                   \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, what); \
    } while (0)

constexpr double kPi = 3.14159265358979323846;

inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

uint64_t fnv(uint64_t h, const void *p, size_t n) {
    const unsigned char *c = static_cast<const unsigned char *>(p);
    for (size_t i = 0; i < n; i++) { h ^= c[i]; h *= 1099511628211ull; }
    return h;
}

uint64_t param_hash(const wasabi_params &P) {
    uint64_t h = 1469598103934665603ull;
    h = fnv(h, &P.wavelength_m, 8); h = fnv(h, &P.pitch_m, 8); h = fnv(h, &P.n_h, 8);
    h = fnv(h, &P.n_depth, 4); h = fnv(h, &P.levels, 4); h = fnv(h, &P.z_min_m, 8);
    h = fnv(h, &P.z_max_m, 8); h = fnv(h, &P.retention, 8); h = fnv(h, &P.tile, 4);
    h = fnv(h, &P.flags, 4);
    return h;
}

wasabi_status validate(const wasabi_params *P) {
    if (!P) return fail(WASABI_EINVAL, "params is NULL");
    if (!(P->wavelength_m > 0) || !std::isfinite(P->wavelength_m)) return fail(WASABI_EINVAL, "wavelength_m must be > 0");
    if (!(P->pitch_m > 0) || !std::isfinite(P->pitch_m)) return fail(WASABI_EINVAL, "pitch_m must be > 0");
    if (!(P->wavelength_m < 2.0 * P->pitch_m))
        return fail(WASABI_EINVAL, "Nyquist: wavelength (%g) must be < 2 * pitch (%g)", P->wavelength_m, P->pitch_m);
    if (P->levels < 1 || P->levels > kMaxLevels) return fail(WASABI_EINVAL, "levels must be in 1..%d", kMaxLevels);
    if (P->tile != 64 && P->tile != 128) return fail(WASABI_EINVAL, "tile must be 64 or 128 (shared-memory tile)");
    if (P->tile % (1 << P->levels)) return fail(WASABI_EINVAL, "tile must be a multiple of 2^levels");
    if (P->n_h <= 0 || P->n_h % P->tile) return fail(WASABI_EINVAL, "n_h (%lld) must be a positive multiple of tile",
                                                     (long long)P->n_h);
    if (P->n_h > (1ll << 24)) return fail(WASABI_EINVAL, "n_h too large");
    if (P->n_depth < 1) return fail(WASABI_EINVAL, "n_depth must be >= 1");
    if (!std::isfinite(P->z_min_m) || !std::isfinite(P->z_max_m) || P->z_max_m < P->z_min_m)
        return fail(WASABI_EINVAL, "need finite z_min <= z_max");
    if (P->n_depth > 1 && !(P->z_max_m > P->z_min_m)) return fail(WASABI_EINVAL, "n_depth > 1 needs z_max > z_min");
    if (!(P->retention > 0) || P->retention > 1) return fail(WASABI_EINVAL, "retention must be in (0, 1]");
    if (llround(P->retention * 1e6) < 1) return fail(WASABI_EINVAL, "retention below 1 ppm");
    if (P->flags & ~(uint32_t)(WASABI_FLAG_EXACT_SHIFT | WASABI_FLAG_COIFLET | WASABI_FLAG_GATHER | WASABI_FLAG_SCATTER))
        return fail(WASABI_EINVAL, "unknown flags 0x%x", P->flags);
    if ((P->flags & WASABI_FLAG_GATHER) && (P->flags & WASABI_FLAG_SCATTER))
        return fail(WASABI_EINVAL, "WASABI_FLAG_GATHER and WASABI_FLAG_SCATTER are exclusive");
    if ((P->flags & WASABI_FLAG_GATHER) && (P->tile != 64 || P->levels < 2 || (P->flags & WASABI_FLAG_COIFLET)))
        return fail(WASABI_EINVAL, "WASABI_FLAG_GATHER needs tile 64, levels >= 2 and Haar tables");
    if ((P->flags & WASABI_FLAG_EXACT_SHIFT) && P->levels > 4)
        return fail(WASABI_EINVAL, "WASABI_FLAG_EXACT_SHIFT needs levels <= 4 (4^L offset-class tables per depth)");
    if (P->flags & WASABI_FLAG_COIFLET) {
        if (P->flags & WASABI_FLAG_EXACT_SHIFT)
            return fail(WASABI_EINVAL, "WASABI_FLAG_COIFLET cannot be combined with WASABI_FLAG_EXACT_SHIFT");
        if (P->levels > 4) return fail(WASABI_EINVAL, "WASABI_FLAG_COIFLET needs levels <= 4 (psi halo of one tile)");
    }
    return WASABI_OK;
}

// Superposition path (wasabi.h WASABI_FLAG_GATHER): the dense gather at high retention.
bool use_gather(const wasabi_params &P) {
    if (P.flags & WASABI_FLAG_GATHER) return true;
    if (P.flags & WASABI_FLAG_SCATTER) return false;
    return llround(P.retention * 1e6) >= 250000 && P.tile == 64 && P.levels >= 2 && !(P.flags & WASABI_FLAG_COIFLET);
}

// Step 2b launcher: the scatter kernel (window LUT) or the dense gather (WASABI_FLAG_GATHER tables);
// the table buffer was built for the same parameters, so use_gather() names its layout.
cudaError_t launch_sup(const wasabi_params &P, const void *d_bins, const void *d_tables, int64_t row0, int tiles_y,
                       float2 *psi, int fused, const double *print4, uint8_t *bits, cudaStream_t s, int tile_row0 = 0,
                       int tile_row1 = -1) {
    const int T = P.tile, tiles_x = (int)(P.n_h / T);
    const int cb = (P.flags & WASABI_FLAG_EXACT_SHIFT) ? P.levels : 0;
    if (use_gather(P))
        return launch_gather(d_bins, d_tables, P.levels, cb, tiles_x, tiles_y, row0, P.n_h, psi, fused, print4,
                             P.pitch_m, bits, s, tile_row0, tile_row1);
    return launch_superpose(d_bins, d_tables, T, T + kWinMargin, P.levels, cb, tiles_x, tiles_y, row0, P.n_h, psi,
                            fused, print4, P.pitch_m, bits, s, tile_row0, tile_row1);
}

wasabi_status validate_band(const wasabi_params *P, int64_t row0, int64_t row1) {
    if (row0 < 0 || row1 > P->n_h || row0 > row1) return fail(WASABI_EINVAL, "band [%lld, %lld) outside [0, n_h)",
                                                              (long long)row0, (long long)row1);
    if (row0 % P->tile || row1 % P->tile) return fail(WASABI_EINVAL, "band rows must be multiples of tile");
    return WASABI_OK;
}

// S_d membership (PAPER.md:90 circ, centre always kept).
inline bool in_support(int64_t dx, int64_t dy, double R) {
    if (dx == 0 && dy == 0) return true;
    return (double)(dx * dx + dy * dy) < R * R;
}

// Structural nnz: coefficient positions whose support block touches S_d (centre (Cx, Cy) in a
// side x side table).  Per block row the disc's x-extent is the union of symmetric row intervals
// [-xm, xm], so the blocks touched are those overlapping [Cx - max xm, Cx + max xm].
int64_t nnz_structural(int64_t side, int64_t Cx, int64_t Cy, double R, int L) {
    std::vector<int64_t> xm(side);
    for (int64_t Y = 0; Y < side; Y++) {
        const int64_t dy = Y - Cy;
        const double s = R * R - (double)(dy * dy);
        int64_t x = s > 0 ? (int64_t)std::floor(std::sqrt(s)) : 0;
        while (x >= 0 && !in_support(x, dy, R)) x--;
        while (x >= 0 && in_support(x + 1, dy, R)) x++;
        xm[Y] = x;  // -1: row empty
    }
    int64_t nnz = 0;
    for (int l = 1; l <= L; l++) {
        const int64_t b = 1ll << l;
        for (int64_t Y0 = 0; Y0 < side; Y0 += b) {
            int64_t X = -1;
            for (int64_t Y = Y0; Y < Y0 + b; Y++) X = std::max(X, xm[Y]);
            if (X < 0) continue;
            const int64_t nblk = (Cx + X) / b - (Cx - X) / b + 1;
            nnz += nblk * (l == L ? 4 : 3);
        }
    }
    return nnz;
}

// Structural nnz of the coif1 transform (R-A21): the coefficient of level l at index (m, n) =
// (X >> l, Y >> l) depends on the input rectangle [2^l m - 2 (2^l - 1), 2^l m + 3 (2^l - 1)] per axis
// (6 taps, offset 2); it can be nonzero iff that rectangle meets S_d, i.e. iff its lattice point
// nearest to the centre (C, C) is in S_d.  Level of a position: t = trailing zeros common to X and Y.
int64_t nnz_coif(int64_t side, int64_t C, double R, int L) {
    int64_t nnz = 0;
    for (int64_t Y = 0; Y < side; Y++)
        for (int64_t X = 0; X < side; X++) {
            int t = 0;
            while (t < L && !((X >> t) & 1) && !((Y >> t) & 1)) t++;
            const int l = t >= L ? L : t + 1;
            const int64_t b = 1ll << l, mx = X >> l, my = Y >> l;
            const int64_t x0 = b * mx - 2 * (b - 1), x1 = b * mx + 3 * (b - 1);
            const int64_t y0 = b * my - 2 * (b - 1), y1 = b * my + 3 * (b - 1);
            const int64_t nx = std::min(std::max(C, x0), x1), ny = std::min(std::max(C, y0), y1);
            if (in_support(nx - C, ny - C, R)) nnz++;
        }
    return nnz;
}

struct Geo {
    wasabi_params P;
    double k, tan_theta, dz;
    int T, S, L, nd, nz, cb;   // nd = tables, nz = depth levels, cb = offset-class bits (R-A20)
    int wav = 0;               // 1: coif1 tables (R-A21)
    int gather = 0;            // 1: dense gather superposition (WASABI_FLAG_GATHER / high retention)
    std::vector<int64_t> pre;  // coif: per level, (nd + 1) prefix of analysis work items
    size_t sc_work = 0, sc_tmp = 0, sc_pre = 0;
    std::vector<KDesc> kd;
    std::vector<DDesc> dd;
    std::vector<int32_t> ctabase;
    int64_t total_entries = 0, total_ptrs = 0, total_ctas = 0, total_coef = 0, max_E = 0, total_vptrs = 0;
    TableHeader th;
    size_t table_bytes = 0, scratch_bytes = 0;
    size_t sc_val = 0, sc_key = 0, sc_hist = 0, sc_sel = 0, sc_scan = 0, sc_cursor = 0;
};

double level_z(const wasabi_params &P, double dz, int d) {
    if (P.n_depth <= 1) return P.z_min_m;
    return P.z_min_m + (double)d * dz;
}

wasabi_status compute_geo_uncached(const wasabi_params *P, Geo &g) {
    wasabi_status st = validate(P);
    if (st != WASABI_OK) return st;
    g.P = *P;
    g.T = P->tile; g.S = P->tile + kWinMargin; g.L = P->levels; g.nz = P->n_depth;
    g.cb = (P->flags & WASABI_FLAG_EXACT_SHIFT) ? P->levels : 0;
    g.nd = P->n_depth << (2 * g.cb);
    g.wav = (P->flags & WASABI_FLAG_COIFLET) ? 1 : 0;
    g.gather = use_gather(*P) ? 1 : 0;
    g.k = 2.0 * kPi / P->wavelength_m;
    const double sigma = P->wavelength_m / (2.0 * P->pitch_m);
    g.tan_theta = sigma / std::sqrt(1.0 - sigma * sigma);
    g.dz = P->n_depth > 1 ? (P->z_max_m - P->z_min_m) / (double)(P->n_depth - 1) : 0.0;
    g.kd.assign(g.nd, KDesc{});
    g.dd.assign(g.nd, DDesc{});
    g.ctabase.assign(g.nd + 1, 0);
    const int64_t B = 1ll << g.L;
    int64_t ptr = 0, ctas = 0, coef = 0, entries = 0, vptr = 0;
    for (int d = 0; d < g.nd; d++) {
        const int zi = d >> (2 * g.cb);                      // depth level of table d
        const int cx = d & ((1 << g.cb) - 1), cy = (d >> g.cb) & ((1 << g.cb) - 1);
        const double z = level_z(*P, g.dz, zi);
        const double R = std::fabs(z) * g.tan_theta / P->pitch_m;
        // coif1 tables are padded by 3 2^L so every nonzero coefficient of the disc stays inside (R-A21)
        const int64_t H = B * ((int64_t)std::floor((R + (g.wav ? 3.0 * (double)B : 0.0)) / (double)B) + 1);
        const int64_t side = 2 * H + (g.cb ? B : 0);
        if (side > kMaxTableSide)
            return fail(WASABI_EINVAL, "depth %d: PSF table side %lld exceeds %d (|z| too large for this pitch)", zi,
                        (long long)side, kMaxTableSide);
        const int64_t E = (int64_t)std::ceil(R) + (g.wav ? 7 : 3) * (1ll << (g.L - 1));
        DDesc &D = g.dd[d];
        KDesc &K = g.kd[d];
        D.z = z; D.R = R;
        D.side = (int32_t)side;
        D.cx = cx; D.cy = cy;
        K.side = (int32_t)side;
        D.tiles = (int32_t)((side + 63) / 64);
        D.cta_base = (int32_t)ctas;
        g.ctabase[d] = (int32_t)ctas;
        ctas += (int64_t)D.tiles * D.tiles;
        D.coef_off = coef;
        coef += side * side;
        K.H = (int32_t)H;
        K.E = (int32_t)E;
        {   // PSF-disc reach: the level's disc (D2) and the continuous point's (D1: |z| within half a level
            // of z_d, pixel rounding +-1/2 px), so both direct sums find every contributing point
            const double Rh = (std::fabs(z) + 0.5 * g.dz) * g.tan_theta / P->pitch_m + 1.0;
            K.Ed = (int32_t)std::ceil(Rh);
            K.Qd = (int32_t)std::ceil(Rh * Rh);
        }

        g.max_E = std::max(g.max_E, E);
        D.group_base = (int32_t)ptr;
        for (int l = 1; l <= g.L; l++) {
            const int64_t nb = side >> l, hb = band_blocks(g.T, l), nbands = (nb + hb - 1) / hb;
            K.ptr_base[l - 1] = (int32_t)ptr;
            ptr += nbands * (nb + 1);
        }
        for (int l = g.L + 1; l <= kMaxLevels; l++) K.ptr_base[l - 1] = (int32_t)ptr;
        D.n_groups = (int32_t)(ptr - D.group_base);
        // window LUT pointer rows: per level, variants x bands x (column groups + 1)
        D.vgroup_base = (int32_t)vptr;
        K.vbase = (int32_t)vptr;
        for (int l = 1; l <= g.L; l++) {
            K.vptr_base[l - 1] = (int32_t)vptr;
            vptr += win_slots(D.side, l, g.cb);
        }
        for (int l = g.L + 1; l <= kMaxLevels; l++) K.vptr_base[l - 1] = (int32_t)vptr;
        for (int c = 0; c < 2; c++) {
            K.cls4[c][0] = (int32_t)H;
            for (int j = 0; j < 3; j++) {
                const int l = superpose_class_level(c, j, g.L);
                K.cls4[c][1 + j] = l ? K.vptr_base[l - 1] : 0;
            }
        }
        D.nnz = g.wav ? nnz_coif(side, H, R, g.L) : nnz_structural(side, H + cx, H + cy, R, g.L);
        {
            const int64_t r_ppm = llround(P->retention * 1e6);
            const int64_t n = (r_ppm * D.nnz + 999999) / 1000000;
            D.n_r = std::min(n, D.nnz);
        }
        entries += D.n_r;
        if (ptr > (int64_t)INT32_MAX / 2 || ctas > (int64_t)INT32_MAX / 2 ||
            (!g.gather && (entries * win_variants(1, g.cb) > (int64_t)INT32_MAX / 2 || vptr > (int64_t)INT32_MAX / 2)))
            return fail(WASABI_EINVAL, "table too large for 32-bit indices");
    }
    g.ctabase[g.nd] = (int32_t)ctas;
    g.total_entries = entries; g.total_ptrs = ptr; g.total_ctas = ctas; g.total_coef = coef; g.total_vptrs = vptr;
    // table buffer layout
    TableHeader &h = g.th;
    std::memset(&h, 0, sizeof h);
    h.magic = kTableMagic;
    h.param_hash = param_hash(*P);
    h.n_depth = g.nd; h.levels = g.L; h.tile = g.T; h.S = g.S;
    h.cls_bits = g.cb; h.n_zlevels = g.nz; h.wavelet = g.wav;
    h.total_entries = entries; h.total_ptrs = ptr; h.total_ctas = ctas;
    size_t off = 256;
    h.kdesc_off = off; off = align_up(off + sizeof(KDesc) * g.nd, 256);
    h.ddesc_off = off; off = align_up(off + sizeof(DDesc) * g.nd, 256);
    h.ctabase_off = off; off = align_up(off + 4 * (g.nd + 1), 256);
    h.ptr_off = off; off = align_up(off + 4 * (size_t)(ptr + 1), 256);
    h.ent_off = off; off = align_up(off + 16 * (size_t)entries, 256);
    // window LUT: a level-l entry is stored once per variant (<= win_variants(1) copies)
    if (g.gather) vptr = 0;                // gather mode: no window LUT (the dense tables instead)
    g.total_vptrs = vptr;
    h.gather = g.gather;
    h.total_vptrs = vptr;
    h.vent_cap = g.gather ? 0 : win_variants(1, g.cb) * entries;
    h.vptr_off = off; off = align_up(off + 4 * (size_t)(vptr + 1), 256);
    // + 32 entries of padding: the superposition kernel reads whole 32-entry chunks past a range end
    h.vval_off = off; off = align_up(off + 8 * (size_t)(h.vent_cap + 32), 256);
    h.vpos_off = off; off = align_up(off + 2 * (size_t)(h.vent_cap + 32), 256);
    // dense wavelet tables (gather mode): table t at dense_off + 8 coef_off_t, side_t^2 complex64
    h.dense_off = off;
    if (g.gather) off = align_up(off + 8 * (size_t)coef, 256);
    h.table_bytes = off;
    g.table_bytes = off;
    // build scratch
    size_t so = 0;
    g.sc_val = so; so = align_up(so + 8 * (size_t)coef, 256);
    g.sc_key = so; so = align_up(so + 4 * (size_t)coef, 256);
    g.sc_hist = so; so = align_up(so + 4 * 256 * (size_t)g.nd, 256);
    g.sc_sel = so; so = align_up(so + 24 * (size_t)g.nd, 256);
    g.sc_scan = so; so = align_up(so + scan_scratch_bytes(std::max(ptr, vptr) + 1), 256);
    g.sc_cursor = so; so = align_up(so + 4 * (size_t)(vptr + 1), 256);   // window-LUT slot cursors
    if (g.wav) {   // fp64 work and ping-pong tables, per-level work-item prefixes
        g.pre.assign((size_t)g.L * (g.nd + 1), 0);
        for (int l = 1; l <= g.L; l++)
            for (int d = 0; d < g.nd; d++) {
                const int64_t N = (int64_t)g.dd[d].side >> (l - 1);
                g.pre[(size_t)(l - 1) * (g.nd + 1) + d + 1] = g.pre[(size_t)(l - 1) * (g.nd + 1) + d] + N * (N / 2);
            }
        g.sc_work = so; so = align_up(so + 16 * (size_t)coef, 256);
        g.sc_tmp = so; so = align_up(so + 16 * (size_t)coef, 256);
        g.sc_pre = so; so = align_up(so + 8 * g.pre.size(), 256);
    }
    g.scratch_bytes = so;
    return WASABI_OK;
}

// Every entry point derives the geometry from the parameters; the structural nnz counts make that
// O(table area) host work (tens of ms for 4^L offset-class or coiflet tables), so the last few
// parameter sets are memoised (keyed by the full parameter bytes).
struct GeoCache {
    std::mutex mu;
    std::vector<std::pair<wasabi_params, std::shared_ptr<const Geo>>> items;   // most recent last
};
GeoCache &geo_cache() {
    static GeoCache c;
    return c;
}

wasabi_status compute_geo(const wasabi_params *P, Geo &g) {
    wasabi_status st = validate(P);
    if (st != WASABI_OK) return st;
    GeoCache &c = geo_cache();
    {
        std::lock_guard<std::mutex> lk(c.mu);
        for (auto &it : c.items)
            if (std::memcmp(&it.first, P, sizeof *P) == 0) {
                g = *it.second;
                return WASABI_OK;
            }
    }
    auto fresh = std::make_shared<Geo>();
    if ((st = compute_geo_uncached(P, *fresh)) != WASABI_OK) return st;
    g = *fresh;
    std::lock_guard<std::mutex> lk(c.mu);
    c.items.emplace_back(*P, fresh);
    if (c.items.size() > 8) c.items.erase(c.items.begin());
    return WASABI_OK;
}

// Bin buffer layout.
struct BinLayout {
    BinHeader h;
    size_t bytes;
};

BinLayout bin_layout(const Geo &g, int64_t n, int64_t row0, int64_t row1) {
    BinLayout b;
    BinHeader &h = b.h;
    std::memset(&h, 0, sizeof h);
    h.magic = kBinMagic;
    h.param_hash = param_hash(g.P);
    h.n_points = n; h.row0 = row0; h.row1 = row1;
    h.T = g.T;
    h.tiles_x = (int32_t)(g.P.n_h / g.T);
    h.tiles_y = (int32_t)((row1 - row0) / g.T);
    h.n_tiles = (int64_t)h.tiles_x * h.tiles_y;
    const int64_t span = (2 * g.max_E) / g.T + 2;
    const int64_t per_pt = std::min<int64_t>(h.tiles_x, span) * std::min<int64_t>(h.tiles_y, span);
    h.capacity = n * per_pt;
    size_t off = 512;
    h.ptr_off = off; off = align_up(off + 8 * (size_t)(h.n_tiles + 1), 256);
    h.cnt_off = off; off = align_up(off + 4 * (size_t)(h.n_tiles + 1), 256);
    h.scan_off = off;
    off = align_up(off + scan_scratch_bytes(h.n_tiles + 1) + 4 * (size_t)h.n_tiles + 4, 256);
    h.pts_off = off; off = align_up(off + 16 * (size_t)n, 256);
    h.idx_off = off; off = align_up(off + 4 * (size_t)h.capacity, 256);
    h.idx2_off = off; off = align_up(off + 4 * (size_t)h.capacity, 256);
    h.bin_bytes = off;
    b.bytes = off;
    return b;
}

bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }

int cls_bits(const wasabi_params &P) { return (P.flags & WASABI_FLAG_EXACT_SHIFT) ? P.levels : 0; }

}  // namespace

extern "C" {

const char *wasabi_last_error(void) { return g_err.c_str(); }

const char *wasabi_version(void) { return "wasabi-b200 0.1 (sm_100a)"; }

unsigned long long wasabi_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

wasabi_status wasabi_psf_tables_bytes(const wasabi_params *params, size_t *table_bytes, size_t *scratch_bytes) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (table_bytes) *table_bytes = g.table_bytes;
    if (scratch_bytes) *scratch_bytes = g.scratch_bytes;
    return WASABI_OK;
}

wasabi_status wasabi_depth_geometry(const wasabi_params *params, int32_t depth, wasabi_depth_info *out) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (depth < 0 || depth >= g.nd || !out) return fail(WASABI_EINVAL, "table index out of range");
    out->z_m = g.dd[depth].z;
    out->radius_px = g.dd[depth].R;
    out->half = g.kd[depth].H;
    out->footprint = g.kd[depth].E;
    out->nnz = g.dd[depth].nnz;
    out->n_r = g.dd[depth].n_r;
    return WASABI_OK;
}

int64_t wasabi_coif_halo_rows(const wasabi_params *params) {
    // the coif1 synthesis of L <= 4 levels reaches 3 (2^L - 1) <= 45 rows: one tile (a multiple of it)
    return (params && (params->flags & WASABI_FLAG_COIFLET)) ? (int64_t)std::max(64, params->tile) : 0;
}

wasabi_status wasabi_table_count(const wasabi_params *params, int64_t *n_tables) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (n_tables) *n_tables = g.nd;
    return WASABI_OK;
}

wasabi_status wasabi_build_psf_tables(const wasabi_params *params, void *d_tables, size_t table_bytes,
                                      void *d_scratch, size_t scratch_bytes, cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (!d_tables || !d_scratch) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_tables, 256) || !aligned(d_scratch, 256)) return fail(WASABI_EINVAL, "buffers must be 256-byte aligned");
    if (table_bytes < g.table_bytes) return fail(WASABI_ENOSPC, "table buffer needs %zu bytes", g.table_bytes);
    if (scratch_bytes < g.scratch_bytes) return fail(WASABI_ENOSPC, "scratch buffer needs %zu bytes", g.scratch_bytes);
    char *tb = static_cast<char *>(d_tables);
    char *sb = static_cast<char *>(d_scratch);
    CK(launch_write_blob(tb, &g.th, sizeof g.th, stream), "write table header");
    CK(launch_write_blob(tb + g.th.kdesc_off, g.kd.data(), sizeof(KDesc) * g.nd, stream), "write kdesc");
    CK(launch_write_blob(tb + g.th.ddesc_off, g.dd.data(), sizeof(DDesc) * g.nd, stream), "write ddesc");
    CK(launch_write_blob(tb + g.th.ctabase_off, g.ctabase.data(), 4 * (g.nd + 1), stream), "write ctabase");
    float2 *cval = reinterpret_cast<float2 *>(sb + g.sc_val);
    uint32_t *ckey = reinterpret_cast<uint32_t *>(sb + g.sc_key);
    if (g.wav) {
        std::vector<int64_t> last(g.L);
        for (int l = 1; l <= g.L; l++) last[l - 1] = g.pre[(size_t)(l - 1) * (g.nd + 1) + g.nd];
        CK(launch_write_blob(sb + g.sc_pre, g.pre.data(), 8 * g.pre.size(), stream), "write coif prefixes");
        CK(launch_coif_tables(g.th, d_tables, reinterpret_cast<double2 *>(sb + g.sc_work),
                              reinterpret_cast<double2 *>(sb + g.sc_tmp), reinterpret_cast<const int64_t *>(sb + g.sc_pre),
                              last.data(), cval, ckey, g.total_coef, g.k, params->pitch_m, g.L, stream),
           "coif tables");
    } else {
        CK(launch_psf_haar(g.th, d_tables, cval, ckey, g.k, params->pitch_m, g.L, g.nd, stream), "psf_haar");
    }
    CK(launch_select(g.th, d_tables, ckey, reinterpret_cast<unsigned int *>(sb + g.sc_hist),
                     reinterpret_cast<unsigned long long *>(sb + g.sc_sel), g.nd, stream),
       "select");
    CK(cudaMemsetAsync(tb + g.th.ptr_off, 0, 4 * (size_t)(g.total_ptrs + 1), stream), "memset ptr");
    const unsigned long long *sel = reinterpret_cast<const unsigned long long *>(sb + g.sc_sel);
    CK(launch_groups(g.th, d_tables, cval, ckey, sel, 0, stream), "groups count");
    CK(launch_scan_i32(reinterpret_cast<int32_t *>(tb + g.th.ptr_off), g.total_ptrs + 1, sb + g.sc_scan, stream),
       "scan ptr");
    CK(launch_groups(g.th, d_tables, cval, ckey, sel, 1, stream), "groups scatter");
    if (g.gather) {   // dense tables: zeros, then every kept coefficient at its table position
        CK(cudaMemsetAsync(tb + g.th.dense_off, 0, 8 * (size_t)g.total_coef, stream), "memset dense");
        CK(launch_dense_fill(g.th, d_tables, stream), "dense fill");
        return WASABI_OK;
    }
    // the superposition kernel's window LUT, re-grouped from the canonical lists
    CK(cudaMemsetAsync(tb + g.th.vptr_off, 0, 4 * (size_t)(g.total_vptrs + 1), stream), "memset vptr");
    int32_t *cursor = reinterpret_cast<int32_t *>(sb + g.sc_cursor);
    CK(launch_ventries(g.th, d_tables, 0, cursor, stream), "window LUT count");
    CK(launch_scan_i32(reinterpret_cast<int32_t *>(tb + g.th.vptr_off), g.total_vptrs + 1, sb + g.sc_scan, stream),
       "scan vptr");
    CK(cudaMemcpyAsync(cursor, tb + g.th.vptr_off, 4 * (size_t)(g.total_vptrs + 1), cudaMemcpyDeviceToDevice, stream),
       "window LUT cursors");
    CK(launch_ventries(g.th, d_tables, 1, cursor, stream), "window LUT scatter");
    return WASABI_OK;
}

wasabi_status wasabi_bin_points_bytes(const wasabi_params *params, int64_t n, int64_t row0, int64_t row1,
                                      size_t *bin_bytes) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(WASABI_EINVAL, "n out of range");
    if (bin_bytes) *bin_bytes = bin_layout(g, n, row0, row1).bytes;
    return WASABI_OK;
}

namespace {
wasabi_status bin_points_impl(const wasabi_params *params, const void *d_tables, const float *d_points, int64_t n,
                              int64_t row0, int64_t row1, void *d_bins, size_t bin_bytes, int psf,
                              cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(WASABI_EINVAL, "n out of range");
    if (!d_tables || !d_bins || (n > 0 && !d_points)) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_bins, 256)) return fail(WASABI_EINVAL, "d_bins must be 256-byte aligned");
    if (n > 0 && !aligned(d_points, 16)) return fail(WASABI_EINVAL, "d_points must be 16-byte aligned");
    BinLayout b = bin_layout(g, n, row0, row1);
    if (bin_bytes < b.bytes) return fail(WASABI_ENOSPC, "bin buffer needs %zu bytes", b.bytes);
    CK(launch_write_blob(d_bins, &b.h, sizeof b.h, stream), "write bin header");
    const KDesc *kd = reinterpret_cast<const KDesc *>(static_cast<const char *>(d_tables) + g.th.kdesc_off);
    CK(launch_bin(b.h, d_bins, kd, reinterpret_cast<const float4 *>(d_points), params->pitch_m, params->n_h,
                  params->z_min_m, g.dz, g.nz, g.cb, psf, stream),
       "bin");
    return WASABI_OK;
}
}  // namespace

wasabi_status wasabi_bin_points(const wasabi_params *params, const void *d_tables, const float *d_points, int64_t n,
                                int64_t row0, int64_t row1, void *d_bins, size_t bin_bytes, cudaStream_t stream) {
    return bin_points_impl(params, d_tables, d_points, n, row0, row1, d_bins, bin_bytes, 0, stream);
}

wasabi_status wasabi_bin_points_psf(const wasabi_params *params, const void *d_tables, const float *d_points,
                                    int64_t n, int64_t row0, int64_t row1, void *d_bins, size_t bin_bytes,
                                    cudaStream_t stream) {
    if (params && (params->flags & (WASABI_FLAG_EXACT_SHIFT | WASABI_FLAG_COIFLET)))
        return fail(WASABI_EINVAL, "wasabi_bin_points_psf: standard (one table per depth) parameters only");
    return bin_points_impl(params, d_tables, d_points, n, row0, row1, d_bins, bin_bytes, 1, stream);
}

wasabi_status wasabi_count_accumulations(const wasabi_params *params, const void *d_tables, const float *d_points,
                                        int64_t n, int64_t row0, int64_t row1, void *d_scratch, int64_t *h_count,
                                        cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (row0 < 0 || row1 > params->n_h || row1 < row0) return fail(WASABI_EINVAL, "rows out of range");
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(WASABI_EINVAL, "n out of range");
    if (!d_tables || !d_scratch || !h_count || (n > 0 && !d_points)) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_scratch, 8) || (n > 0 && !aligned(d_points, 16))) return fail(WASABI_EINVAL, "misaligned buffer");
    unsigned long long *cnt = static_cast<unsigned long long *>(d_scratch);
    CK(launch_count_acc(g.th, d_tables, reinterpret_cast<const float4 *>(d_points), n, params->pitch_m, params->n_h,
                        params->z_min_m, g.dz, g.nz, g.cb, g.L, row0, row1, cnt, nullptr, stream),
       "count accumulations");
    unsigned long long c = 0;
    CK(cudaMemcpyAsync(&c, cnt, sizeof c, cudaMemcpyDeviceToHost, stream), "read count");
    CK(cudaStreamSynchronize(stream), "sync");
    *h_count = (int64_t)c;
    return WASABI_OK;
}

wasabi_status wasabi_row_work(const wasabi_params *params, const void *d_tables, const float *d_points, int64_t n,
                              double *d_row_work, void *d_scratch, cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(WASABI_EINVAL, "n out of range");
    if (!d_tables || !d_scratch || !d_row_work || (n > 0 && !d_points)) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_scratch, 8) || !aligned(d_row_work, 8) || (n > 0 && !aligned(d_points, 16)))
        return fail(WASABI_EINVAL, "misaligned buffer");
    CK(launch_count_acc(g.th, d_tables, reinterpret_cast<const float4 *>(d_points), n, params->pitch_m, params->n_h,
                        params->z_min_m, g.dz, g.nz, g.cb, g.L, 0, params->n_h,
                        static_cast<unsigned long long *>(d_scratch), d_row_work, stream),
       "row work");
    return WASABI_OK;
}

wasabi_status wasabi_superpose(const wasabi_params *params, const void *d_tables, const void *d_bins, int64_t row0,
                               int64_t row1, float *d_psi, cudaStream_t stream) {
    wasabi_status st = validate(params);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (!d_tables || !d_bins || (!d_psi && row1 > row0)) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_psi, 16)) return fail(WASABI_EINVAL, "d_psi must be 16-byte aligned");
    const int T = params->tile;
    CK(launch_sup(*params, d_bins, d_tables, row0, (int)((row1 - row0) / T), reinterpret_cast<float2 *>(d_psi), 0,
                  nullptr, nullptr, stream),
       "superpose");
    return WASABI_OK;
}

wasabi_status wasabi_superpose_inverse(const wasabi_params *params, const void *d_tables, const void *d_bins,
                                       int64_t row0, int64_t row1, const wasabi_print_params *print, float *d_u,
                                       uint8_t *d_bits, cudaStream_t stream) {
    wasabi_status st = validate(params);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (!d_tables || !d_bins) return fail(WASABI_EINVAL, "NULL buffer");
    if (params->flags & WASABI_FLAG_COIFLET)
        return fail(WASABI_EINVAL, "WASABI_FLAG_COIFLET: the coiflet inverse is not tile-local; use wasabi_superpose "
                                   "on the halo band + wasabi_inverse_wt");
    if (d_bits && !print) return fail(WASABI_EINVAL, "d_bits needs print params");
    if (!aligned(d_u, 16)) return fail(WASABI_EINVAL, "d_u must be 16-byte aligned");
    double p4[4];
    if (print) { p4[0] = print->x_r_m; p4[1] = print->y_r_m; p4[2] = print->z_r_m; p4[3] = 1.0 / params->wavelength_m; }
    const int T = params->tile;
    CK(launch_sup(*params, d_bins, d_tables, row0, (int)((row1 - row0) / T), reinterpret_cast<float2 *>(d_u), 1,
                  print ? p4 : nullptr, d_bits, stream),
       "superpose_inverse");
    return WASABI_OK;
}

wasabi_status wasabi_inverse_wt(const wasabi_params *params, float *d_psi, float *d_u, int64_t row0,
                                int64_t row1, const wasabi_print_params *print, uint8_t *d_bits, cudaStream_t stream) {
    wasabi_status st = validate(params);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (params->n_h % 64 || (row1 - row0) % 64) return fail(WASABI_EINVAL, "n_h and band height must be multiples of 64");
    if (!d_psi && row1 > row0) return fail(WASABI_EINVAL, "NULL d_psi");
    if (d_bits && !print) return fail(WASABI_EINVAL, "d_bits needs print params");
    if (!aligned(d_psi, 16) || !aligned(d_u, 16)) return fail(WASABI_EINVAL, "fields must be 16-byte aligned");
    double p4[4];
    if (print) { p4[0] = print->x_r_m; p4[1] = print->y_r_m; p4[2] = print->z_r_m; p4[3] = 1.0 / params->wavelength_m; }
    if (params->flags & WASABI_FLAG_COIFLET) {   // R-A21: in place on the halo band, then u rows, then bits
        const int64_t H = wasabi_coif_halo_rows(params);
        const int64_t e0 = std::max<int64_t>(0, row0 - H), e1 = std::min<int64_t>(params->n_h, row1 + H);
        float2 *pe = reinterpret_cast<float2 *>(d_psi);
        // does d_u overlap the psi halo band? (address ranges compared as integers)
        const uintptr_t ub = reinterpret_cast<uintptr_t>(d_u), pb = reinterpret_cast<uintptr_t>(d_psi);
        const bool u_in_psi = d_u && ub < pb + 8 * (uintptr_t)((e1 - e0) * params->n_h) &&
                              ub + 8 * (uintptr_t)((row1 - row0) * params->n_h) > pb;
        if ((d_u || d_bits) && !u_in_psi) {   // fused tile synthesis + quantise; d_psi is only read (wasabi.h)
            if (row1 > row0)
                CK(launch_coif_fused(pe, e0, e1, row0, row1, params->n_h, params->levels, print ? p4 : nullptr,
                                     params->pitch_m, reinterpret_cast<float2 *>(d_u), d_bits, stream),
                   "coif fused inverse");
            return WASABI_OK;
        }
        // line passes in place on the halo band (wasabi.h)
        if (e1 > e0) CK(launch_coif_inverse(pe, e1 - e0, params->n_h, params->levels, stream), "coif inverse");
        float2 *uc = pe + (row0 - e0) * params->n_h;
        if (d_u && reinterpret_cast<float2 *>(d_u) != uc && row1 > row0)
            CK(cudaMemcpyAsync(d_u, uc, 8 * (size_t)(row1 - row0) * (size_t)params->n_h, cudaMemcpyDeviceToDevice,
                               stream), "copy u");
        if (d_bits && row1 > row0)
            CK(launch_quantize(uc, row1 - row0, params->n_h, row0, p4, params->pitch_m, d_bits, stream), "quantize");
        return WASABI_OK;
    }
    CK(launch_inverse(reinterpret_cast<const float2 *>(d_psi), reinterpret_cast<float2 *>(d_u), row1 - row0,
                      params->n_h, row0, params->levels, print ? p4 : nullptr, params->pitch_m, d_bits, stream),
       "inverse_wt");
    return WASABI_OK;
}

wasabi_status wasabi_quantize(const wasabi_params *params, const wasabi_print_params *print, const float *d_u,
                              int64_t row0, int64_t row1, uint8_t *d_bits, cudaStream_t stream) {
    wasabi_status st = validate(params);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (!print) return fail(WASABI_EINVAL, "print params NULL");
    if ((!d_u || !d_bits) && row1 > row0) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_u, 16)) return fail(WASABI_EINVAL, "d_u must be 16-byte aligned");
    double p4[4] = {print->x_r_m, print->y_r_m, print->z_r_m, 1.0 / params->wavelength_m};
    CK(launch_quantize(reinterpret_cast<const float2 *>(d_u), row1 - row0, params->n_h, row0, p4, params->pitch_m,
                       d_bits, stream),
       "quantize");
    return WASABI_OK;
}

// ---------------------------------------------------------------- conventional baseline (direct sum)

namespace {
struct DenseLayout {
    std::vector<DenseDesc> dd;
    size_t data_off = 0, bytes = 0;
    int64_t ctas = 0;
};
DenseLayout dense_layout(const Geo &g) {
    // one unshrunk PSF per depth level (side 2H, centre (H, H)), whatever the table mode
    DenseLayout L;
    L.dd.resize(g.nz);
    int64_t off = 0, ctas = 0;
    for (int d = 0; d < g.nz; d++) {
        DenseDesc &D = L.dd[d];
        const int td = d << (2 * g.cb);
        D.z = g.dd[td].z; D.R = g.dd[td].R; D.side = 2 * g.kd[td].H; D.off = off; D.cta_base = (int32_t)ctas;
        off += (int64_t)D.side * D.side;
        const int64_t t = (D.side + 63) / 64;
        ctas += t * t;
    }
    L.ctas = ctas;
    L.data_off = align_up(sizeof(DenseDesc) * g.nz, 256);
    L.bytes = L.data_off + 8 * (size_t)off;
    return L;
}
}  // namespace

wasabi_status wasabi_psf_dense_bytes(const wasabi_params *params, size_t *bytes) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if (bytes) *bytes = dense_layout(g).bytes;
    return WASABI_OK;
}

wasabi_status wasabi_build_psf_dense(const wasabi_params *params, void *d_dense, size_t bytes, cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    DenseLayout L = dense_layout(g);
    if (!d_dense || !aligned(d_dense, 256)) return fail(WASABI_EINVAL, "d_dense NULL or not 256-byte aligned");
    if (bytes < L.bytes) return fail(WASABI_ENOSPC, "dense table buffer needs %zu bytes", L.bytes);
    char *b = static_cast<char *>(d_dense);
    CK(launch_write_blob(b, L.dd.data(), sizeof(DenseDesc) * g.nz, stream), "write dense desc");
    CK(launch_psf_dense(reinterpret_cast<const DenseDesc *>(b), g.nz, reinterpret_cast<float2 *>(b + L.data_off), g.k,
                        params->pitch_m, L.ctas, stream),
       "psf_dense");
    return WASABI_OK;
}

wasabi_status wasabi_direct_sum(const wasabi_params *params, const void *d_dense, const void *d_bins, int64_t row0,
                                int64_t row1, float *d_u, cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (!d_dense || !d_bins || (!d_u && row1 > row0)) return fail(WASABI_EINVAL, "NULL buffer");
    DenseLayout L = dense_layout(g);
    const char *b = static_cast<const char *>(d_dense);
    const int T = params->tile;
    CK(launch_stamp(d_bins, reinterpret_cast<const DenseDesc *>(b), reinterpret_cast<const float2 *>(b + L.data_off),
                    (int)(params->n_h / T), (int)((row1 - row0) / T), row0, params->n_h, T,
                    reinterpret_cast<float2 *>(d_u), stream),
       "direct_sum");
    return WASABI_OK;
}

wasabi_status wasabi_direct_exact(const wasabi_params *params, const float *d_points, int64_t n, const void *d_bins,
                                  int64_t row0, int64_t row1, float *d_u, cudaStream_t stream) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(params, row0, row1)) != WASABI_OK) return st;
    if (!d_bins || (!d_u && row1 > row0) || (n > 0 && !d_points)) return fail(WASABI_EINVAL, "NULL buffer");
    if (n > 0 && !aligned(d_points, 16)) return fail(WASABI_EINVAL, "d_points must be 16-byte aligned");
    const int T = params->tile;
    CK(launch_exact(d_bins, reinterpret_cast<const float4 *>(d_points), (int)(params->n_h / T), (int)((row1 - row0) / T),
                    row0, params->n_h, T, params->pitch_m, g.tan_theta, params->wavelength_m,
                    reinterpret_cast<float2 *>(d_u), stream),
       "direct_exact");
    return WASABI_OK;
}

// ---------------------------------------------------------------- whole path from host buffers

namespace {
struct WsLayout {
    int64_t e0, e1;   // psi band (the band itself, or its coiflet halo band)
    size_t tables, scratch, points, bins, field, bits, total;
    size_t table_bytes, scratch_bytes, bin_bytes;
};
wasabi_status ws_layout(const wasabi_params *P, int64_t n, int64_t row0, int64_t row1, WsLayout &w) {
    Geo g;
    wasabi_status st = compute_geo(P, g);
    if (st != WASABI_OK) return st;
    if ((st = validate_band(P, row0, row1)) != WASABI_OK) return st;
    if (n < 0 || n > (int64_t)INT32_MAX) return fail(WASABI_EINVAL, "n out of range");
    const int64_t Hh = wasabi_coif_halo_rows(P);
    w.e0 = std::max<int64_t>(0, row0 - Hh);
    w.e1 = std::min<int64_t>(P->n_h, row1 + Hh);
    w.table_bytes = g.table_bytes;
    w.scratch_bytes = g.scratch_bytes;
    w.bin_bytes = bin_layout(g, n, w.e0, w.e1).bytes;
    size_t o = 0;
    w.tables = o; o = align_up(o + w.table_bytes, 256);
    w.scratch = o; o = align_up(o + w.scratch_bytes, 256);
    w.points = o; o = align_up(o + 16 * (size_t)n, 256);
    w.bins = o; o = align_up(o + w.bin_bytes, 256);
    w.field = o; o = align_up(o + 8 * (size_t)(w.e1 - w.e0) * (size_t)P->n_h, 256);
    w.bits = o; o = align_up(o + (size_t)(row1 - row0) * (size_t)(P->n_h / 8), 256);
    w.total = o;
    return WASABI_OK;
}
}  // namespace

wasabi_status wasabi_hologram_workspace_bytes(const wasabi_params *params, int64_t n, int64_t row0, int64_t row1,
                                              size_t *workspace_bytes) {
    WsLayout w;
    wasabi_status st = ws_layout(params, n, row0, row1, w);
    if (st != WASABI_OK) return st;
    if (workspace_bytes) *workspace_bytes = w.total;
    return WASABI_OK;
}

wasabi_status wasabi_hologram_host(const wasabi_params *params, const wasabi_print_params *print, const float *h_points,
                                   int64_t n, int64_t row0, int64_t row1, void *d_workspace, size_t workspace_bytes,
                                   uint8_t *h_bits, float *h_u, cudaStream_t stream) {
    WsLayout w;
    wasabi_status st = ws_layout(params, n, row0, row1, w);
    if (st != WASABI_OK) return st;
    if (!print) return fail(WASABI_EINVAL, "print params NULL");
    if (!d_workspace || (n > 0 && !h_points)) return fail(WASABI_EINVAL, "NULL buffer");
    if (!aligned(d_workspace, 256)) return fail(WASABI_EINVAL, "workspace must be 256-byte aligned");
    if (workspace_bytes < w.total) return fail(WASABI_ENOSPC, "workspace needs %zu bytes", w.total);
    char *ws = static_cast<char *>(d_workspace);
    float *d_pts = reinterpret_cast<float *>(ws + w.points);
    float *d_field = reinterpret_cast<float *>(ws + w.field);
    uint8_t *d_bits = reinterpret_cast<uint8_t *>(ws + w.bits);
    // A side stream carries the copies: the points' H2D overlaps the table build, and the bits / u
    // of each row chunk go to the host while the next chunk is superposed (PCIe under the compute).
    // The copy stream and the join event are created once per host thread and device and reused
    // (no per-call stream/event creation).
    struct CopyCtx {
        int dev = -1;
        cudaStream_t cs = nullptr;
        cudaEvent_t ev = nullptr;
    };
    thread_local CopyCtx ctx;
    int dev = 0;
    CK(cudaGetDevice(&dev), "current device");
    if (ctx.dev != dev) {
        if (ctx.cs) cudaStreamDestroy(ctx.cs);   // another device: release the old pair
        if (ctx.ev) cudaEventDestroy(ctx.ev);
        ctx.cs = nullptr; ctx.ev = nullptr; ctx.dev = -1;
        CK(cudaStreamCreateWithFlags(&ctx.cs, cudaStreamNonBlocking), "copy stream");
        CK(cudaEventCreateWithFlags(&ctx.ev, cudaEventDisableTiming), "join event");
        ctx.dev = dev;
    }
    cudaStream_t cs = ctx.cs;
    // record + wait are enqueued at once (the wait captures the event's state at the call), so one
    // event serves every join
    auto join = [&](cudaStream_t waiter, cudaStream_t waited) -> cudaError_t {
        cudaError_t r = cudaEventRecord(ctx.ev, waited);
        if (r == cudaSuccess) r = cudaStreamWaitEvent(waiter, ctx.ev, 0);
        return r;
    };
    CK(join(cs, stream), "order copy stream");
    if (n > 0) CK(cudaMemcpyAsync(d_pts, h_points, 16 * (size_t)n, cudaMemcpyHostToDevice, cs), "H2D points");
    if ((st = wasabi_build_psf_tables(params, ws + w.tables, w.table_bytes, ws + w.scratch, w.scratch_bytes, stream)))
        return st;
    CK(join(stream, cs), "wait for points");
    if ((st = wasabi_bin_points(params, ws + w.tables, d_pts, n, w.e0, w.e1, ws + w.bins, w.bin_bytes, stream)))
        return st;
    const size_t bpr = (size_t)(params->n_h / 8), upr = 8 * (size_t)params->n_h;   // bytes per row
    if (params->flags & WASABI_FLAG_COIFLET) {   // unfused: psi on the halo band, coif1 synthesis, bits
        if ((st = wasabi_superpose(params, ws + w.tables, ws + w.bins, w.e0, w.e1, d_field, stream))) return st;
        // with u wanted: in place on the halo band (u = its rows [row0, row1)); print only: fused tiles
        float *d_urows = d_field + 2 * (row0 - w.e0) * params->n_h;   // u rows [row0, row1) inside the halo band
        if ((st = wasabi_inverse_wt(params, d_field, h_u ? d_urows : nullptr, row0, row1, print, d_bits, stream)))
            return st;
        d_field = d_urows;
        CK(join(cs, stream), "wait for u");
        if (h_bits && row1 > row0)
            CK(cudaMemcpyAsync(h_bits, d_bits, bpr * (size_t)(row1 - row0), cudaMemcpyDeviceToHost, cs), "D2H bits");
        if (h_u && row1 > row0)
            CK(cudaMemcpyAsync(h_u, d_field, upr * (size_t)(row1 - row0), cudaMemcpyDeviceToHost, cs), "D2H u");
    } else if (row1 > row0) {
        const int T = params->tile;
        const int tiles_y = (int)((row1 - row0) / T);
        const int chunk = std::max(1, (tiles_y + 7) / 8);   // 8 row chunks
        double p4[4] = {print->x_r_m, print->y_r_m, print->z_r_m, 1.0 / params->wavelength_m};
        for (int ty = 0; ty < tiles_y; ty += chunk) {
            const int ty1 = std::min(tiles_y, ty + chunk);
            CK(launch_sup(*params, ws + w.bins, ws + w.tables, row0, tiles_y,
                          h_u ? reinterpret_cast<float2 *>(d_field) : nullptr, 1, p4, d_bits, stream, ty, ty1),
               "superpose_inverse chunk");
            CK(join(cs, stream), "chunk done");
            const size_t r0 = (size_t)ty * T, nr = (size_t)(ty1 - ty) * T;
            if (h_bits) CK(cudaMemcpyAsync(h_bits + r0 * bpr, d_bits + r0 * bpr, nr * bpr, cudaMemcpyDeviceToHost, cs),
                           "D2H bits");
            if (h_u)
                CK(cudaMemcpyAsync(reinterpret_cast<char *>(h_u) + r0 * upr,
                                   reinterpret_cast<char *>(d_field) + r0 * upr, nr * upr, cudaMemcpyDeviceToHost, cs),
                   "D2H u");
        }
    }
    CK(join(stream, cs), "join copy stream");   // the caller's stream covers every copy
    return WASABI_OK;
}

// ---------------------------------------------------------------- diagnostics

wasabi_status wasabi_tables_check(const wasabi_params *params, const void *d_tables) {
    wasabi_status st = validate(params);
    if (st != WASABI_OK) return st;
    TableHeader h;
    CK(cudaMemcpy(&h, d_tables, sizeof h, cudaMemcpyDeviceToHost), "read table header");
    if (h.magic != kTableMagic) return fail(WASABI_ESTATE, "not a WASABI table buffer");
    if (h.param_hash != param_hash(*params)) return fail(WASABI_ESTATE, "table buffer was built with other params");
    return WASABI_OK;
}

wasabi_status wasabi_export_reach(const wasabi_params *params, const void *d_tables, int32_t depth, int32_t *h_ek,
                                  int32_t *h_q) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if ((st = wasabi_tables_check(params, d_tables)) != WASABI_OK) return st;
    if (depth < 0 || depth >= g.nd) return fail(WASABI_EINVAL, "depth out of range");
    if (!h_ek || !h_q) return fail(WASABI_EINVAL, "null output");
    KDesc K;
    CK(cudaMemcpy(&K, static_cast<const char *>(d_tables) + g.th.kdesc_off + sizeof(KDesc) * (size_t)depth,
                  sizeof K, cudaMemcpyDeviceToHost),
       "read kdesc");
    *h_ek = K.Ek;
    *h_q = K.Q;
    return WASABI_OK;
}

wasabi_status wasabi_export_table(const wasabi_params *params, const void *d_tables, int32_t depth, int32_t *h_level,
                                  int32_t *h_dx, int32_t *h_dy, float *h_val, int64_t cap, int64_t *n_out) {
    Geo g;
    wasabi_status st = compute_geo(params, g);
    if (st != WASABI_OK) return st;
    if ((st = wasabi_tables_check(params, d_tables)) != WASABI_OK) return st;
    if (depth < 0 || depth >= g.nd) return fail(WASABI_EINVAL, "depth out of range");
    const char *tb = static_cast<const char *>(d_tables);
    const KDesc K = g.kd[depth];
    const DDesc D = g.dd[depth];
    std::vector<int32_t> ptr(D.n_groups + 1);
    CK(cudaMemcpy(ptr.data(), tb + g.th.ptr_off + 4 * (size_t)D.group_base, 4 * ptr.size(), cudaMemcpyDeviceToHost),
       "read ptr");
    const int64_t e0 = ptr[0], e1 = ptr[D.n_groups];
    const int64_t n = e1 - e0;
    if (n_out) *n_out = n;
    if (n != D.n_r) return fail(WASABI_ESTATE, "depth %d holds %lld entries, expected N_r = %lld", depth,
                                (long long)n, (long long)D.n_r);
    if (cap < n) return fail(WASABI_ENOSPC, "need capacity %lld", (long long)n);
    std::vector<uint32_t> ent(4 * (size_t)n);
    if (n)
        CK(cudaMemcpy(ent.data(), tb + g.th.ent_off + 16 * (size_t)e0, 16 * (size_t)n, cudaMemcpyDeviceToHost),
           "read entries");
    struct Rec { int32_t l, Y, X; int64_t i; };
    std::vector<Rec> rec;
    rec.reserve(n);
    for (int64_t i = 0; i < n; i++) {
        const uint32_t p = ent[4 * i];
        rec.push_back(Rec{(int32_t)(p >> 28), (int32_t)((p >> 14) & 0x3fff), (int32_t)(p & 0x3fff), i});
    }
    const int64_t H = K.H;
    std::sort(rec.begin(), rec.end(), [](const Rec &a, const Rec &b) {
        if (a.l != b.l) return a.l < b.l;
        if (a.Y != b.Y) return a.Y < b.Y;
        return a.X < b.X;
    });
    for (int64_t k = 0; k < n; k++) {
        if (h_level) h_level[k] = rec[k].l;
        if (h_dx) h_dx[k] = (int32_t)(rec[k].X - H);
        if (h_dy) h_dy[k] = (int32_t)(rec[k].Y - H);
        if (h_val) {
            memcpy(&h_val[2 * k], &ent[4 * rec[k].i + 1], 4);
            memcpy(&h_val[2 * k + 1], &ent[4 * rec[k].i + 2], 4);
        }
    }
    return WASABI_OK;
}

wasabi_status wasabi_bins_stats(const void *d_bins, int64_t out[8]) {
    if (!d_bins || !out) return fail(WASABI_EINVAL, "NULL argument");
    BinHeader h;
    CK(cudaMemcpy(&h, d_bins, sizeof h, cudaMemcpyDeviceToHost), "read bin header");
    if (h.magic != kBinMagic) return fail(WASABI_ESTATE, "not a WASABI bin buffer");
    out[0] = (int64_t)h.n_valid; out[1] = (int64_t)h.n_skipped; out[2] = (int64_t)h.total_entries;
    out[3] = h.capacity; out[4] = h.row0; out[5] = h.row1; out[6] = h.n_tiles; out[7] = (int64_t)h.status;
    return WASABI_OK;
}

wasabi_status wasabi_export_bins(const wasabi_params *params, const void *d_bins, int64_t *h_tile_ptr,
                                 int32_t *h_point_idx, int64_t cap, int64_t *n_out) {
    wasabi_status st = validate(params);
    if (st != WASABI_OK) return st;
    BinHeader h;
    CK(cudaMemcpy(&h, d_bins, sizeof h, cudaMemcpyDeviceToHost), "read bin header");
    if (h.magic != kBinMagic) return fail(WASABI_ESTATE, "not a WASABI bin buffer");
    if (h.param_hash != param_hash(*params)) return fail(WASABI_ESTATE, "bins were built with other params");
    if (h.status) return fail(WASABI_ESTATE, "bin buffer overflowed (status %llu)", (unsigned long long)h.status);
    const char *bb = static_cast<const char *>(d_bins);
    std::vector<unsigned long long> ptr(h.n_tiles + 1);
    CK(cudaMemcpy(ptr.data(), bb + h.ptr_off, 8 * ptr.size(), cudaMemcpyDeviceToHost), "read bin ptr");
    const int64_t n = (int64_t)ptr[h.n_tiles];
    if (n_out) *n_out = n;
    if (h_tile_ptr)
        for (int64_t i = 0; i <= h.n_tiles; i++) h_tile_ptr[i] = (int64_t)ptr[i];
    if (h_point_idx) {
        if (cap < n) return fail(WASABI_ENOSPC, "need capacity %lld", (long long)n);
        if (n) CK(cudaMemcpy(h_point_idx, bb + h.idx_off, 4 * (size_t)n, cudaMemcpyDeviceToHost), "read bin idx");
    }
    return WASABI_OK;
}

}  // extern "C"
