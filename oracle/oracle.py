"""ctypes wrapper of the fp64 C oracle (oracle/wasabi_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product path (paper_1708_04233_b200) never
imports this module and shares no code with it.  Argument marshalling only: every step
of the oracle's arithmetic is in the C file, which cites the paper passage it follows.
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "wasabi_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, fp64, no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c11", "-fPIC",
                               "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


class _Params(C.Structure):
    _fields_ = [("wavelength", C.c_double), ("pitch", C.c_double), ("n_h", C.c_int64),
                ("n_depth", C.c_int32), ("levels", C.c_int32), ("z_min", C.c_double),
                ("z_max", C.c_double), ("retention", C.c_double), ("exact", C.c_int32), ("wavelet", C.c_int32)]


@dataclasses.dataclass(frozen=True)
class Params:
    wavelength: float
    pitch: float
    n_h: int
    n_depth: int
    levels: int
    z_min: float
    z_max: float
    retention: float
    exact: bool = False      # R-A20 offset-class tables
    wavelet: int = 0         # 0 Haar (R-A1), 1 coif1 (R-A21)

    @staticmethod
    def from_config(cfg, exact: bool = False, wavelet: int = 0) -> "Params":
        return Params(cfg.wavelength, cfg.pitch, cfg.n_h, cfg.n_depth, cfg.levels, cfg.z_min,
                      cfg.z_max, cfg.retention, exact, wavelet)

    @property
    def n_tables(self) -> int:
        return self.n_depth << (2 * self.levels) if self.exact else self.n_depth

    def table_index(self, ix, iy, iz):
        """Table of a point (R-A20): iz, or iz 4^L + (iy mod 2^L) 2^L + (ix mod 2^L) in exact mode."""
        if not self.exact:
            return iz
        m = (1 << self.levels) - 1
        return (np.asarray(iz, np.int64) << (2 * self.levels)) | ((np.asarray(iy) & m) << self.levels) | (np.asarray(ix) & m)

    def c(self) -> _Params:
        return _Params(self.wavelength, self.pitch, self.n_h, self.n_depth, self.levels, self.z_min,
                       self.z_max, self.retention, int(self.exact), int(self.wavelet))


_dp = C.POINTER(C.c_double)
_i64p = C.POINTER(C.c_int64)
_i32p = C.POINTER(C.c_int32)
_i8p = C.POINTER(C.c_int8)
_u8p = C.POINTER(C.c_uint8)
_pp = C.POINTER(_Params)


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = C.CDLL(build())
            L.orc_geometry.argtypes = [_pp, _dp, _dp, _i64p, _i64p, _i64p, _i64p]
            L.orc_depth_info.argtypes = [_pp, C.c_int, _dp, _i64p]
            L.orc_psf_table.argtypes = [_pp, C.c_int64, _dp]
            L.orc_haar_fwd.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, C.c_int]
            L.orc_haar_inv.argtypes = [_dp, C.c_int64, C.c_int64, C.c_int64, C.c_int]
            L.orc_table_coeffs.argtypes = [_pp, C.c_int64, _dp]
            L.orc_select.argtypes = [_pp, C.c_int64, _i32p, _i32p, _i32p, _dp, C.c_int64]
            L.orc_table_info.argtypes = [_pp, C.c_int64, _i64p]
            L.orc_filter_bank.argtypes = [C.c_int, _dp, _dp, C.POINTER(C.c_int)]
            L.orc_fb_fwd.argtypes = [C.c_int, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int]
            L.orc_fb_inv.argtypes = [C.c_int, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int]
            L.orc_nnz_footprint.argtypes = [_pp, C.c_int64]
            L.orc_nnz_footprint.restype = C.c_int64
            L.orc_hologram_window.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                              C.c_int64, _dp, _dp]
            L.orc_hologram_window.restype = C.c_int64
            L.orc_n_tables.argtypes = [_pp]
            L.orc_n_tables.restype = C.c_int64
            L.orc_select.restype = C.c_int64
            L.orc_lut_new.argtypes = [_pp]
            L.orc_lut_new.restype = C.c_void_p
            L.orc_lut_free.argtypes = [C.c_void_p]
            L.orc_lut_build_depth.argtypes = [C.c_void_p, C.c_int64]
            L.orc_lut_build_depth.restype = C.c_int64
            L.orc_points.argtypes = [_pp, _dp, C.c_int64, _i64p, _i64p, _i32p, _i8p]
            L.orc_lut_reach.argtypes = [C.c_void_p, C.c_int64, _i64p, _i64p]
            L.orc_bins.argtypes = [_pp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p,
                                   _i64p, _i32p, C.c_int64]
            L.orc_bins.restype = C.c_int64
            L.orc_bin_tile.argtypes = [_pp, C.c_int64, _dp, C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p,
                                       _i32p, C.c_int64]
            L.orc_bin_tile.restype = C.c_int64
            L.orc_wasabi_window.argtypes = [C.c_void_p, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                            C.c_int64, _dp]
            L.orc_wasabi_window.restype = C.c_int64
            L.orc_quantize.argtypes = [_pp, C.c_double, C.c_double, C.c_double, _dp, C.c_int64,
                                       C.c_int64, C.c_int64, C.c_int64, _u8p, _dp]
            L.orc_direct_d1.argtypes = [_pp, _dp, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                                        _dp]
            L.orc_direct_d2.argtypes = L.orc_direct_d1.argtypes
            L.orc_level_shift.argtypes = [_pp, C.c_int64, C.c_int]
            L.orc_level_shift.restype = C.c_int64
            _lib = L
    return _lib


def _ptr(a, t):
    return a.ctypes.data_as(t)


def _pts64(pts) -> np.ndarray:
    a = np.ascontiguousarray(np.asarray(pts, dtype=np.float64).reshape(-1, 4))
    return a


def _cplx_buf(z: np.ndarray) -> np.ndarray:
    """complex128 (h, w) -> contiguous float64 (h, w, 2) view copy."""
    return np.ascontiguousarray(z.astype(np.complex128)).view(np.float64).reshape(z.shape + (2,))


def geometry(P: Params) -> dict:
    n = P.n_depth
    z = np.zeros(n); R = np.zeros(n)
    H = np.zeros(n, np.int64); E = np.zeros(n, np.int64)
    nnz = np.zeros(n, np.int64); nr = np.zeros(n, np.int64)
    lib().orc_geometry(C.byref(P.c()), _ptr(z, _dp), _ptr(R, _dp), _ptr(H, _i64p), _ptr(E, _i64p),
                       _ptr(nnz, _i64p), _ptr(nr, _i64p))
    return dict(z=z, R=R, H=H, E=E, nnz=nnz, n_r=nr)


def table_info(P: Params, t: int) -> dict:
    """Table t (R-A20): H (aligned centre), side, structural nnz, N_r."""
    h = np.zeros(4, np.int64)
    lib().orc_table_info(C.byref(P.c()), int(t), _ptr(h, _i64p))
    return dict(H=int(h[0]), side=int(h[1]), nnz=int(h[2]), n_r=int(h[3]))


def psf_table(P: Params, d: int) -> np.ndarray:
    side = table_info(P, d)["side"]
    f = np.zeros((side, side, 2))
    lib().orc_psf_table(C.byref(P.c()), d, _ptr(f, _dp))
    return f[..., 0] + 1j * f[..., 1]


def geometry_one(P: Params, d: int) -> dict:
    zr = np.zeros(2)
    hen = np.zeros(4, np.int64)
    lib().orc_depth_info(C.byref(P.c()), d, _ptr(zr, _dp), _ptr(hen, _i64p))
    return dict(z=zr[0], R=zr[1], H=int(hen[0]), E=int(hen[1]), nnz=int(hen[2]), n_r=int(hen[3]))


def haar_fwd(f: np.ndarray, L: int) -> np.ndarray:
    b = _cplx_buf(f)
    h, w = f.shape
    lib().orc_haar_fwd(_ptr(b, _dp), h, w, w, L)
    return b[..., 0] + 1j * b[..., 1]


def filter_bank(wavelet: int):
    """(h0, h1, off) of the wavelet's analysis filters (R-A21: coif1 closed form; Haar)."""
    h0 = np.zeros(6); h1 = np.zeros(6); off = C.c_int()
    taps = lib().orc_filter_bank(wavelet, _ptr(h0, _dp), _ptr(h1, _dp), C.byref(off))
    return h0[:taps], h1[:taps], off.value


def fb_fwd(wavelet: int, f: np.ndarray, L: int) -> np.ndarray:
    b = _cplx_buf(f)
    h, w = f.shape
    lib().orc_fb_fwd(wavelet, _ptr(b, _dp), h, w, w, L)
    return b[..., 0] + 1j * b[..., 1]


def fb_inv(wavelet: int, f: np.ndarray, L: int) -> np.ndarray:
    b = _cplx_buf(f)
    h, w = f.shape
    lib().orc_fb_inv(wavelet, _ptr(b, _dp), h, w, w, L)
    return b[..., 0] + 1j * b[..., 1]


def nnz_footprint(P: Params, t: int) -> int:
    return int(lib().orc_nnz_footprint(C.byref(P.c()), int(t)))


def haar_inv(f: np.ndarray, L: int) -> np.ndarray:
    b = _cplx_buf(f)
    h, w = f.shape
    lib().orc_haar_inv(_ptr(b, _dp), h, w, w, L)
    return b[..., 0] + 1j * b[..., 1]


def table_coeffs(P: Params, d: int, H: int = None) -> np.ndarray:
    side = table_info(P, d)["side"]
    c = np.zeros((side, side, 2))
    lib().orc_table_coeffs(C.byref(P.c()), d, _ptr(c, _dp))
    return c[..., 0] + 1j * c[..., 1]


def select(P: Params, d: int, cap: int):
    lv = np.zeros(cap, np.int32); dx = np.zeros(cap, np.int32); dy = np.zeros(cap, np.int32)
    val = np.zeros((cap, 2))
    n = lib().orc_select(C.byref(P.c()), d, _ptr(lv, _i32p), _ptr(dx, _i32p), _ptr(dy, _i32p),
                         _ptr(val, _dp), cap)
    if n < 0:
        raise ValueError("cap too small")
    return lv[:n], dx[:n], dy[:n], val[:n, 0] + 1j * val[:n, 1]


def points(P: Params, pts):
    p = _pts64(pts)
    n = p.shape[0]
    ix = np.zeros(n, np.int64); iy = np.zeros(n, np.int64); iz = np.zeros(n, np.int32)
    ok = np.zeros(n, np.int8)
    lib().orc_points(C.byref(P.c()), _ptr(p, _dp), n, _ptr(ix, _i64p), _ptr(iy, _i64p), _ptr(iz, _i32p),
                     _ptr(ok, _i8p))
    return ix, iy, iz, ok.astype(bool)


_reach_cache = {}


def reach(P: Params):
    """Per-depth footprint reach (ek, q) of the kept lists (orc_lut_reach, R-A19); cached per params."""
    key = tuple(sorted(P.__dict__.items()))
    if key not in _reach_cache:
        lut = Lut(P)
        ek = np.zeros(P.n_tables, np.int64)
        q = np.zeros(P.n_tables, np.int64)
        for d in range(P.n_tables):
            a = np.zeros(1, np.int64); b = np.zeros(1, np.int64)
            lib().orc_lut_reach(lut.h, d, _ptr(a, _i64p), _ptr(b, _i64p))
            ek[d] = a[0]; q[d] = b[0]
        lut.close()
        _reach_cache[key] = (ek, q)
    return _reach_cache[key]


def reach_one(P: Params, d: int):
    """(ek, q) of one depth (orc_lut_reach)."""
    lut = Lut(P)
    a = np.zeros(1, np.int64); b = np.zeros(1, np.int64)
    lib().orc_lut_reach(lut.h, d, _ptr(a, _i64p), _ptr(b, _i64p))
    lut.close()
    return int(a[0]), int(b[0])


def bins(P: Params, T: int, pts, row0: int, row1: int, cap: int = None):
    ek, q = reach(P)
    p = _pts64(pts)
    n = p.shape[0]
    nt = (P.n_h // T) * ((row1 - row0) // T)
    ptr = np.zeros(nt + 1, np.int64)
    cap = cap if cap is not None else max(1, n * 16)
    while True:
        idx = np.zeros(cap, np.int32)
        tot = lib().orc_bins(C.byref(P.c()), T, _ptr(p, _dp), n, row0, row1, _ptr(ek, _i64p), _ptr(q, _i64p),
                             _ptr(ptr, _i64p), _ptr(idx, _i32p), cap)
        if tot >= 0:
            return ptr, idx[:tot]
        cap = -tot


def bin_tile(P: Params, T: int, pts, X0: int, Y0: int) -> np.ndarray:
    ek, q = reach(P)
    p = _pts64(pts)
    n = p.shape[0]
    cap = max(1, n)
    idx = np.zeros(cap, np.int32)
    tot = lib().orc_bin_tile(C.byref(P.c()), T, _ptr(p, _dp), n, X0, Y0, _ptr(ek, _i64p), _ptr(q, _i64p),
                             _ptr(idx, _i32p), cap)
    return idx[:tot]


class Lut:
    """Lazily built per-depth lists (orc_select) kept for repeated windows."""

    def __init__(self, P: Params):
        self.P = P
        self._c = P.c()
        self.h = lib().orc_lut_new(C.byref(self._c))

    def build_depth(self, d: int) -> int:
        return lib().orc_lut_build_depth(self.h, d)

    def wasabi_window(self, pts, x0: int, y0: int, w: int, h: int):
        """psi on hologram window [x0, x0+w) x [y0, y0+h) (Eq.(2)); returns (psi complex128, count)."""
        p = _pts64(pts)
        psi = np.zeros((h, w, 2))
        cnt = lib().orc_wasabi_window(self.h, _ptr(p, _dp), p.shape[0], x0, y0, w, h, _ptr(psi, _dp))
        return psi[..., 0] + 1j * psi[..., 1], cnt

    def hologram_window(self, pts, x0: int, y0: int, w: int, h: int):
        """u = inverse FWT of psi on a 2^L-aligned window (steps 2-3; orc_hologram_window)."""
        p = _pts64(pts)
        u = np.zeros((h, w, 2))
        psi = np.zeros((h, w, 2))
        cnt = lib().orc_hologram_window(self.h, _ptr(p, _dp), p.shape[0], x0, y0, w, h, _ptr(u, _dp),
                                        _ptr(psi, _dp))
        return u[..., 0] + 1j * u[..., 1], psi[..., 0] + 1j * psi[..., 1], cnt

    def close(self):
        if self.h:
            lib().orc_lut_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def quantize(P: Params, ref, u: np.ndarray, x0: int, y0: int):
    h, w = u.shape
    b = _cplx_buf(u)
    bits = np.zeros((h, w // 8), np.uint8)
    I = np.zeros((h, w))
    lib().orc_quantize(C.byref(P.c()), float(ref[0]), float(ref[1]), float(ref[2]), _ptr(b, _dp), x0, y0,
                       w, h, _ptr(bits, _u8p), _ptr(I, _dp))
    return bits, I


def level_shift(P: Params, i: int, l: int) -> int:
    """The oracle's level-l coefficient shift s_l(i) of pixel index i (R-A8; R-A20 in exact mode)."""
    return int(lib().orc_level_shift(C.byref(P.c()), int(i), int(l)))


def direct_d1(P: Params, pts, x0: int, y0: int, w: int, h: int) -> np.ndarray:
    p = _pts64(pts)
    u = np.zeros((h, w, 2))
    lib().orc_direct_d1(C.byref(P.c()), _ptr(p, _dp), p.shape[0], x0, y0, w, h, _ptr(u, _dp))
    return u[..., 0] + 1j * u[..., 1]


def direct_d2(P: Params, pts, x0: int, y0: int, w: int, h: int) -> np.ndarray:
    p = _pts64(pts)
    u = np.zeros((h, w, 2))
    lib().orc_direct_d2(C.byref(P.c()), _ptr(p, _dp), p.shape[0], x0, y0, w, h, _ptr(u, _dp))
    return u[..., 0] + 1j * u[..., 1]
