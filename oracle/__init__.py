"""Parity ORACLE (test infrastructure only).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
``--impl reference`` legs may import this package.  It wraps ``liboracle.so``
(oracle/oracle.cpp), a plain fp64 CPU implementation of GS(p), SpMV, the
canonical dot product, SELL-C-sigma layout, Bi-CGSTAB and GMRES(m) written from
the paper (see the header of oracle.cpp for the passages and DESIGN.md §4 for the
arithmetic contract).  It shares no code with ``paper_0812_2769_b200``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

STATUS = {0: "CONVERGED", 1: "MAXIT", 2: "BREAKDOWN", 3: "DIVERGED"}


class Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("history_len", ctypes.c_int32),
                ("breakdown_at", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("relres", ctypes.c_double), ("true_relres", ctypes.c_double),
                ("true_relres_w", ctypes.c_double), ("best_relres", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run make (or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        vp, i64, d, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        lib.orc_num_threads.restype = i32
        lib.orc_dot.argtypes = [i64, vp, vp]
        lib.orc_dot.restype = d
        lib.orc_wnorm2.argtypes = [i64, vp, vp]
        lib.orc_wnorm2.restype = d
        lib.orc_spmv.argtypes = [i64, vp, vp, vp, vp, vp]
        lib.orc_spmv.restype = None
        lib.orc_gs_scale.argtypes = [i64, vp, vp, vp, i32, vp, vp, vp, vp]
        lib.orc_gs_scale.restype = i32
        lib.orc_gs_scale_sym.argtypes = [i64, vp, vp, vp, vp, i32, vp, vp, vp, vp]
        lib.orc_gs_scale_sym.restype = i32
        lib.orc_unscale.argtypes = [i64, vp, vp, vp]
        lib.orc_unscale.restype = None
        lib.orc_sell_size.argtypes = [i64, vp, i32, i32]
        lib.orc_sell_size.restype = i64
        lib.orc_sell_build.argtypes = [i64, vp, vp, vp, i32, i32, vp, vp, vp, vp, vp]
        lib.orc_sell_build.restype = i32
        lib.orc_sell_dict_size.argtypes = [i64, i32, i32, vp, vp, vp]
        lib.orc_sell_dict_size.restype = i64
        lib.orc_sell_dict.argtypes = [i64, i32, i32, vp, vp, vp, vp, vp, vp]
        lib.orc_sell_dict.restype = i32
        lib.orc_set_fault.argtypes = [i32, i32]
        lib.orc_set_fault.restype = None
        lib.orc_sell_uniform.argtypes = [i64, i32, i32, i32] + [vp] * 8
        lib.orc_sell_uniform.restype = i64
        lib.orc_row_classes.argtypes = [i64, vp, vp, vp, i32, i32, vp, vp, vp, vp]
        lib.orc_row_classes.restype = i64
        lib.orc_bicgstab.argtypes = [i64, vp, vp, vp, vp, vp, vp, d, i32, vp, vp,
                                     ctypes.POINTER(Report)]
        lib.orc_bicgstab.restype = i32
        lib.orc_gmres.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, d, i32, vp, vp,
                                  ctypes.POINTER(Report)]
        lib.orc_gmres.restype = i32
        lib.orc_gmres_orth.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, d, i32, i32, vp, vp,
                                       ctypes.POINTER(Report)]
        lib.orc_gmres_orth.restype = i32
        lib.orc_gmres_wstop.argtypes = [i64, vp, vp, vp, vp, vp, vp, i32, d, i32, i32, i32, vp, vp,
                                        ctypes.POINTER(Report)]
        lib.orc_gmres_wstop.restype = i32
        _LIB = lib
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data


def _f64(a):
    return None if a is None else np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


def num_threads() -> int:
    return _lib().orc_num_threads()


def dot(a, b) -> float:
    a, b = _f64(a), _f64(b)
    return _lib().orc_dot(a.size, _p(a), _p(b))


def wnorm2(a, w=None) -> float:
    a, w = _f64(a), _f64(w)
    return _lib().orc_wnorm2(a.size, _p(a), _p(w))


def spmv(row_ptr, col, val, x):
    row_ptr, col, val, x = _i32(row_ptr), _i32(col), _f64(val), _f64(x)
    n = row_ptr.size - 1
    y = np.empty(n, np.float64)
    _lib().orc_spmv(n, _p(row_ptr), _p(col), _p(val), _p(x), _p(y))
    return y


class ZeroRowError(ValueError):
    def __init__(self, row):
        super().__init__(f"row {row} has zero L_p norm")
        self.row = row


def gs_scale(row_ptr, val, b, p):
    """Return (val', b', d) = (D A, D b, diag D) with D = diag(1/||a_i||_p)."""
    row_ptr, val = _i32(row_ptr), _f64(val)
    b = _f64(b)
    n = row_ptr.size - 1
    vo = np.empty_like(val)
    bo = None if b is None else np.empty_like(b)
    d = np.empty(n, np.float64)
    bad = ctypes.c_int32(-1)
    rc = _lib().orc_gs_scale(n, _p(row_ptr), _p(val), _p(b), int(p), _p(vo), _p(bo), _p(d),
                             ctypes.addressof(bad))
    if rc == -1:
        raise ValueError("p must be >= 1")
    if rc == -2:
        raise ZeroRowError(bad.value)
    return vo, bo, d


def gs_scale_sym(row_ptr, col, val, b, p):
    """Two-sided scaling: returns (val', b', s) with
    A' = D^1/2 A D^1/2, b' = D^1/2 b, s = diag(D^1/2)."""
    row_ptr, col, val, b = _i32(row_ptr), _i32(col), _f64(val), _f64(b)
    n = row_ptr.size - 1
    vo = np.empty_like(val)
    bo = None if b is None else np.empty_like(b)
    sv = np.empty(n, np.float64)
    bad = ctypes.c_int32(-1)
    rc = _lib().orc_gs_scale_sym(n, _p(row_ptr), _p(col), _p(val), _p(b), int(p), _p(vo), _p(bo),
                                 _p(sv), ctypes.addressof(bad))
    if rc == -1:
        raise ValueError("p must be >= 1")
    if rc == -2:
        raise ZeroRowError(bad.value)
    return vo, bo, sv


def unscale(s, y):
    """x = D^1/2 y."""
    s, y = _f64(s), _f64(y)
    x = np.empty_like(y)
    _lib().orc_unscale(y.size, _p(s), _p(y), _p(x))
    return x


def sell_build(row_ptr, col, val, C=32, sigma=256):
    row_ptr, col, val = _i32(row_ptr), _i32(col), _f64(val)
    n = row_ptr.size - 1
    nch = (n + C - 1) // C
    tot = _lib().orc_sell_size(n, _p(row_ptr), C, sigma)
    out = {"chunk_ptr": np.zeros(nch + 1, np.int32), "chunk_len": np.zeros(nch, np.int32),
           "scol": np.zeros(tot, np.int32), "sval": np.zeros(tot, np.float64),
           "roff": np.zeros(nch * C, np.uint8)}
    rc = _lib().orc_sell_build(n, _p(row_ptr), _p(col), _p(val), C, sigma,
                               *(_p(out[k]) for k in ("chunk_ptr", "chunk_len", "scol", "sval", "roff")))
    if rc != 0:
        raise ValueError("bad SELL parameters")
    return out


def sell_dict(n, S, C=32, sigma=256):
    """Delta-dictionary encoding of a SELL layout's column indices (None if some chunk
    has more than 32 distinct col - row deltas)."""
    cp, sc, ro = _i32(S["chunk_ptr"]), _i32(S["scol"]), np.ascontiguousarray(S["roff"], np.uint8)
    tot = _lib().orc_sell_dict_size(n, C, sigma, _p(cp), _p(sc), _p(ro))
    if tot < 0:
        return None
    nch = (n + C - 1) // C
    out = {"dict_ptr": np.zeros(nch + 1, np.int32), "dict": np.zeros(max(tot, 1), np.int32),
           "sidx": np.zeros(sc.size, np.uint8)}
    rc = _lib().orc_sell_dict(n, C, sigma, _p(cp), _p(sc), _p(ro), _p(out["dict_ptr"]), _p(out["dict"]),
                              _p(out["sidx"]))
    if rc != 0:
        return None
    out["dict"] = out["dict"][:tot]
    return out


def sell_uniform(row_ptr, col, val, S, C=32, sigma=256, maxu=8):
    """SELL-U encoding (chunk-uniform column deltas) of a SELL layout S (sell_build):
    uptr, udel, umask, uval — or None if some chunk has more than maxu deltas."""
    row_ptr, col, val = _i32(row_ptr), _i32(col), _f64(val)
    ro = np.ascontiguousarray(S["roff"], np.uint8)
    n = row_ptr.size - 1
    nch = (n + C - 1) // C
    tot = _lib().orc_sell_uniform(n, C, sigma, maxu, _p(ro), _p(row_ptr), _p(col), _p(val), None, None, None, None)
    if tot < 0:
        return None
    out = {"uptr": np.zeros(nch + 1, np.int32), "udel": np.zeros(nch * maxu, np.int32),
           "umask": np.zeros(nch * maxu, np.uint32), "uval": np.zeros(max(tot, 1), np.float64)}
    _lib().orc_sell_uniform(n, C, sigma, maxu, _p(ro), _p(row_ptr), _p(col), _p(val),
                            *(_p(out[k]) for k in ("uptr", "udel", "umask", "uval")))
    out["uval"] = out["uval"][:tot]
    return out


def row_classes(row_ptr, col, val, maxlen=8, maxcls=4096):
    """Row-class dictionary of a CSR matrix (oracle.cpp, "RCD"): rows with the same
    length, deltas col - row and bit-identical values share a class, numbered by first
    occurrence.  Returns {"cls" uint16 [n], "len" int32 [K], "delta" int32 [K, maxlen],
    "val" float64 [K, maxlen]} or None when a row is longer than maxlen or there are more
    than maxcls classes."""
    row_ptr, col, val = _i32(row_ptr), _i32(col), _f64(val)
    n = row_ptr.size - 1
    cls = np.zeros(n, np.uint16)
    dlen = np.zeros(maxcls, np.int32)
    ddel = np.zeros((maxcls, maxlen), np.int32)
    dval = np.zeros((maxcls, maxlen), np.float64)
    k = _lib().orc_row_classes(n, _p(row_ptr), _p(col), _p(val), maxlen, maxcls,
                               _p(cls), _p(dlen), _p(ddel), _p(dval))
    if k < 0:
        return None
    return {"cls": cls, "len": dlen[:k].copy(), "delta": ddel[:k].copy(), "val": dval[:k].copy()}


FAULTS = {"none": 0, "rho0": 1, "omega0": 2, "nan": 3}


def set_fault(kind="none", iteration=0):
    """Test-only fault hook of Bi-CGSTAB (the GPU's GSK_FAULT mirrors it):
    "rho0" / "omega0" force rho = 0 at the end of / omega = 0 in the given iteration,
    "nan" writes NaN into r_0 in its update.  set_fault() clears it."""
    _lib().orc_set_fault(FAULTS[kind], int(iteration))


def bicgstab(row_ptr, col, val, b, tol, maxit, x0=None, weights=None):
    """Returns (x, hist, report-dict)."""
    row_ptr, col, val, b = _i32(row_ptr), _i32(col), _f64(val), _f64(b)
    x0, w = _f64(x0), _f64(weights)
    n = row_ptr.size - 1
    x = np.empty(n, np.float64)
    hist = np.empty(maxit + 1, np.float64)
    rep = Report()
    rc = _lib().orc_bicgstab(n, _p(row_ptr), _p(col), _p(val), _p(b), _p(x0), _p(w),
                             float(tol), int(maxit), _p(x), _p(hist), ctypes.byref(rep))
    if rc != 0:
        raise ValueError("bad arguments")
    return x, hist[:rep.history_len].copy(), rep.as_dict()


def gmres(row_ptr, col, val, b, m, tol, maxit, x0=None, weights=None, orth="mgs", wstop=False):
    """Returns (x, hist, report-dict).  orth: "mgs" (north star) or "cgs2" (AZTEC's
    double classical Gram-Schmidt).  wstop: stop on the weighted true
    residual at cycle ends instead of the least-squares estimate (reading B2w)."""
    row_ptr, col, val, b = _i32(row_ptr), _i32(col), _f64(val), _f64(b)
    x0, w = _f64(x0), _f64(weights)
    n = row_ptr.size - 1
    x = np.empty(n, np.float64)
    hist = np.empty(maxit + 1, np.float64)
    rep = Report()
    rc = _lib().orc_gmres_wstop(n, _p(row_ptr), _p(col), _p(val), _p(b), _p(x0), _p(w), int(m),
                                float(tol), int(maxit), {"mgs": 0, "cgs2": 1}[orth], int(bool(wstop)),
                                _p(x), _p(hist), ctypes.byref(rep))
    if rc != 0:
        raise ValueError("bad arguments")
    return x, hist[:rep.history_len].copy(), rep.as_dict()
