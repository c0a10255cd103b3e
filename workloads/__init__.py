"""Seeded synthetic workloads (shared INPUT module; none of the method's arithmetic).

Both the oracle (``oracle/``) and the CUDA path (``paper_0812_2769_b200``) are fed
from here.  The systems follow the paper's discretisation (§2.1)
and BASELINE.json's five configs; the readings are listed in DESIGN.md §3.

``generate(name)`` returns a dict of numpy arrays: ``row_ptr`` (int32, n+1),
``col`` (int32, nnz), ``val`` (float64, nnz), ``xstar`` and ``b`` (float64, n) and
``perm`` (int32, n; C5's symmetric permutation, identity otherwise).
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libgskgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)}` "
                               "(or __graft_entry__.build())")
        lib = ctypes.CDLL(path)
        i64p = ctypes.POINTER(ctypes.c_int64)
        lib.gen_dims.argtypes = [ctypes.c_int, ctypes.c_int, i64p, i64p]
        lib.gen_dims.restype = ctypes.c_int
        lib.gen_fill.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                 ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.gen_fill.restype = ctypes.c_int
        lib.gen_uniform.argtypes = [ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int64,
                                    ctypes.c_double, ctypes.c_double, ctypes.c_void_p]
        lib.gen_uniform.restype = None
        lib.gen_dims_stacked.argtypes = [ctypes.c_int, ctypes.c_int, i64p, i64p]
        lib.gen_dims_stacked.restype = ctypes.c_int
        lib.gen_fill_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_double,
                                      ctypes.c_int64, ctypes.c_int64] + [ctypes.c_void_p] * 5
        lib.gen_fill_rows.restype = ctypes.c_int
        _LIB = lib
    return _LIB


@dataclass(frozen=True)
class Config:
    """A BASELINE.json config (or a paper-pin workload) and its solve recipe."""
    name: str
    cfg: int            # generator id
    N: int              # interior points per axis
    seed: int
    tol: float
    maxit: int
    m: int              # the config's own GMRES restart
    scalings: tuple = ("none", 2)
    tols: tuple = ()
    param: float = 0.0
    sell: bool = False  # config lists a SELL-C-sigma copy (C4)
    extra_m: tuple = field(default=(30,))


# BASELINE.json "configs" [0..4]  (seeds = config number, M15)
CONFIGS = {
    "C1": Config("C1", 1, 32, 1, 1e-8, 2000, 20, ("none", 2), (1e-8,)),
    "C2": Config("C2", 2, 512, 2, 1e-10, 10000, 30, ("none", 1, 2), (1e-6, 1e-8, 1e-10)),
    "C3": Config("C3", 3, 128, 3, 1e-8, 10000, 30, ("none", 2), (1e-8,)),
    "C4": Config("C4", 4, 256, 4, 1e-8, 10000, 30, ("none", 2), (1e-8,), sell=True),
    "C5": Config("C5", 5, 2048, 5, 1e-8, 10000, 50, ("none", 1, 2), (1e-8,)),
}

# paper-pin workloads (tests only): PAPER.md:328-347 (P1), :878-895 (P4)
PAPER = {
    "P1": Config("P1", 11, 128, 0, 1e-10, 10000, 10, param=1e3),
    "P1cont": Config("P1cont", 12, 128, 0, 1e-10, 10000, 10, param=1e3),
    "P4": Config("P4", 14, 80, 0, 1e-10, 10000, 10, param=1e4),
    "P4conv": Config("P4conv", 15, 40, 0, 1e-10, 10000, 10, param=100.0),
}


# Weak-scaling variant of C4: G copies of C4's layered medium stacked
# in z, 256 x 256 x 256G nodes, G = param (one 256^3 block per GPU); G = 1 is C4.
STACKED = Config("C4w", 24, 256, 4, 1e-8, 10000, 30, ("none", 2), (1e-8,), param=1.0, sell=True)


def dims(cfg: int, N: int, param: float = 0.0):
    n = ctypes.c_int64()
    nnz = ctypes.c_int64()
    rc = (_lib().gen_dims_stacked(N, int(param) if param >= 1 else 1, ctypes.byref(n), ctypes.byref(nnz))
          if cfg == 24 else _lib().gen_dims(cfg, N, ctypes.byref(n), ctypes.byref(nnz)))
    if rc != 0:
        raise ValueError(f"unknown generator cfg {cfg} / N {N}")
    return n.value, nnz.value


def generate_raw(cfg: int, N: int, seed: int = 0, param: float = 0.0) -> dict:
    n, nnz = dims(cfg, N, param)
    out = {
        "row_ptr": np.empty(n + 1, np.int32), "col": np.empty(nnz, np.int32),
        "val": np.empty(nnz, np.float64), "xstar": np.empty(n, np.float64),
        "b": np.empty(n, np.float64), "perm": np.empty(n, np.int32),
    }
    rc = _lib().gen_fill(cfg, N, seed, param, *(out[k].ctypes.data for k in
                                                 ("row_ptr", "col", "val", "xstar", "b", "perm")))
    if rc != 0:
        raise ValueError(f"gen_fill failed for cfg {cfg}")
    out["n"] = n
    out["nnz"] = nnz
    return out


def generate(name: str, N: int | None = None, seed: int | None = None, param: float | None = None) -> dict:
    """Generate config ``name`` (C1..C5, P1, P1cont, P4, lap2d, lap3d); ``N``
    overrides the grid size (reduced-size parity cases)."""
    if name in CONFIGS or name in PAPER:
        c = CONFIGS.get(name) or PAPER[name]
        return generate_raw(c.cfg, N or c.N, c.seed if seed is None else seed,
                            c.param if param is None else param)
    if name == "C4w":
        c = STACKED
        return generate_raw(c.cfg, N or c.N, c.seed if seed is None else seed, c.param if param is None else param)
    if name == "lap2d":
        return generate_raw(20, N or 16, 0)
    if name == "lap3d":
        return generate_raw(21, N or 8, 0)
    raise KeyError(name)


def generate_rows(name: str, lo: int, hi: int, N: int | None = None, param: float | None = None) -> dict:
    """Rows [lo, hi) of config ``name`` (global column indices; row_ptr starts at 0), with
    x* and b = A x* on those rows — one rank's block of a row-block sharded solve,
    without generating the rest (not for C5, whose permutation is global).  Row for
    row identical to ``generate``.  ``n`` is the global row count."""
    c = STACKED if name == "C4w" else CONFIGS[name]
    N = N or c.N
    param = c.param if param is None else param
    n, _ = dims(c.cfg, N, param)
    # exact nnz of the block from the row lengths' closed form is config-specific;
    # bound it by 7 (3D) / 5 (2D) entries per row and trim
    cap = (7 if c.cfg in (3, 4, 24) else 5) * (hi - lo)
    out = {"row_ptr": np.empty(hi - lo + 1, np.int32), "col": np.empty(cap, np.int32),
           "val": np.empty(cap, np.float64), "xstar": np.empty(hi - lo, np.float64),
           "b": np.empty(hi - lo, np.float64)}
    rc = _lib().gen_fill_rows(c.cfg, N, c.seed, param, lo, hi,
                              *(out[k].ctypes.data for k in ("row_ptr", "col", "val", "xstar", "b")))
    if rc != 0:
        raise ValueError(f"gen_fill_rows failed for {name} rows [{lo}, {hi})")
    nnz = int(out["row_ptr"][-1])
    out["col"], out["val"] = out["col"][:nnz].copy(), out["val"][:nnz].copy()
    out.update(n=n, nnz=nnz, lo=lo, hi=hi)
    return out


def uniform(n: int, seed: int, stream: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Counter-based U[lo,hi) vector (same SplitMix64 as the generator)."""
    out = np.empty(n, np.float64)
    _lib().gen_uniform(seed, stream, n, lo, hi, out.ctypes.data)
    return out
