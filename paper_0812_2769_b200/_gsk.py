"""ctypes binding of libgsk.so (include/gsk.h): argument marshalling only.

Every step of the path runs in the library's sm_100a kernels; PyTorch provides
device memory and the current stream.  There is no CPU fallback: if the in-tree
``libgsk.so`` is missing or CUDA is unavailable, every call raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GSK_LIB") or os.path.join(_HERE, "libgsk.so")  # GSK_LIB: A/B builds

GSK_OK, GSK_E_INVALID, GSK_E_ZERO_ROW, GSK_E_CUDA, GSK_E_NOMEM = 0, -1, -2, -3, -4
STATUS = {0: "CONVERGED", 1: "MAXIT", 2: "BREAKDOWN", 3: "DIVERGED"}
FMT = {"csr": 0, "sell": 1}
SCHEDULE = {"auto": 0, "fused": 1, "split": 2, "split4": 3}
ENGINE = {"auto": 0, "graph": 1, "coop": 2, "small": 3, "cluster": 4}
ORTH = {"mgs": 0, "cgs2": 1}

# exported symbols (include/gsk.h); tests check the library exports all of them
SYMBOLS = ("gsk_gs_scale", "gsk_gs_scale_sym", "gsk_gs_unscale", "gsk_spmv", "gsk_dot", "gsk_plan_create", "gsk_plan_refresh",
           "gsk_plan_spmv", "gsk_plan_sell_info", "gsk_plan_sell_copy", "gsk_plan_sell_dict", "gsk_plan_sell_uniform", "gsk_plan_row_classes", "gsk_plan_class_slots", "gsk_plan_destroy",
           "gsk_bicgstab_solve", "gsk_bicgstab_solve_plan", "gsk_gmres_solve",
           "gsk_gmres_solve_plan", "gsk_plan_residual_norm", "gsk_plan_probe",
           "gsk_shard_rows", "gsk_shard_halo_host", "gsk_plan_create_sharded", "gsk_nccl_unique_id",
           "gsk_nccl_comm_create", "gsk_nccl_comm_destroy",
           "gsk_last_error", "gsk_launch_count", "gsk_version")


class CsrStruct(ctypes.Structure):
    _fields_ = [("n", ctypes.c_int32), ("nnz", ctypes.c_int32), ("row_ptr", ctypes.c_void_p),
                ("col_idx", ctypes.c_void_p), ("values", ctypes.c_void_p)]


class Report(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("iterations", ctypes.c_int32),
                ("restarts", ctypes.c_int32), ("history_len", ctypes.c_int32),
                ("breakdown_at", ctypes.c_int32), ("pad_", ctypes.c_int32),
                ("relres", ctypes.c_double), ("true_relres", ctypes.c_double),
                ("true_relres_w", ctypes.c_double), ("best_relres", ctypes.c_double),
                ("solve_ms", ctypes.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}


class Opts(ctypes.Structure):
    _fields_ = [("format", ctypes.c_int32), ("poll", ctypes.c_int32), ("weights", ctypes.c_void_p),
                ("bicg_schedule", ctypes.c_int32), ("gmres_orth", ctypes.c_int32),
                ("sell_index", ctypes.c_int32), ("engine", ctypes.c_int32),
                ("gmres_wstop", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class ShardOpts(ctypes.Structure):
    _fields_ = [("nshards", ctypes.c_int32), ("first", ctypes.c_int32), ("count", ctypes.c_int32),
                ("local_input", ctypes.c_int32), ("nccl_comm", ctypes.c_void_p),
                ("peer_reduce", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class GskError(RuntimeError):
    def __init__(self, code, msg, bad_row=None):
        super().__init__(f"gsk error {code}: {msg}")
        self.code = code
        self.bad_row = bad_row


_LIB = None


def load(path: str = LIB_PATH):
    """Load libgsk.so (raises if it is missing: no fallback path exists)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(path):
        raise RuntimeError(f"{path} is missing: build it with `make` or __graft_entry__.build()")
    lib = ctypes.CDLL(path)
    vp, i32, i64, d = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    P = ctypes.POINTER
    lib.gsk_gs_scale.argtypes = [P(CsrStruct), vp, i32, vp, vp, vp, P(ctypes.c_int32), vp]
    lib.gsk_gs_scale_sym.argtypes = [P(CsrStruct), vp, i32, vp, vp, vp, P(ctypes.c_int32), vp]
    lib.gsk_gs_unscale.argtypes = [i64, vp, vp, vp, vp]
    lib.gsk_spmv.argtypes = [P(CsrStruct), vp, vp, vp]
    lib.gsk_dot.argtypes = [i64, vp, vp, P(d), vp]
    lib.gsk_plan_create.argtypes = [P(CsrStruct), P(Opts), P(vp), vp]
    lib.gsk_plan_refresh.argtypes = [vp, vp]
    lib.gsk_plan_spmv.argtypes = [vp, vp, vp, vp]
    lib.gsk_plan_sell_info.argtypes = [vp, P(i64), P(i64)]
    lib.gsk_plan_sell_copy.argtypes = [vp, vp, vp, vp, vp, vp, vp]
    lib.gsk_plan_sell_dict.argtypes = [vp, P(i64), vp, vp, vp, vp]
    lib.gsk_plan_sell_uniform.argtypes = [vp, P(i64), vp, vp, vp, vp, vp]
    lib.gsk_plan_row_classes.argtypes = [vp, P(i64), vp, vp, vp]
    lib.gsk_plan_class_slots.argtypes = [vp, P(ctypes.c_int32), vp, vp, vp]
    lib.gsk_plan_destroy.argtypes = [vp]
    lib.gsk_plan_destroy.restype = None
    lib.gsk_bicgstab_solve.argtypes = [P(CsrStruct), vp, vp, d, i32, vp, vp, P(Report), vp]
    lib.gsk_bicgstab_solve_plan.argtypes = [vp, vp, vp, d, i32, vp, vp, P(Report), vp]
    lib.gsk_gmres_solve.argtypes = [P(CsrStruct), vp, vp, i32, d, i32, vp, vp, P(Report), vp]
    lib.gsk_gmres_solve_plan.argtypes = [vp, vp, vp, i32, d, i32, vp, vp, P(Report), vp]
    lib.gsk_plan_residual_norm.argtypes = [vp, vp, vp, vp, P(d), vp]
    lib.gsk_plan_probe.argtypes = [vp, i32, P(d), P(i64)]
    lib.gsk_shard_rows.argtypes = [i64, i32, i32, P(i64), P(i64)]
    lib.gsk_shard_halo_host.argtypes = [i64, vp, vp, i32, i32, P(ctypes.c_int32), P(ctypes.c_int32)]
    lib.gsk_plan_create_sharded.argtypes = [P(CsrStruct), P(Opts), P(ShardOpts), P(vp), vp]
    lib.gsk_nccl_unique_id.argtypes = [ctypes.c_char_p]
    lib.gsk_nccl_comm_create.argtypes = [ctypes.c_char_p, i32, i32, P(vp)]
    lib.gsk_nccl_comm_destroy.argtypes = [vp]
    lib.gsk_last_error.restype = ctypes.c_char_p
    lib.gsk_launch_count.restype = i64
    for name in SYMBOLS:
        if name not in ("gsk_last_error", "gsk_launch_count", "gsk_plan_destroy"):
            getattr(lib, name).restype = ctypes.c_int
    _LIB = lib
    return lib


def _check(rc, bad_row=None):
    if rc != GSK_OK:
        msg = load().gsk_last_error().decode(errors="replace")
        raise GskError(rc, msg, bad_row)


def _stream():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _dev_f64(t, n=None):
    if t is None:
        return None
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.ascontiguousarray(t, dtype=np.float64))
    t = t.to(device="cuda", dtype=torch.float64).contiguous()
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} entries, got {t.numel()}")
    return t


def _out_f64(t, n, name, avoid=()):
    """A caller-supplied OUTPUT buffer: the kernels write n doubles through its raw
    pointer, so it must be a contiguous CUDA float64 tensor of exactly n entries and
    must not overlap an input."""
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda" or t.dtype != torch.float64:
        raise TypeError(f"{name}: expected a CUDA float64 tensor")
    if not t.is_contiguous() or t.numel() != n:
        raise ValueError(f"{name}: expected a contiguous tensor of {n} entries, got shape {tuple(t.shape)}")
    a0, a1 = t.data_ptr(), t.data_ptr() + 8 * n
    for u in avoid:
        if u is not None and u.numel() and a0 < u.data_ptr() + u.numel() * u.element_size() and u.data_ptr() < a1:
            raise ValueError(f"{name} overlaps an input of the same call")
    return t


def _dev_i32(t):
    if not isinstance(t, torch.Tensor):
        t = torch.as_tensor(np.ascontiguousarray(t, dtype=np.int32))
    return t.to(device="cuda", dtype=torch.int32).contiguous()


class CSR:
    """A CSR matrix resident on the GPU (int32 indices, fp64 values)."""

    def __init__(self, row_ptr, col, val):
        if not torch.cuda.is_available():
            raise RuntimeError("CUDA device required (no CPU fallback)")
        self.row_ptr = _dev_i32(row_ptr)
        self.col = _dev_i32(col)
        self.val = _dev_f64(val)
        self.n = self.row_ptr.numel() - 1
        self.nnz = self.col.numel()
        if self.val.numel() != self.nnz:
            raise ValueError("col / val size mismatch")

    @classmethod
    def from_system(cls, s: dict):
        return cls(s["row_ptr"], s["col"], s["val"])

    def struct(self, values=None) -> CsrStruct:
        v = self.val if values is None else values
        return CsrStruct(self.n, self.nnz, self.row_ptr.data_ptr(), self.col.data_ptr(), v.data_ptr())


def gs_scale(A: CSR, b=None, p: int = 2, inplace: bool = False, out=None):
    """GS(p) (Eq. (2)): returns (A', b', d) with A' = D A, b' = D b.
    ``out=(values, b, d)`` writes into preallocated device tensors."""
    lib = load()
    b = _dev_f64(b, A.n)
    if out is not None:
        vout, bout, d = out
        _out_f64(vout, A.val.numel(), "out[0] (values)")
        if bout is not None:
            _out_f64(bout, A.n, "out[1] (b)")
        _out_f64(d, A.n, "out[2] (d)")
    else:
        vout = A.val if inplace else torch.empty_like(A.val)
        bout = None if b is None else (b if inplace else torch.empty_like(b))
        d = torch.empty(A.n, dtype=torch.float64, device="cuda")
    bad = ctypes.c_int32(-1)
    rc = lib.gsk_gs_scale(ctypes.byref(A.struct()), _ptr(b), int(p), _ptr(vout), _ptr(bout), _ptr(d),
                          ctypes.byref(bad), _stream())
    _check(rc, bad.value if rc == GSK_E_ZERO_ROW else None)
    As = A if (inplace and out is None) else CSR.__new__(CSR)
    if As is not A:
        As.row_ptr, As.col, As.val, As.n, As.nnz = A.row_ptr, A.col, vout, A.n, A.nnz
    return As, bout, d


def gs_scale_sym(A: CSR, b=None, p: int = 2):
    """Two-sided scaling: returns (A', b', s) with
    A' = D^1/2 A D^1/2, b' = D^1/2 b and s = diag(D^1/2); solve A' y = b', then
    x = gs_unscale(s, y)."""
    lib = load()
    b = _dev_f64(b, A.n)
    vout = torch.empty_like(A.val)
    bout = None if b is None else torch.empty_like(b)
    sv = torch.empty(A.n, dtype=torch.float64, device="cuda")
    bad = ctypes.c_int32(-1)
    rc = lib.gsk_gs_scale_sym(ctypes.byref(A.struct()), _ptr(b), int(p), _ptr(vout), _ptr(bout), _ptr(sv),
                              ctypes.byref(bad), _stream())
    _check(rc, bad.value if rc == GSK_E_ZERO_ROW else None)
    As = CSR.__new__(CSR)
    As.row_ptr, As.col, As.val, As.n, As.nnz = A.row_ptr, A.col, vout, A.n, A.nnz
    return As, bout, sv


def gs_unscale(s, y):
    s, y = _dev_f64(s), _dev_f64(y)
    x = torch.empty_like(y)
    _check(load().gsk_gs_unscale(y.numel(), _ptr(s), _ptr(y), _ptr(x), _stream()))
    return x


def spmv(A: CSR, x):
    x = _dev_f64(x, A.n)
    y = torch.empty_like(x)
    _check(load().gsk_spmv(ctypes.byref(A.struct()), _ptr(x), _ptr(y), _stream()))
    return y


def dot(a, b) -> float:
    a, b = _dev_f64(a), _dev_f64(b)
    out = ctypes.c_double()
    _check(load().gsk_dot(a.numel(), _ptr(a), _ptr(b), ctypes.byref(out), _stream()))
    return out.value


def launch_count() -> int:
    return int(load().gsk_launch_count())


SELL_INDEX = {"plain": 0, "dict": 1, "uniform": 2, "classes": 3}


class Plan:
    """gsk_plan: SELL build, workspace and captured graphs reused across solves."""

    def __init__(self, A: CSR, fmt: str = "csr", weights=None, poll: int = 0, schedule: str = "auto",
                 orth: str = "mgs", sell_index: str = "plain", engine: str = "auto", gmres_wstop: bool = False):
        """engine: "auto" (one launch per solve on one CTA up to 2048 / 1024 rows or on
        one thread-block cluster up to 32768 / 65536 rows for Bi-CGSTAB / GMRES, or a
        persistent cooperative grid up to 81920 rows for Bi-CGSTAB, where measured
        faster; else graph passes), "graph" (always the passes), "coop" (persistent
        cooperative multi-CTA Bi-CGSTAB whenever its grid fits), "small" (one CTA, n <= 4096) or "cluster"
        (one cluster, n <= 65536)."""
        lib = load()
        self.A = A
        self.weights = _dev_f64(weights, A.n)
        opts = Opts(FMT[fmt], int(poll), None if self.weights is None else self.weights.data_ptr(),
                    SCHEDULE[schedule], ORTH[orth], SELL_INDEX[sell_index], ENGINE[engine],
                    int(bool(gmres_wstop)), 0)
        self._csr = A.struct()
        h = ctypes.c_void_p()
        _check(lib.gsk_plan_create(ctypes.byref(self._csr), ctypes.byref(opts), ctypes.byref(h), _stream()))
        self.h = h
        self.fmt = fmt
        self.nloc = A.n

    def close(self):
        if getattr(self, "h", None):
            load().gsk_plan_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def refresh(self):
        _check(load().gsk_plan_refresh(self.h, _stream()))

    def spmv(self, x, y=None):
        x = _dev_f64(x, self.nloc)
        y = torch.empty_like(x) if y is None else _out_f64(y, self.nloc, "y", avoid=(x,))
        _check(load().gsk_plan_spmv(self.h, _ptr(x), _ptr(y), _stream()))
        return y

    def residual_norm(self, b, x, w=None) -> float:
        out = ctypes.c_double()
        b, x, w = _dev_f64(b, self.A.n), _dev_f64(x, self.A.n), _dev_f64(w, self.A.n)
        _check(load().gsk_plan_residual_norm(self.h, _ptr(b), _ptr(x), _ptr(w), ctypes.byref(out), _stream()))
        return out.value

    def sell_arrays(self):
        lib = load()
        nch, nsl = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.gsk_plan_sell_info(self.h, ctypes.byref(nch), ctypes.byref(nsl)))
        dev = "cuda"
        out = {"chunk_ptr": torch.empty(nch.value + 1, dtype=torch.int32, device=dev),
               "chunk_len": torch.empty(nch.value, dtype=torch.int32, device=dev),
               "scol": torch.empty(max(nsl.value, 1), dtype=torch.int32, device=dev),
               "sval": torch.empty(max(nsl.value, 1), dtype=torch.float64, device=dev),
               "roff": torch.empty(nch.value * 32, dtype=torch.uint8, device=dev)}
        _check(lib.gsk_plan_sell_copy(self.h, *(_ptr(out[k]) for k in
                                                ("chunk_ptr", "chunk_len", "scol", "sval", "roff")), _stream()))
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["scol"] = res["scol"][:nsl.value]
        res["sval"] = res["sval"][:nsl.value]
        return res

    def sell_dict(self):
        """The plan's SELL column dictionary (None when it uses plain int32 columns)."""
        lib = load()
        nd = ctypes.c_int64()
        _check(lib.gsk_plan_sell_dict(self.h, ctypes.byref(nd), None, None, None, _stream()))
        if nd.value < 0:
            return None
        nch, nsl = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.gsk_plan_sell_info(self.h, ctypes.byref(nch), ctypes.byref(nsl)))
        out = {"dict_ptr": torch.empty(nch.value + 1, dtype=torch.int32, device="cuda"),
               "dict": torch.empty(max(nd.value, 1), dtype=torch.int32, device="cuda"),
               "sidx": torch.empty(max(nsl.value, 1), dtype=torch.uint8, device="cuda")}
        _check(lib.gsk_plan_sell_dict(self.h, ctypes.byref(nd), _ptr(out["dict_ptr"]), _ptr(out["dict"]),
                                      _ptr(out["sidx"]), _stream()))
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["dict"] = res["dict"][:nd.value]
        res["sidx"] = res["sidx"][:nsl.value]
        return res

    def row_classes(self):
        """The plan's row-class dictionary (sell_index="classes"; None when inapplicable):
        {"cls" uint16 [n], "len" [K], "delta" [K, 8], "val" [K, 8]}."""
        lib = load()
        k = ctypes.c_int64()
        _check(lib.gsk_plan_row_classes(self.h, ctypes.byref(k), None, None, _stream()))
        if k.value < 0:
            return None
        cls = torch.empty(self.A.n, dtype=torch.int16, device="cuda")
        ent = torch.empty(max(k.value, 1) * 128, dtype=torch.uint8, device="cuda")
        _check(lib.gsk_plan_row_classes(self.h, ctypes.byref(k), _ptr(cls), _ptr(ent), _stream()))
        rec = ent.cpu().numpy()[:k.value * 128].view(
            np.dtype([("v", "<f8", 8), ("len", "<i4"), ("d", "<i4", 8), ("pad", "<i4", 7)]))
        assert not rec["pad"].any()
        return {"cls": cls.cpu().numpy().view(np.uint16), "len": rec["len"].copy(),
                "delta": rec["d"].copy(), "val": rec["v"].copy()}

    def class_slots(self):
        """Stencil slots of the plan's classes (None when they do not share one symmetric
        5- / 7-delta set): {"deltas" [ns], "mask" uint32 [K], "val" [K, 8]}."""
        lib = load()
        ns = ctypes.c_int32()
        dl = (ctypes.c_int32 * 8)()
        _check(lib.gsk_plan_class_slots(self.h, ctypes.byref(ns), dl, None, _stream()))
        if ns.value < 0:
            return None
        k = self.num_classes()
        buf = torch.empty(k * 128, dtype=torch.uint8, device="cuda")
        _check(lib.gsk_plan_class_slots(self.h, ctypes.byref(ns), dl, _ptr(buf), _stream()))
        rec = buf.cpu().numpy().view(np.dtype([("v", "<f8", 8), ("mask", "<u4"), ("pad", "<u4", 15)]))
        assert not rec["pad"].any()
        return {"deltas": np.array(dl[:ns.value]), "mask": rec["mask"].copy(), "val": rec["v"].copy()}

    def num_slots(self) -> int:
        """Deltas of the classes' shared stencil (5 or 7), or -1 (no stencil slots)."""
        ns = ctypes.c_int32()
        _check(load().gsk_plan_class_slots(self.h, ctypes.byref(ns), None, None, _stream()))
        return ns.value

    def num_classes(self) -> int:
        """Classes of the plan's row-class dictionary (-1: not built or inapplicable)."""
        k = ctypes.c_int64()
        _check(load().gsk_plan_row_classes(self.h, ctypes.byref(k), None, None, _stream()))
        return k.value

    def sell_uniform(self):
        """The plan's SELL-U arrays (chunk-uniform column deltas; None when not built)."""
        lib = load()
        nu = ctypes.c_int64()
        _check(lib.gsk_plan_sell_uniform(self.h, ctypes.byref(nu), None, None, None, None, _stream()))
        if nu.value < 0:
            return None
        nch, nsl = ctypes.c_int64(), ctypes.c_int64()
        _check(lib.gsk_plan_sell_info(self.h, ctypes.byref(nch), ctypes.byref(nsl)))
        out = {"uptr": torch.empty(nch.value + 1, dtype=torch.int32, device="cuda"),
               "udel": torch.empty(nch.value * 8, dtype=torch.int32, device="cuda"),
               "umask": torch.empty(nch.value * 8, dtype=torch.int32, device="cuda"),
               "uval": torch.empty(max(nu.value, 1), dtype=torch.float64, device="cuda")}
        _check(lib.gsk_plan_sell_uniform(self.h, ctypes.byref(nu), *(_ptr(out[k]) for k in
                                                                    ("uptr", "udel", "umask", "uval")), _stream()))
        res = {k: v.cpu().numpy() for k, v in out.items()}
        res["umask"] = res["umask"].view(np.uint32)
        res["uval"] = res["uval"][:nu.value]
        return res

    def probe(self, kind: int):
        ms, cnt = ctypes.c_double(), ctypes.c_int64()
        _check(load().gsk_plan_probe(self.h, kind, ctypes.byref(ms), ctypes.byref(cnt)))
        return ms.value, cnt.value

    def _solve(self, which, b, x0, tol, maxit, m=None, x=None, hist=True):
        lib = load()
        b = _dev_f64(b, self.nloc)
        x0 = _dev_f64(x0, self.nloc)
        x = torch.empty(self.nloc, dtype=torch.float64, device="cuda") if x is None else \
            _out_f64(x, self.nloc, "x", avoid=(b,))
        H = np.empty(maxit + 1, np.float64) if hist else None
        rep = Report()
        hp = None if H is None else H.ctypes.data_as(ctypes.c_void_p)
        if which == "bicgstab":
            rc = lib.gsk_bicgstab_solve_plan(self.h, _ptr(b), _ptr(x0), float(tol), int(maxit), _ptr(x),
                                             hp, ctypes.byref(rep), _stream())
        else:
            rc = lib.gsk_gmres_solve_plan(self.h, _ptr(b), _ptr(x0), int(m), float(tol), int(maxit), _ptr(x),
                                          hp, ctypes.byref(rep), _stream())
        _check(rc)
        r = rep.as_dict()
        return x, (None if H is None else H[:rep.history_len].copy()), r

    def bicgstab(self, b, x0=None, tol=1e-8, maxit=10000, x=None, hist=True):
        """Bi-CGSTAB on the plan's system; returns (x, hist, report)."""
        return self._solve("bicgstab", b, x0, tol, maxit, x=x, hist=hist)

    def gmres(self, b, x0=None, m=30, tol=1e-8, maxit=10000, x=None, hist=True):
        """Restarted GMRES(m) on the plan's system; returns (x, hist, report).  GMRES stops
        on its least-squares estimate in the SOLVED frame; the plan's frame weights only
        enter report["true_relres_w"] (gsk.h, reading B2)."""
        return self._solve("gmres", b, x0, tol, maxit, m=m, x=x, hist=hist)


def shard_rows(n: int, nshards: int, r: int):
    """Rows [lo, hi) of shard r of n rows in nshards row blocks (host only)."""
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(load().gsk_shard_rows(int(n), int(nshards), int(r), ctypes.byref(lo), ctypes.byref(hi)))
    return lo.value, hi.value


def shard_halo(row_ptr, col, nshards: int, r: int):
    """Halo widths (left, right) of shard r from a host CSR with global columns."""
    rp = np.ascontiguousarray(row_ptr, np.int32)
    ci = np.ascontiguousarray(col, np.int32)
    hl, hr = ctypes.c_int32(), ctypes.c_int32()
    _check(load().gsk_shard_halo_host(rp.size - 1, rp.ctypes.data_as(ctypes.c_void_p),
                                      ci.ctypes.data_as(ctypes.c_void_p), int(nshards), int(r),
                                      ctypes.byref(hl), ctypes.byref(hr)))
    return hl.value, hr.value


class NcclComm:
    """NCCL communicator over the ranks of a torch.distributed process group (one GPU
    per rank); rank 0's unique id is broadcast through the group."""

    def __init__(self, group=None):
        import torch.distributed as dist
        lib = load()
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)
        buf = ctypes.create_string_buffer(128)
        if self.rank == 0:
            _check(lib.gsk_nccl_unique_id(buf))
        obj = [bytes(buf.raw) if self.rank == 0 else None]
        dist.broadcast_object_list(obj, src=0, group=group)
        h = ctypes.c_void_p()
        _check(lib.gsk_nccl_comm_create(ctypes.c_char_p(obj[0]), self.world, self.rank, ctypes.byref(h)))
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            load().gsk_nccl_comm_destroy(self.h)
            self.h = None


class ShardedPlan(Plan):
    """Row-block sharded plan: `shards` row blocks of the GLOBAL matrix A.
    On one GPU (comm=None) this process holds all shards; with an NcclComm each rank
    holds shard `comm.rank` of `comm.world`.  Solves take and return this process's
    rows; the history is global.  Bit-identical to the unsharded solvers.

    ``n_global`` (with a comm only): A holds just this rank's rows [lo, hi) with global
    column indices (gsk_shard_opts.local_input), so no rank holds the whole system.
    ``peer_reduce``: the reductions' shard values travel by device-initiated peer
    stores + epoch flags instead of ncclAllGather (gsk_shard_opts.peer_reduce)."""

    def __init__(self, A: CSR, shards: int = 2, fmt: str = "csr", weights=None, poll: int = 0,
                 comm: "NcclComm" = None, n_global: int = None, sell_index: str = "plain",
                 peer_reduce: bool = False, gmres_wstop: bool = False):
        lib = load()
        self.A = A
        if comm is None:
            if n_global is not None:
                raise ValueError("n_global (local input) needs an NcclComm: one shard per rank")
            first, count, ch = 0, int(shards), None
        else:
            shards, first, count, ch = comm.world, comm.rank, 1, comm.h
        ng = A.n if n_global is None else int(n_global)
        lo, _ = shard_rows(ng, shards, first)
        _, hi = shard_rows(ng, shards, first + count - 1)
        if n_global is not None and hi - lo != A.n:
            raise ValueError(f"local input: A has {A.n} rows, shard {first} of {ng} rows owns {hi - lo}")
        self.rows = (lo, hi)
        self.nloc = hi - lo
        self.weights = _dev_f64(weights, self.nloc)
        opts = Opts(FMT[fmt], int(poll), None if self.weights is None else self.weights.data_ptr(),
                    SCHEDULE["split"], ORTH["mgs"], SELL_INDEX[sell_index],
                    ENGINE["graph"], int(bool(gmres_wstop)), 0)
        so = ShardOpts(int(shards), int(first), int(count), int(n_global is not None), ch, int(peer_reduce), 0)
        self._csr = A.struct()
        self._csr.n = ng
        h = ctypes.c_void_p()
        _check(lib.gsk_plan_create_sharded(ctypes.byref(self._csr), ctypes.byref(opts), ctypes.byref(so),
                                           ctypes.byref(h), _stream()))
        self.h = h
        self.fmt = fmt
        self.shards = shards


def bicgstab_solve(A: CSR, b, x0=None, tol=1e-8, maxit=10000):
    """bicgstab_solve(csr, b, x0, tol, maxit) of the north star (plan-less, CSR)."""
    lib = load()
    b, x0 = _dev_f64(b, A.n), _dev_f64(x0, A.n)
    x = torch.empty(A.n, dtype=torch.float64, device="cuda")
    H = np.empty(maxit + 1, np.float64)
    rep = Report()
    _check(lib.gsk_bicgstab_solve(ctypes.byref(A.struct()), _ptr(b), _ptr(x0), float(tol), int(maxit),
                                  _ptr(x), H.ctypes.data_as(ctypes.c_void_p), ctypes.byref(rep), _stream()))
    return x, H[:rep.history_len].copy(), rep.as_dict()


def gmres_solve(A: CSR, b, x0=None, m=30, tol=1e-8, maxit=10000):
    """gmres_solve(csr, b, x0, m, tol, maxit) of the north star (plan-less, CSR)."""
    lib = load()
    b, x0 = _dev_f64(b, A.n), _dev_f64(x0, A.n)
    x = torch.empty(A.n, dtype=torch.float64, device="cuda")
    H = np.empty(maxit + 1, np.float64)
    rep = Report()
    _check(lib.gsk_gmres_solve(ctypes.byref(A.struct()), _ptr(b), _ptr(x0), int(m), float(tol), int(maxit),
                               _ptr(x), H.ctypes.data_as(ctypes.c_void_p), ctypes.byref(rep), _stream()))
    return x, H[:rep.history_len].copy(), rep.as_dict()
