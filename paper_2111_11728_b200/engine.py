"""Python mirror of the reference's solver entry points over the C-ABI.

``FetiSystem`` wraps one ``fetigpu_ctx`` (include/fetigpu.h) and exposes the
reference's operator / plugin interface for this path with the same names
and argument meaning: ``apply_F`` (DualOperator::apply),
``apply_precond`` (apply_coarse_preconditioner), ``project``
(CoarseSpace::project / project_block, decomposition.hpp:136-138), ``rhs``
(d and lambda0), ``solve`` (pcg / simultaneous_pcg,
SPEC.md:426-443) and ``recover`` (recover_primal).  Errors are
raised as the reference's exception types (proj/include/feti/errors.hpp).

There is no CPU fallback: constructing a system without the CUDA library or
without a GPU raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

from .problems import Problem

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FETIGPU_LIB") or os.path.join(_HERE, "lib", "libfetigpu.so")
_lib = None

D = C.POINTER(C.c_double)
I = C.POINTER(C.c_int)


# ---- errors (proj/include/feti/errors.hpp:7-69) ---------------------------
class FetiError(RuntimeError):
    code = -1


def _mk(name, code):
    return type(name, (FetiError,), {"code": code})


NotPositiveDefinite = _mk("NotPositiveDefinite", 1)
IndefiniteInput = _mk("IndefiniteInput", 2)
IncompatibleRhs = _mk("IncompatibleRhs", 3)
EdgeNotOnBoundary = _mk("EdgeNotOnBoundary", 4)
DimensionMismatch = _mk("DimensionMismatch", 5)
NodeNotFound = _mk("NodeNotFound", 6)
InsufficientCorners = _mk("InsufficientCorners", 7)
ZeroStiffnessDiagonal = _mk("ZeroStiffnessDiagonal", 8)
SingularInterior = _mk("SingularInterior", 9)
CoarseSingular = _mk("CoarseSingular", 10)
SingularRemainder = _mk("SingularRemainder", 11)
SingularCoarse = _mk("SingularCoarse", 12)
SingularGlobal = _mk("SingularGlobal", 13)
NegativeInnerProduct = _mk("NegativeInnerProduct", 14)
NotConverged = _mk("NotConverged", 15)
StateSolveFailed = _mk("StateSolveFailed", 16)
ConfigError = _mk("ConfigError", 17)
IoError = _mk("IoError", 18)
InvalidArgument = _mk("InvalidArgument", 20)
DomainError = _mk("DomainError", 21)
CudaError = _mk("CudaError", 100)
NoDevice = _mk("NoDevice", 101)
OutOfMemory = _mk("OutOfMemory", 102)
StateError = _mk("StateError", 103)
_ERRORS = {c.code: c for c in (NotPositiveDefinite, IndefiniteInput, IncompatibleRhs,
                               EdgeNotOnBoundary, DimensionMismatch, NodeNotFound,
                               InsufficientCorners, ZeroStiffnessDiagonal, SingularInterior,
                               CoarseSingular, SingularRemainder, SingularCoarse, SingularGlobal,
                               NegativeInnerProduct, NotConverged, StateSolveFailed, ConfigError,
                               IoError, InvalidArgument, DomainError, CudaError, NoDevice,
                               OutOfMemory, StateError)}

EXPORTED = ["fetigpu_set_device", "fetigpu_create", "fetigpu_build", "fetigpu_destroy", "fetigpu_last_error",
            "fetigpu_stats_get", "fetigpu_rows", "fetigpu_apply_F", "fetigpu_apply_F_device",
            "fetigpu_apply_precond", "fetigpu_apply_precond_device", "fetigpu_project",
            "fetigpu_project_device", "fetigpu_rhs", "fetigpu_solve", "fetigpu_recover",
            "fetigpu_local_operator", "fetigpu_device_alloc", "fetigpu_device_free",
            "fetigpu_host_alloc", "fetigpu_host_free", "fetigpu_memcpy", "fetigpu_fill_random",
            "fetigpu_synchronize", "fetigpu_time_apply", "fetigpu_apply_F_block_device",
            "fetigpu_time_apply_block", "fetigpu_fp64_peak", "fetigpu_hbm_read_peak", "fetigpu_selftest_dmma",
            "fetigpu_pivoted_cholesky", "fetigpu_pivoted_compress", "fetigpu_time_ops",
            "fetigpu_device_memory", "fetigpu_set_rrs_store", "fetigpu_dla_gemm", "fetigpu_dla_tri_inv",
            "fetigpu_dla_time_gemm", "fetigpu_apply_F_zblock", "fetigpu_set_check", "fetigpu_check_result",
            "fetigpu_shard_set_range", "fetigpu_shard_info", "fetigpu_shard_phase1_device",
            "fetigpu_shard_phase2_device", "fetigpu_solve_warm", "fetigpu_rebuild"]


class FgProblem(C.Structure):
    _fields_ = [("sx", C.c_int), ("sy", C.c_int), ("n", C.c_int),
                ("hx", C.c_double), ("hy", C.c_double),
                ("E0", C.c_double), ("Emin", C.c_double), ("nu", C.c_double),
                ("p", C.c_double), ("thickness", C.c_double),
                ("n_designs", C.c_int), ("densities", D), ("module_type", I),
                ("n_dirichlet", C.c_int), ("dir_gnode", I), ("dir_dir", I), ("dir_value", D),
                ("n_tractions", C.c_int), ("tr_sub", I), ("tr_side", I), ("tr_first", I),
                ("tr_count", I), ("tr_txy", D),
                ("n_point_loads", C.c_int), ("pl_gnode", I), ("pl_dir", I), ("pl_value", D),
                ("method", C.c_int), ("scaling", C.c_int), ("precond", C.c_int)]


class FgOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("rel", C.c_int), ("max_it", C.c_int),
                ("directions", C.c_int), ("pivot_tol", C.c_double), ("reorth_passes", C.c_int)]


class FgTrace(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("f_applies", C.c_int),
                ("eps0", C.c_double), ("eps_final", C.c_double), ("cap", C.c_int),
                ("eps", D), ("kept", I), ("f_app", I), ("solve_ms", C.c_double),
                ("phase_ms", C.c_double * 8)]


class FgStats(C.Structure):
    _fields_ = [(k, C.c_int) for k in ("m", "n_sub", "local_dofs", "n_c", "n_kept", "n_iface",
                                       "max_ns", "n_designs", "n_op_slots", "n_pc_slots")] + \
               [(k, C.c_double) for k in ("op_bytes", "op_flops_per_col", "main_kernel_bytes",
                                          "build_ms", "nd_ms", "slot_ms", "coarse_ms",
                                          "device_bytes")] + \
               [("host_pipeline", C.c_int), ("solve_loop", C.c_int), ("stream_bytes", C.c_double),
                ("apply_kernel", C.c_int), ("apply_ring", C.c_int)]


def lib():
    """Load libfetigpu.so; raises if the CUDA extension was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run __graft_entry__.build() (no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        L.fetigpu_last_error.restype = C.c_char_p
        L.fetigpu_destroy.restype = None
        L.fetigpu_create.argtypes = [C.POINTER(FgProblem), C.POINTER(C.c_void_p)]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    if a.dtype == np.int32:
        return a.ctypes.data_as(I)
    return a.ctypes.data_as(D)


def check(rc: int):
    if rc != 0:
        msg = lib().fetigpu_last_error().decode()
        raise _ERRORS.get(rc, FetiError)(f"[{rc}] {msg}")


def fp64_peak():
    """(DMMA, DFMA) FP64 TFLOP/s measured on the current device."""
    a, b = C.c_double(), C.c_double()
    check(lib().fetigpu_fp64_peak(C.byref(a), C.byref(b)))
    return a.value, b.value


def hbm_read_peak(nbytes: int = 2 << 30, reps: int = 10) -> float:
    """Read-only HBM stream bandwidth (GB/s) measured on the current device."""
    g = C.c_double()
    check(lib().fetigpu_hbm_read_peak(C.c_size_t(nbytes), reps, C.byref(g)))
    return g.value


def device_memory(system=None) -> dict:
    """Free / total device bytes, and the bytes `system` (a FetiSystem, or
    None) holds in its cache of freed RRS direction-store chunks
    (fetigpu_device_memory)."""
    f, t, c = C.c_size_t(), C.c_size_t(), C.c_size_t()
    check(lib().fetigpu_device_memory(system.h if system is not None else None, C.byref(f), C.byref(t),
                                      C.byref(c)))
    return {"free": f.value, "total": t.value, "cached": c.value}


def pivoted_cholesky(a: np.ndarray, tol: float = 1e-12):
    """Device rank-revealing pivoted Cholesky (feti::pivoted_cholesky,
    linalg.hpp:80).  Returns (perm, L[:, :rank], rank) with
    A[perm][:, perm] = L L^T on the kept block, like oracle.pyoracle's helper."""
    a = np.asarray(a, dtype=np.float64)
    n = a.shape[0]
    A = np.asfortranarray(a)
    perm = np.zeros(max(n, 1), dtype=np.int32)
    low = np.zeros(max(n * n, 1))
    rank = C.c_int()
    check(lib().fetigpu_pivoted_cholesky(A.ctypes.data_as(D), n, C.c_double(tol), _p(perm), _p(low),
                                         C.byref(rank)))
    L = low[:n * n].reshape(n, n).T[:, :rank.value].copy()
    return perm[:n], L, rank.value


def compress(perm, lower, rank: int, w: np.ndarray) -> np.ndarray:
    """Device W N^T [L~^{-T}; 0] (PivotedCholesky::compress, linalg.hpp:79);
    `lower` is the n x rank block from pivoted_cholesky."""
    n = len(perm)
    low = np.zeros((n, n))
    low[:, :rank] = lower
    lowf = np.ascontiguousarray(low.T).reshape(-1)      # column-major n x n
    pv = np.ascontiguousarray(perm, dtype=np.int32)
    W = np.asfortranarray(w, dtype=np.float64)
    out = np.zeros((w.shape[0], max(rank, 1)), order="F")
    check(lib().fetigpu_pivoted_compress(_p(pv), _p(lowf), n, rank, W.ctypes.data_as(D), w.shape[0],
                                         out.ctypes.data_as(D)))
    return np.ascontiguousarray(out[:, :rank])


def dla_gemm(A: np.ndarray, B: np.ndarray, ta: bool = False, tb: bool = False, alpha: float = 1.0,
             beta: float = 0.0, C0: np.ndarray = None, flags: int = 0) -> np.ndarray:
    """alpha op(A) op(B) + beta C0 through the engine's DMMA GEMM (dla.cuh),
    column-major like BLAS dgemm."""
    A = np.asfortranarray(A, dtype=np.float64)
    B = np.asfortranarray(B, dtype=np.float64)
    M = A.shape[1] if ta else A.shape[0]
    K = A.shape[0] if ta else A.shape[1]
    N = B.shape[0] if tb else B.shape[1]
    Cm = np.asfortranarray(np.zeros((M, N)) if C0 is None else C0, dtype=np.float64).copy(order="F")
    check(lib().fetigpu_dla_gemm(int(ta), int(tb), M, N, K, C.c_double(alpha), A.ctypes.data_as(D),
                                 C.c_longlong(max(1, A.shape[0])), B.ctypes.data_as(D),
                                 C.c_longlong(max(1, B.shape[0])), C.c_double(beta), Cm.ctypes.data_as(D),
                                 C.c_longlong(max(1, M)), flags))
    return Cm


def dla_tri_inv(L: np.ndarray) -> np.ndarray:
    """L^{-1} of the lower triangle of L through the engine's kernels."""
    Lf = np.asfortranarray(L, dtype=np.float64)
    n = Lf.shape[0]
    X = np.zeros((n, n), order="F")
    check(lib().fetigpu_dla_tri_inv(Lf.ctypes.data_as(D), n, C.c_longlong(n), X.ctypes.data_as(D)))
    return X


def dla_time_gemm(M: int, N: int, K: int, ta: bool = False, tb: bool = False, reps: int = 5) -> float:
    ms = C.c_double()
    check(lib().fetigpu_dla_time_gemm(int(ta), int(tb), M, N, K, reps, C.byref(ms)))
    return ms.value


def dmma_selftest(A: np.ndarray, B: np.ndarray) -> np.ndarray:
    A = np.ascontiguousarray(A, dtype=np.float64)
    B = np.ascontiguousarray(B, dtype=np.float64)
    Cm = np.zeros((8, 8))
    check(lib().fetigpu_selftest_dmma(_p(A), _p(B), _p(Cm)))
    return Cm


def make_struct(prob: Problem, keep: list) -> FgProblem:
    a = prob.arrays()
    keep.append(a)
    s = FgProblem()
    s.sx, s.sy, s.n = prob.sx, prob.sy, prob.n
    s.hx, s.hy = prob.hx, prob.hy
    s.E0, s.Emin, s.nu, s.p, s.thickness = prob.E0, prob.Emin, prob.nu, prob.p, prob.thickness
    s.n_designs = int(prob.densities.shape[0])
    s.densities, s.module_type = _p(a["densities"]), _p(a["module_type"])
    s.n_dirichlet = len(prob.dirichlet)
    s.dir_gnode, s.dir_dir, s.dir_value = _p(a["dir_gnode"]), _p(a["dir_dir"]), _p(a["dir_value"])
    s.n_tractions = len(prob.tractions)
    s.tr_sub, s.tr_side, s.tr_first, s.tr_count, s.tr_txy = (
        _p(a["tr_sub"]), _p(a["tr_side"]), _p(a["tr_first"]), _p(a["tr_count"]), _p(a["tr_txy"]))
    s.n_point_loads = len(prob.point_loads)
    s.pl_gnode, s.pl_dir, s.pl_value = _p(a["pl_gnode"]), _p(a["pl_dir"]), _p(a["pl_value"])
    s.method, s.scaling, s.precond = prob.method, prob.scaling, prob.precond
    return s


class FetiSystem:
    """A T-FETI or FETI-DP dual system resident on the GPU (TfetiSystem /
    FetidpSystem of SPEC.md:346-353)."""

    def __init__(self, prob: Problem, build: bool = True):
        self.prob = prob
        self._keep = []
        st = make_struct(prob, self._keep)
        h = C.c_void_p()
        check(lib().fetigpu_create(C.byref(st), C.byref(h)))
        self.h = h
        s = self.stats()
        self.m, self.n_sub, self.local_dofs = s["m"], s["n_sub"], s["local_dofs"]
        self.n_c = s["n_c"]
        self.built = False
        if build:
            self.build()

    def build(self):
        """Device build (K1-K3, K6); host setup already ran in fetigpu_create."""
        check(lib().fetigpu_build(self.h))
        self.built = True

    def close(self):
        if getattr(self, "h", None):
            lib().fetigpu_destroy(self.h)
            self.h = None

    __del__ = close

    def stats(self) -> dict:
        s = FgStats()
        check(lib().fetigpu_stats_get(self.h, C.byref(s)))
        return {k: getattr(s, k) for k, _ in FgStats._fields_}

    def rows(self) -> dict:
        m = self.m
        out = {k: np.zeros(m, dtype=np.int32) for k in ("kind", "sub_plus", "dof_plus",
                                                         "sub_minus", "dof_minus", "mult")}
        gap, wp, wm = np.zeros(m), np.zeros(m), np.zeros(m)
        check(lib().fetigpu_rows(self.h, _p(out["kind"]), _p(out["sub_plus"]), _p(out["dof_plus"]),
                                 _p(out["sub_minus"]), _p(out["dof_minus"]), _p(gap),
                                 _p(out["mult"]), _p(wp), _p(wm)))
        out.update(gap=gap, w_plus=wp, w_minus=wm)
        return out

    def apply_F(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x, dtype=np.float64)
        cols = 1 if x.ndim == 1 else x.shape[1]
        X = np.ascontiguousarray(x.reshape(self.m, cols).T)
        Y = np.zeros_like(X)
        check(lib().fetigpu_apply_F(self.h, _p(X), _p(Y), C.c_int(cols), C.c_int(self.m)))
        return Y.T.reshape(x.shape).copy()

    def apply_precond(self, r: np.ndarray, columns: bool = False):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.m)
        Z = np.zeros((self.n_sub, self.m)) if columns else None
        check(lib().fetigpu_apply_precond(self.h, _p(r), _p(z), _p(Z) if columns else None))
        return (z, Z.T.copy()) if columns else z

    def project(self, v: np.ndarray) -> np.ndarray:
        v = np.asarray(v, dtype=np.float64)
        cols = 1 if v.ndim == 1 else v.shape[1]
        V = np.ascontiguousarray(v.reshape(self.m, cols).T)
        check(lib().fetigpu_project(self.h, _p(V), C.c_int(cols), C.c_int(self.m)))
        return V.T.reshape(v.shape).copy()

    def rhs(self):
        d, l0 = np.zeros(self.m), np.zeros(self.m)
        check(lib().fetigpu_rhs(self.h, _p(d), _p(l0)))
        return d, l0

    def solve(self, tol: float = 1e-6, max_it: int = 1000, directions: int = 0, rel: bool = True,
              pivot_tol: float = 1e-12, reorth_passes: int = 2):
        o = FgOpts(tol, 1 if rel else 0, max_it, directions, pivot_tol, reorth_passes)
        cap = max_it + 2
        eps, kept, fap = np.zeros(cap), np.zeros(cap, dtype=np.int32), np.zeros(cap, dtype=np.int32)
        tr = FgTrace(0, 0, 0, 0.0, 0.0, cap, _p(eps), _p(kept), _p(fap), 0.0)
        tr.phase_ms = (C.c_double * 8)(*([0.0] * 8))
        lam = np.zeros(self.m)
        check(lib().fetigpu_solve(self.h, C.byref(o), _p(lam), C.byref(tr)))
        n = tr.iterations + 1
        return lam, dict(status=tr.status, iterations=tr.iterations, f_applies=tr.f_applies,
                         eps0=tr.eps0, eps_final=tr.eps_final, eps=eps[:n].copy(),
                         kept=kept[:n].copy(), f_app=fap[:n].copy(), solve_ms=tr.solve_ms,
                         phase_ms=list(tr.phase_ms))

    def solve_warm(self, lam0, tol: float = 1e-6, max_it: int = 1000, directions: int = 0, rel: bool = True,
                   pivot_tol: float = 1e-12, reorth_passes: int = 2):
        """solve() started from lam0 (fetigpu_solve_warm)."""
        o = FgOpts(tol, 1 if rel else 0, max_it, directions, pivot_tol, reorth_passes)
        cap = max_it + 2
        eps, kept, fap = np.zeros(cap), np.zeros(cap, dtype=np.int32), np.zeros(cap, dtype=np.int32)
        tr = FgTrace(0, 0, 0, 0.0, 0.0, cap, _p(eps), _p(kept), _p(fap), 0.0)
        tr.phase_ms = (C.c_double * 8)(*([0.0] * 8))
        lam = np.zeros(self.m)
        l0 = np.ascontiguousarray(lam0, dtype=np.float64)
        check(lib().fetigpu_solve_warm(self.h, C.byref(o), _p(l0), _p(lam), C.byref(tr)))
        n = tr.iterations + 1
        return lam, dict(status=tr.status, iterations=tr.iterations, f_applies=tr.f_applies,
                         eps0=tr.eps0, eps_final=tr.eps_final, eps=eps[:n].copy(),
                         kept=kept[:n].copy(), f_app=fap[:n].copy(), solve_ms=tr.solve_ms,
                         phase_ms=list(tr.phase_ms))

    def rebuild(self, prob: Problem):
        """Next snapshot of the same problem in place (fetigpu_rebuild)."""
        self._keep = []
        st = make_struct(prob, self._keep)
        check(lib().fetigpu_rebuild(self.h, C.byref(st)))
        self.prob = prob

    RRS_STORE = {"auto": 0, "explicit": 1, "implicit": 2}

    def set_rrs_store(self, mode: str = "auto"):
        """Direction store of RRS solves (fetigpu_set_rrs_store): "explicit"
        (W_j, F W_j dense, Alg. 1 as written), "implicit" (FETI-DP: W_j as
        coefficients over the packed preconditioner blocks) or "auto"."""
        check(lib().fetigpu_set_rrs_store(self.h, self.RRS_STORE[mode]))

    def recover(self, lam: np.ndarray) -> np.ndarray:
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        u = np.zeros((self.n_sub, self.local_dofs))
        check(lib().fetigpu_recover(self.h, _p(lam), _p(u)))
        return u

    def apply_F_block(self, W: np.ndarray) -> np.ndarray:
        """K5 block apply Q = F W on the device (W: m x k, row-major blocks)."""
        W = np.ascontiguousarray(W, dtype=np.float64)
        m, k = W.shape
        L = lib()
        nbytes = C.c_size_t(W.nbytes)
        dW, dQ = C.c_void_p(), C.c_void_p()
        check(L.fetigpu_device_alloc(self.h, nbytes, C.byref(dW)))
        check(L.fetigpu_device_alloc(self.h, nbytes, C.byref(dQ)))
        try:
            Q = np.empty_like(W)
            check(L.fetigpu_memcpy(self.h, dW, W.ctypes.data_as(C.c_void_p), nbytes, 1))
            check(L.fetigpu_apply_F_block_device(self.h, C.cast(dW, D), C.c_int(k), C.cast(dQ, D),
                                                 C.c_int(k), C.c_int(k)))
            check(L.fetigpu_memcpy(self.h, Q.ctypes.data_as(C.c_void_p), dQ, nbytes, 2))
            check(L.fetigpu_synchronize(self.h))
        finally:
            L.fetigpu_device_free(self.h, dW)
            L.fetigpu_device_free(self.h, dQ)
        return Q

    def set_check(self, on: bool = True):
        """Invariant check of later FO / RRS solves (fetigpu_set_check)."""
        check(lib().fetigpu_set_check(self.h, int(on)))

    def check_result(self):
        """(max |W^T F W - I| over the last solve's stored directions, their number)"""
        e, n = C.c_double(), C.c_int()
        check(lib().fetigpu_check_result(self.h, C.byref(e), C.byref(n)))
        return e.value, n.value

    def apply_F_zblock(self, Z: np.ndarray) -> np.ndarray:
        """Q = F Z through the sparse-aware K5z path (Z: m x N_s per-subdomain
        preconditioner columns, as apply_precond(columns=True) returns)."""
        Z = np.ascontiguousarray(Z, dtype=np.float64)
        Q = np.empty_like(Z)
        check(lib().fetigpu_apply_F_zblock(self.h, Z.ctypes.data_as(D), Q.ctypes.data_as(D)))
        return Q

    def time_ops(self, reps: int = 200) -> dict:
        """Device time per call of F, the preconditioner and the projector (ms)."""
        ms = (C.c_double * 3)()
        check(lib().fetigpu_time_ops(self.h, reps, ms))
        return {"F_ms": ms[0], "precond_ms": ms[1], "project_ms": ms[2]}

    def local_operator(self, s: int):
        cap = 8 * self.prob.n
        ns = C.c_int()
        dofs = np.zeros(cap, dtype=np.int32)
        F = np.zeros(cap * cap)
        check(lib().fetigpu_local_operator(self.h, s, C.byref(ns), _p(dofs), _p(F), cap))
        n = ns.value
        return dofs[:n].copy(), F[:n * n].reshape(n, n).copy()
