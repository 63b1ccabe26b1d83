"""ctypes binding of the CPU oracle (oracle/_build/libfeti_oracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / ``--impl reference`` legs, never by the product.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libfeti_oracle.so")
_lib = None

D = C.POINTER(C.c_double)
I = C.POINTER(C.c_int)


class FoProblem(C.Structure):
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


class FoOpts(C.Structure):
    _fields_ = [("tol", C.c_double), ("rel", C.c_int), ("max_it", C.c_int),
                ("directions", C.c_int), ("pivot_tol", C.c_double), ("reorth_passes", C.c_int)]


class FoTrace(C.Structure):
    _fields_ = [("status", C.c_int), ("iterations", C.c_int), ("f_applies", C.c_int),
                ("eps0", C.c_double), ("eps_final", C.c_double), ("cap", C.c_int),
                ("eps", D), ("kept", I), ("f_app", I)]


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.fo_last_error.restype = C.c_char_p
        L.fo_admissibility_error.restype = C.c_double
        L.fo_coarse_residual.restype = C.c_double
        L.fo_create.argtypes = [C.POINTER(FoProblem), C.POINTER(C.c_void_p)]
        L.fo_destroy.argtypes = [C.c_void_p]
        _lib = L
    return _lib


def _p(a):
    if a is None:
        return None
    if a.dtype == np.int32:
        return a.ctypes.data_as(I)
    return a.ctypes.data_as(D)


def _check(rc: int):
    if rc != 0:
        raise OracleError(rc, lib().fo_last_error().decode())


def make_struct(prob, keep: list) -> FoProblem:
    a = prob.arrays()
    keep.append(a)
    s = FoProblem()
    s.sx, s.sy, s.n = prob.sx, prob.sy, prob.n
    s.hx, s.hy = prob.hx, prob.hy
    s.E0, s.Emin, s.nu, s.p, s.thickness = prob.E0, prob.Emin, prob.nu, prob.p, prob.thickness
    s.n_designs = int(prob.densities.shape[0])
    s.densities = _p(a["densities"])
    s.module_type = _p(a["module_type"])
    s.n_dirichlet = len(prob.dirichlet)
    s.dir_gnode, s.dir_dir, s.dir_value = _p(a["dir_gnode"]), _p(a["dir_dir"]), _p(a["dir_value"])
    s.n_tractions = len(prob.tractions)
    s.tr_sub, s.tr_side, s.tr_first, s.tr_count, s.tr_txy = (
        _p(a["tr_sub"]), _p(a["tr_side"]), _p(a["tr_first"]), _p(a["tr_count"]), _p(a["tr_txy"]))
    s.n_point_loads = len(prob.point_loads)
    s.pl_gnode, s.pl_dir, s.pl_value = _p(a["pl_gnode"]), _p(a["pl_dir"]), _p(a["pl_value"])
    s.method, s.scaling, s.precond = prob.method, prob.scaling, prob.precond
    return s


class Oracle:
    """CPU restatement of the reference dual operators and engine."""

    def __init__(self, prob):
        self.prob = prob
        self._keep = []
        st = make_struct(prob, self._keep)
        h = C.c_void_p()
        _check(lib().fo_create(C.byref(st), C.byref(h)))
        self.h = h
        info = np.zeros(8, dtype=np.int32)
        lib().fo_info(self.h, _p(info))
        self.m, self.n_sub, self.local_dofs, self.n_c, self.n_kept, self.n_iface, self.max_ns = (
            int(x) for x in info[:7])

    def __del__(self):
        if getattr(self, "h", None):
            lib().fo_destroy(self.h)
            self.h = None

    def rows(self) -> dict:
        m = self.m
        out = {k: np.zeros(m, dtype=np.int32) for k in ("kind", "sub_plus", "dof_plus",
                                                         "sub_minus", "dof_minus", "mult")}
        gap, wp, wm = np.zeros(m), np.zeros(m), np.zeros(m)
        lib().fo_rows(self.h, _p(out["kind"]), _p(out["sub_plus"]), _p(out["dof_plus"]),
                      _p(out["sub_minus"]), _p(out["dof_minus"]), _p(gap), _p(out["mult"]),
                      _p(wp), _p(wm))
        out.update(gap=gap, w_plus=wp, w_minus=wm)
        return out

    def apply_F(self, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.m)
        _check(lib().fo_apply_F(self.h, _p(x), _p(y)))
        return y

    def apply_precond(self, r: np.ndarray, columns: bool = False):
        r = np.ascontiguousarray(r, dtype=np.float64)
        z = np.zeros(self.m)
        Z = np.zeros((self.n_sub, self.m)) if columns else None
        _check(lib().fo_apply_precond(self.h, _p(r), _p(z), _p(Z) if columns else None))
        return (z, Z.T.copy()) if columns else z

    def project(self, v: np.ndarray) -> np.ndarray:
        v = np.array(v, dtype=np.float64, copy=True)
        _check(lib().fo_project(self.h, _p(v)))
        return v

    def rhs(self):
        d, l0 = np.zeros(self.m), np.zeros(self.m)
        _check(lib().fo_rhs(self.h, _p(d), _p(l0)))
        return d, l0

    def solve(self, tol: float = 1e-6, max_it: int = 1000, directions: int = 0, rel: bool = True,
              pivot_tol: float = 1e-12, reorth_passes: int = 2):
        o = FoOpts(tol, 1 if rel else 0, max_it, directions, pivot_tol, reorth_passes)
        cap = max_it + 2
        eps, kept, fap = np.zeros(cap), np.zeros(cap, dtype=np.int32), np.zeros(cap, dtype=np.int32)
        tr = FoTrace(0, 0, 0, 0.0, 0.0, cap, _p(eps), _p(kept), _p(fap))
        lam = np.zeros(self.m)
        _check(lib().fo_solve(self.h, C.byref(o), _p(lam), C.byref(tr)))
        n = tr.iterations + 1
        return lam, dict(status=tr.status, iterations=tr.iterations, f_applies=tr.f_applies,
                         eps0=tr.eps0, eps_final=tr.eps_final, eps=eps[:n].copy(),
                         kept=kept[:n].copy(), f_app=fap[:n].copy())

    def recover(self, lam: np.ndarray) -> np.ndarray:
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        u = np.zeros((self.n_sub, self.local_dofs))
        _check(lib().fo_recover(self.h, _p(lam), _p(u)))
        return u

    def local_diag(self) -> np.ndarray:
        d = np.zeros((self.n_sub, self.local_dofs))
        lib().fo_local_diag(self.h, _p(d))
        return d

    def loads(self) -> np.ndarray:
        f = np.zeros((self.n_sub, self.local_dofs))
        lib().fo_load_vectors(self.h, _p(f))
        return f

    def admissibility_error(self) -> float:
        return float(lib().fo_admissibility_error(self.h))

    def local_apply(self, s: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.zeros(self.local_dofs)
        _check(lib().fo_local_apply(self.h, s, _p(x), _p(y)))
        return y

    def coarse_residual(self, lam: np.ndarray) -> float:
        lam = np.ascontiguousarray(lam, dtype=np.float64)
        return float(lib().fo_coarse_residual(self.h, _p(lam)))

    def pseudo_solve(self, s: int, rhs: np.ndarray) -> np.ndarray:
        rhs = np.ascontiguousarray(rhs, dtype=np.float64)
        x = np.zeros(self.local_dofs)
        _check(lib().fo_pseudo_solve(self.h, s, _p(rhs), _p(x)))
        return x

    def fixed_dofs(self):
        out = np.zeros(3, dtype=np.int32)
        _check(lib().fo_fixed_dofs(self.h, _p(out)))
        return out.tolist()

    def direct(self) -> np.ndarray:
        u = np.zeros((self.n_sub, self.local_dofs))
        _check(lib().fo_direct_solve(self.h, _p(u)))
        return u


def set_check(on: bool = True):
    lib().fo_set_check(int(on))


def check_result():
    e, n = C.c_double(), C.c_int()
    lib().fo_check_result(C.byref(e), C.byref(n))
    return e.value, n.value


# ---- kernel-level helpers (SPEC examples) ---------------------------------
def simp_modulus(rho, E0=1.0, Emin=1e-9, p=3.0) -> float:
    out = C.c_double()
    _check(lib().fo_simp_modulus(C.c_double(rho), C.c_double(E0), C.c_double(Emin),
                                 C.c_double(p), C.byref(out)))
    return out.value


def q4_element_stiffness(nu=0.3, thickness=1.0, modulus=1.0, hx=1.0, hy=1.0) -> np.ndarray:
    k = np.zeros(64)
    _check(lib().fo_q4_element_stiffness(C.c_double(nu), C.c_double(thickness),
                                         C.c_double(modulus), C.c_double(hx), C.c_double(hy),
                                         _p(k)))
    return k.reshape(8, 8).T.copy()


def pivoted_cholesky(a: np.ndarray, tol: float = 1e-12):
    n = a.shape[0]
    A = np.asfortranarray(a, dtype=np.float64)
    perm = np.zeros(n, dtype=np.int32)
    low = np.zeros(n * n)
    rank = C.c_int()
    _check(lib().fo_pivoted_cholesky(n, A.ctypes.data_as(D), C.c_double(tol), _p(perm), _p(low),
                                     C.byref(rank)))
    L = low.reshape(n, n).T[:, :rank.value].copy()
    return perm, L, rank.value


def compress(perm, lower, rank, w: np.ndarray) -> np.ndarray:
    n = len(perm)
    low = np.zeros((n, n))
    low[:, :rank] = lower
    lowf = np.ascontiguousarray(low.T).reshape(-1)
    W = np.asfortranarray(w, dtype=np.float64)
    out = np.zeros(w.shape[0] * rank)
    _check(lib().fo_compress(n, _p(np.asarray(perm, dtype=np.int32)), _p(lowf), rank,
                             w.shape[0], W.ctypes.data_as(D), _p(out)))
    return out.reshape(rank, w.shape[0]).T.copy()


def select_fixing_dofs(basis: np.ndarray):
    B = np.asfortranarray(basis, dtype=np.float64)
    out = np.zeros(basis.shape[1], dtype=np.int32)
    _check(lib().fo_select_fixing_dofs(basis.shape[0], basis.shape[1], B.ctypes.data_as(D),
                                       _p(out)))
    return out.tolist()


def rigid_body_modes(n: int, hx=1.0, hy=1.0) -> np.ndarray:
    R = np.zeros(2 * (n + 1) ** 2 * 3)
    lib().fo_rigid_body_modes(n, C.c_double(hx), C.c_double(hy), _p(R))
    return R.reshape(3, -1).T.copy()


def cholesky_solve(a: np.ndarray, b: np.ndarray) -> np.ndarray:
    A = np.asfortranarray(a, dtype=np.float64)
    x = np.array(b, dtype=np.float64, copy=True)
    _check(lib().fo_band_cholesky_solve(a.shape[0], A.ctypes.data_as(D), _p(x)))
    return x
