"""Seeded synthetic problem generators for the five BASELINE.json configs.

The reference defines no input files for this path (its MBB snapshots and
module layouts are absent), so BASELINE.json's configs are
realised here as seeded synthetic density fields with the shapes, contrasts,
supports and loads each config names.  Everything is
deterministic: a portable SplitMix64 stream (never numpy's generators) drives
uniform / Bernoulli / Box-Muller normal draws.

A :class:`Problem` mirrors the reference's build inputs
(``build_partition`` + ``assemble_subdomain`` + ``apply_traction`` +
``build_constraints``; proj/include/feti/decomposition.hpp:47-117,
proj/include/feti/fem.hpp:78-99) and is consumed by both the GPU library
(``fetigpu_problem``) and the CPU oracle (``fo_problem``).
"""
from __future__ import annotations

import dataclasses
from typing import List, Optional

import numpy as np

TFETI, FETIDP = 0, 1
MULTIPLICITY, KSCALING = 0, 1
LUMPED, DIRICHLET, SUPERLUMPED = 0, 1, 2
SINGLE, FO, RRS = 0, 1, 2
LEFT, RIGHT, BOTTOM, TOP = 0, 1, 2, 3  # fem.hpp:88 Side order

_GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed: int, count: int) -> np.ndarray:
    """``count`` SplitMix64 outputs of the stream started at ``seed``."""
    with np.errstate(over="ignore"):
        idx = np.arange(1, count + 1, dtype=np.uint64)
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + idx * _GOLDEN
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, count: int) -> np.ndarray:
    """U[0,1) = (x >> 11) * 2^-53."""
    return (splitmix64(seed, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def normal(seed: int, count: int) -> np.ndarray:
    """Box-Muller N(0,1) from consecutive uniform pairs."""
    u = uniform(seed, 2 * ((count + 1) // 2)).reshape(-1, 2)
    r = np.sqrt(-2.0 * np.log1p(-u[:, 0]))
    t = 2.0 * np.pi * u[:, 1]
    return np.stack([r * np.cos(t), r * np.sin(t)], axis=1).reshape(-1)[:count]


def gaussian_random_field(seed: int, ny: int, nx: int, length: float) -> np.ndarray:
    """White N(0,1) noise convolved with a Gaussian of sigma = l/sqrt(2)
    (squared-exponential covariance with length scale l), truncated at 4 sigma,
    reflecting boundaries."""
    from scipy.ndimage import gaussian_filter

    white = normal(seed, ny * nx).reshape(ny, nx)
    return gaussian_filter(white, sigma=length / np.sqrt(2.0), mode="reflect", truncate=4.0)


def ramp(solid: np.ndarray, width: float = 2.0) -> np.ndarray:
    """2-element linear ramp across the 0/1 interface: rho = clamp(1/2 + d/2)
    with d the signed Euclidean distance (element units) to the interface."""
    from scipy.ndimage import distance_transform_edt

    if solid.all() or not solid.any():
        return solid.astype(np.float64)
    d_in = distance_transform_edt(solid) - 0.5
    d_out = distance_transform_edt(~solid) - 0.5
    d = np.where(solid, d_in, -d_out)
    return np.clip(0.5 + d / width, 0.0, 1.0)


@dataclasses.dataclass
class Problem:
    sx: int
    sy: int
    n: int
    densities: np.ndarray           # (n_designs, n, n), row-major from the bottom row
    module_type: np.ndarray         # (sx*sy,) design id per subdomain (sj*sx + si)
    method: int = TFETI
    scaling: int = MULTIPLICITY
    precond: int = LUMPED
    directions: int = SINGLE
    E0: float = 1.0
    Emin: float = 1e-9
    nu: float = 0.3
    p: float = 3.0
    thickness: float = 1.0
    hx: float = 1.0
    hy: float = 1.0
    dirichlet: List[tuple] = dataclasses.field(default_factory=list)   # (gnode, dir, value)
    tractions: List[tuple] = dataclasses.field(default_factory=list)   # (sub, side, first, count, tx, ty)
    point_loads: List[tuple] = dataclasses.field(default_factory=list) # (gnode, dir, value)
    tol: float = 1e-6
    max_it: int = 1000
    name: str = ""

    @property
    def n_sub(self) -> int:
        return self.sx * self.sy

    @property
    def gx_nodes(self) -> int:
        return self.sx * self.n + 1

    @property
    def gy_nodes(self) -> int:
        return self.sy * self.n + 1

    @property
    def local_dofs(self) -> int:
        return 2 * (self.n + 1) ** 2

    def gnode(self, gx: int, gy: int) -> int:
        return gy * self.gx_nodes + gx

    def replace(self, **kw) -> "Problem":
        return dataclasses.replace(self, **kw)

    # ---- flat arrays for the C structs ------------------------------------
    def arrays(self) -> dict:
        d = np.ascontiguousarray(self.densities, dtype=np.float64).reshape(-1)
        mt = np.ascontiguousarray(self.module_type, dtype=np.int32)
        dg = np.array([t[0] for t in self.dirichlet], dtype=np.int32)
        dd = np.array([t[1] for t in self.dirichlet], dtype=np.int32)
        dv = np.array([t[2] for t in self.dirichlet], dtype=np.float64)
        ts = np.array([t[0] for t in self.tractions], dtype=np.int32)
        tside = np.array([t[1] for t in self.tractions], dtype=np.int32)
        tf = np.array([t[2] for t in self.tractions], dtype=np.int32)
        tc = np.array([t[3] for t in self.tractions], dtype=np.int32)
        txy = np.array([[t[4], t[5]] for t in self.tractions], dtype=np.float64).reshape(-1)
        pg = np.array([t[0] for t in self.point_loads], dtype=np.int32)
        pd = np.array([t[1] for t in self.point_loads], dtype=np.int32)
        pv = np.array([t[2] for t in self.point_loads], dtype=np.float64)
        return dict(densities=d, module_type=mt, dir_gnode=dg, dir_dir=dd, dir_value=dv,
                    tr_sub=ts, tr_side=tside, tr_first=tf, tr_count=tc, tr_txy=txy,
                    pl_gnode=pg, pl_dir=pd, pl_value=pv)


# ---- supports and loads (SURVEY.md 8d "Common inputs") ---------------------
def left_clamp(sx: int, sy: int, n: int) -> List[tuple]:
    gxn = sx * n + 1
    return [(gy * gxn, d, 0.0) for gy in range(sy * n + 1) for d in (0, 1)]


def bottom_corner_pins(sx: int, sy: int, n: int) -> List[tuple]:
    return [(0, 0, 0.0), (0, 1, 0.0), (sx * n, 0, 0.0), (sx * n, 1, 0.0)]


def right_edge_traction(sx: int, sy: int, n: int, ty: float = -1.0) -> List[tuple]:
    return [(sj * sx + (sx - 1), RIGHT, 0, n, 0.0, ty) for sj in range(sy)]


def split_global(field: np.ndarray, sx: int, sy: int, n: int) -> np.ndarray:
    """(sy*n, sx*n) global element field -> (sx*sy, n, n) per-module blocks."""
    out = np.empty((sx * sy, n, n))
    for sj in range(sy):
        for si in range(sx):
            out[sj * sx + si] = field[sj * n:(sj + 1) * n, si * n:(si + 1) * n]
    return out


# ---- the five BASELINE.json configs (optionally shrunk for CPU parity) ------
def config1(seed: int = 1, sx: int = 4, sy: int = 2, n: int = 16, random_blocks: bool = False,
            block: int = 4) -> Problem:
    """C1: T-FETI, multiplicity, single direction, lumped; 4x4-element blocks
    with rho = 0.1 on a seeded checkerboard (phase = seed & 1), else 1.
    ``random_blocks`` is the test-only C1b variant (independent blocks)."""
    gy, gx = sy * n, sx * n
    by, bx = np.meshgrid(np.arange(gy) // block, np.arange(gx) // block, indexing="ij")
    if random_blocks:
        nbx = (gx + block - 1) // block
        nby = (gy + block - 1) // block
        draw = uniform(seed, nbx * nby).reshape(nby, nbx) < 0.5
        low = draw[by, bx]
    else:
        low = (bx + by + (seed & 1)) % 2 == 0
    field = np.where(low, 0.1, 1.0)
    dens = split_global(field, sx, sy, n)
    return Problem(sx, sy, n, dens, np.arange(sx * sy, dtype=np.int32), method=TFETI,
                   scaling=MULTIPLICITY, precond=LUMPED, directions=SINGLE, Emin=1e-9,
                   dirichlet=left_clamp(sx, sy, n), tractions=right_edge_traction(sx, sy, n),
                   name="C1b" if random_blocks else "C1")


def config2(seed: int = 1, sx: int = 8, sy: int = 4, n: int = 32) -> Problem:
    """C2: FETI-DP, k-scaling, single, Dirichlet; rho ~ Bernoulli(0.5) in {0,1},
    Emin = 1e-6; left clamp; unit point load at the bottom-right node."""
    field = (uniform(seed, sy * n * sx * n) < 0.5).astype(np.float64).reshape(sy * n, sx * n)
    dens = split_global(field, sx, sy, n)
    gxn = sx * n + 1
    return Problem(sx, sy, n, dens, np.arange(sx * sy, dtype=np.int32), method=FETIDP,
                   scaling=KSCALING, precond=DIRICHLET, directions=SINGLE, Emin=1e-6,
                   dirichlet=left_clamp(sx, sy, n), point_loads=[(sx * n, 1, -1.0)], name="C2")


def config3(seed: int = 1, method: int = TFETI, sx: int = 16, sy: int = 8, n: int = 32,
            length: float = 4.0) -> Problem:
    """C3: T-FETI or FETI-DP, k-scaling, FO, Dirichlet; thresholded GRF with a
    2-element ramp; pins at the bottom corners; unit load at top mid-span."""
    grf = gaussian_random_field(seed, sy * n, sx * n, length)
    field = ramp(grf > 0.0)
    dens = split_global(field, sx, sy, n)
    gxn = sx * n + 1
    top_mid = (sy * n) * gxn + (sx * n) // 2
    return Problem(sx, sy, n, dens, np.arange(sx * sy, dtype=np.int32), method=method,
                   scaling=KSCALING, precond=DIRICHLET, directions=FO, Emin=1e-9,
                   dirichlet=bottom_corner_pins(sx, sy, n), point_loads=[(top_mid, 1, -1.0)],
                   name="C3-" + ("tfeti" if method == TFETI else "fetidp"))


def config4(seed: int = 1, sx: int = 64, sy: int = 32, n: int = 64) -> Problem:
    """C4: FETI-DP, k-scaling, RRS, Dirichlet; rho ~ U(0,1); left clamp;
    uniform downward traction on the right edge (throughput config)."""
    field = uniform(seed, sy * n * sx * n).reshape(sy * n, sx * n)
    dens = split_global(field, sx, sy, n)
    return Problem(sx, sy, n, dens, np.arange(sx * sy, dtype=np.int32), method=FETIDP,
                   scaling=KSCALING, precond=DIRICHLET, directions=RRS, Emin=1e-9,
                   dirichlet=left_clamp(sx, sy, n), tractions=right_edge_traction(sx, sy, n),
                   name="C4")


def config5(seed: int = 1, sx: int = 32, sy: int = 16, n: int = 48, n_designs: int = 10,
            length: float = 6.0, volume_fraction: float = 0.4) -> Problem:
    """C5: FETI-DP, k-scaling, RRS, Dirichlet with F_s per distinct design;
    10 thresholded-GRF module designs (volume fraction 0.4) placed by a seeded
    uniform assignment; pins at the bottom corners; unit top mid-span load."""
    dens = np.empty((n_designs, n, n))
    for k in range(n_designs):
        grf = gaussian_random_field(seed * 1000 + k, n, n, length)
        thr = np.percentile(grf, 100.0 * (1.0 - volume_fraction))
        dens[k] = (grf > thr).astype(np.float64)
    mt = np.minimum((uniform(seed * 7919 + 13, sx * sy) * n_designs).astype(np.int32), n_designs - 1)
    gxn = sx * n + 1
    top_mid = (sy * n) * gxn + (sx * n) // 2
    return Problem(sx, sy, n, dens, mt.astype(np.int32), method=FETIDP, scaling=KSCALING,
                   precond=DIRICHLET, directions=RRS, Emin=1e-9,
                   dirichlet=bottom_corner_pins(sx, sy, n), point_loads=[(top_mid, 1, -1.0)],
                   name="C5")


CONFIGS = {"C1": config1, "C2": config2, "C3": config3, "C4": config4, "C5": config5}


# ---- academic presets (Fig. 2), SURVEY.md 8f rank 3 ----
def _layers(n: int, count: int) -> np.ndarray:
    """n x n module with `count` horizontal layers alternating stiff (1) /
    compliant (0), stiff at the bottom; n must be divisible by count."""
    if n % count:
        raise ValueError("element rows per subdomain must be divisible by the layer count")
    rows = (np.arange(n) // (n // count)) % 2 == 0
    return np.repeat(rows[:, None], n, axis=1).astype(np.float64)


def laminated_beam(n: int = 14, count: int = 9, layers: int = 7, contrast: float = 1e4,
                   method: int = TFETI, scaling: int = KSCALING, precond: int = DIRICHLET) -> Problem:
    """1 x 9 row of square modules with 7 alternating layers, clamped left,
    tensile normal + tangential traction on the right edge."""
    dens = _layers(n, layers)[None]
    return Problem(count, 1, n, dens, np.zeros(count, np.int32), method=method, scaling=scaling,
                   precond=precond, Emin=1.0 / contrast, p=1.0, dirichlet=left_clamp(count, 1, n),
                   tractions=[(count - 1, RIGHT, 0, n, 1.0, 1.0)], name="laminated_beam")


def grid3x3_layered(n: int = 14, layers: int = 7, contrast: float = 1e4, method: int = TFETI,
                    scaling: int = KSCALING, precond: int = DIRICHLET) -> Problem:
    """3 x 3 grid of layered modules (cross points)."""
    dens = _layers(n, layers)[None]
    return Problem(3, 3, n, dens, np.zeros(9, np.int32), method=method, scaling=scaling, precond=precond,
                   Emin=1.0 / contrast, p=1.0, dirichlet=left_clamp(3, 3, n),
                   tractions=[(sj * 3 + 2, RIGHT, 0, n, 1.0, 1.0) for sj in range(3)], name="grid3x3_layered")


def grid4x4_inclusion(n: int = 8, contrast: float = 1e4, inclusion: int = None, method: int = TFETI,
                      scaling: int = KSCALING, precond: int = DIRICHLET) -> Problem:
    """4 x 4 grid of compliant modules each with a centred stiff square
    inclusion that does not touch the module boundary."""
    inc = n // 2 if inclusion is None else inclusion
    d = np.zeros((n, n))
    a = (n - inc) // 2
    if inc > 0:
        d[a:a + inc, a:a + inc] = 1.0
    return Problem(4, 4, n, d[None], np.zeros(16, np.int32), method=method, scaling=scaling, precond=precond,
                   Emin=1.0 / contrast, p=1.0, dirichlet=left_clamp(4, 4, n),
                   tractions=[(sj * 4 + 3, RIGHT, 0, n, 1.0, 1.0) for sj in range(4)], name="grid4x4_inclusion")


PRESETS = {"laminated_beam": laminated_beam, "grid3x3_layered": grid3x3_layered,
           "grid4x4_inclusion": grid4x4_inclusion}
