"""Subdomain-sharded F-apply and PCG over several GPUs.

One process per GPU.  The module grid is cut into row bands (rank r owns the
module rows [sy r / N, sy (r+1) / N), a contiguous subdomain range, so the
device kernels run on a slice of their per-subdomain descriptor arrays).
Every rank holds the full problem's operators (a replicated build: the
apply work is what shards; memory is not the constraint on one B200, where
C4 fits), applies only its own subdomains, and exchanges:

* FETI-DP coarse step: the owned t_s = A''_s^T x_s (tot_c values over all
  subdomains, zero outside the owned slice) are summed over ranks -- exact,
  one nonzero contributor per entry -- so every rank gathers
  g = sum_s B_c^T t_s in the fixed owner order and solves the coarse problem
  redundantly (no reduction-order dependence);
* halo rows: a dual row whose two owners sit on different ranks gets one
  partial from each; the partials are summed over ranks on the compact list
  of halo rows (a + b == b + a exactly, zeros elsewhere), so the N-rank
  apply equals the 1-GPU apply bit for bit;
* PCG scalars: each dual row is counted by the rank of its first owner, and
  the partial dot products are summed over ranks (allreduce of 8-byte
  scalars; their order differs from the 1-GPU reduction, so iterates agree to
  rounding, not bitwise).

The exchanges go through a small communicator interface: ``TorchComm`` wraps
torch.distributed (NCCL on GPUs, gloo on CPU), ``LocalComm`` emulates N
ranks inside one process (tests on one GPU).  Reference: the reference has no
distributed backend; its per-subdomain fan-out with fixed-order
reductions is what the exchanges preserve.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np


def row_bands(sx: int, sy: int, nranks: int) -> List[tuple]:
    """Owned subdomain ranges [s0, s1) of a row-band partition of the
    sx x sy module grid (subdomain s = sj * sx + si)."""
    out = []
    for r in range(nranks):
        j0, j1 = sy * r // nranks, sy * (r + 1) // nranks
        out.append((j0 * sx, j1 * sx))
    return out


class ShardPlan:
    """Exchange bookkeeping of a partition: which ranks own each subdomain,
    the rows every rank touches, the halo rows (owners on two ranks, global
    order, identical on every rank) and the rows each rank counts in dot
    products (first owner's rank)."""

    def __init__(self, rows: dict, ranges: Sequence[tuple]):
        self.ranges = list(ranges)
        n_sub = max(r[1] for r in self.ranges)
        self.rank_of_sub = np.full(n_sub, -1, dtype=np.int64)
        for rk, (s0, s1) in enumerate(self.ranges):
            self.rank_of_sub[s0:s1] = rk
        sp = np.asarray(rows["sub_plus"], dtype=np.int64)
        sm = np.asarray(rows["sub_minus"], dtype=np.int64)
        self.m = len(sp)
        ra = self.rank_of_sub[sp]
        rb = np.where(sm >= 0, self.rank_of_sub[np.maximum(sm, 0)], ra)
        self.row_ranks = (ra, rb)
        self.halo = np.nonzero(ra != rb)[0].astype(np.int64)           # global order
        self.dot_rank = np.minimum(ra, rb)                                # row counted once

    def touched(self, rank: int) -> np.ndarray:
        ra, rb = self.row_ranks
        return np.nonzero((ra == rank) | (rb == rank))[0]

    def dot_mask(self, rank: int) -> np.ndarray:
        return (self.dot_rank == rank).astype(np.float64)


# ------------------------------------------------------------ communicators
class TorchComm:
    """torch.distributed sum-allreduce of torch tensors (NCCL or gloo)."""

    def __init__(self, dist, device):
        self.dist = dist
        self.device = device
        self.rank = dist.get_rank()
        self.size = dist.get_world_size()

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM)
        return t


class LocalComm:
    """N emulated ranks in one process, one host thread each (tests on one
    GPU): ``rank(r)`` returns rank r's communicator.  allreduce_sum deposits
    the rank's tensor, waits for all ranks, and every rank adds the deposits
    in rank order (deterministic)."""

    def __init__(self, n: int):
        import threading
        self.n = n
        self.slots = [None] * n
        self.bar = threading.Barrier(n)

    def rank(self, r: int):
        return _LocalRank(self, r)


class _LocalRank:
    def __init__(self, c: LocalComm, r: int):
        self.c, self.rank, self.size = c, r, c.n

    def allreduce_sum(self, t):
        c = self.c
        c.slots[self.rank] = t.clone()
        c.bar.wait()
        acc = c.slots[0].clone()
        for k in range(1, c.n):
            acc += c.slots[k]
        c.bar.wait()
        t.copy_(acc)
        return t


# --------------------------------------------------- sharded device system
class ShardedSystem:
    """One rank's view: a full FetiSystem (engine.FetiSystem) restricted to
    the rank's subdomains for F / preconditioner applies.  Vectors are torch
    CUDA tensors of length m (the rows the rank touches are kept exact)."""

    def __init__(self, system, rank: int, ranges: Sequence[tuple], comm=None):
        import torch
        from . import engine
        self.g = system
        self.rank = rank
        self.comm = comm
        self.plan = ShardPlan(system.rows(), ranges)
        s0, s1 = ranges[rank]
        engine.check(engine.lib().fetigpu_shard_set_range(system.h, s0, s1))
        tc = C.c_int()
        engine.check(engine.lib().fetigpu_shard_info(system.h, C.byref(tc)))
        self.tot_c = tc.value
        self.m = system.m
        dev = torch.device("cuda", torch.cuda.current_device())
        self.dev = dev
        self.halo = torch.as_tensor(self.plan.halo, device=dev)
        self.mask = torch.as_tensor(self.plan.dot_mask(rank), device=dev)
        self.tbuf = torch.zeros(max(1, self.tot_c), dtype=torch.float64, device=dev)

    # phase 1 / 2 through the C-ABI on the context stream, then a device sync
    # before torch touches the buffers (torch uses its own stream)
    def _p(self, t):
        return C.cast(C.c_void_p(t.data_ptr()), C.POINTER(C.c_double))

    def phase1(self, x, y, precond=False):
        import torch
        from . import engine
        L = engine.lib()
        self.tbuf.zero_()
        torch.cuda.current_stream().synchronize()    # torch-side producers of x / tbuf
        engine.check(L.fetigpu_shard_phase1_device(self.g.h, self._p(x), self._p(y), self._p(self.tbuf),
                                                   int(precond)))
        engine.check(L.fetigpu_synchronize(self.g.h))

    def phase2(self, tall, y):
        import torch
        from . import engine
        L = engine.lib()
        torch.cuda.current_stream().synchronize()
        engine.check(L.fetigpu_shard_phase2_device(self.g.h, self._p(tall), self._p(y)))
        engine.check(L.fetigpu_synchronize(self.g.h))

    def apply(self, x, precond=False):
        """y = F x (or the preconditioner), exact on the rows this rank touches."""
        import torch
        y = torch.empty(self.m, dtype=torch.float64, device=self.dev)
        self.phase1(x, y, precond)
        if not precond and self.g.prob.method == 1:
            self.comm.allreduce_sum(self.tbuf)
            self.phase2(self.tbuf, y)
        if self.halo.numel():
            h = y.index_select(0, self.halo)
            self.comm.allreduce_sum(h)
            y.index_copy_(0, self.halo, h)
        return y

    def dot(self, a, b):
        import torch
        t = torch.stack([(a * b * self.mask).sum()])
        self.comm.allreduce_sum(t)
        return float(t.item())


def apply_emulated(systems: Sequence[ShardedSystem], xs, precond=False):
    """N ranks inside one process (one GPU): the same phases and exchanges as
    ShardedSystem.apply, with the sum-allreduces done on the device by
    adding the ranks' buffers (in rank order; exact for the same reasons)."""
    import torch
    ys = []
    for s, x in zip(systems, xs):
        y = torch.empty(s.m, dtype=torch.float64, device=s.dev)
        s.phase1(x, y, precond)
        ys.append(y)
    if not precond and systems[0].g.prob.method == 1:
        tall = torch.zeros_like(systems[0].tbuf)
        for s in systems:
            tall += s.tbuf
        for s, y in zip(systems, ys):
            s.phase2(tall, y)
    halo = systems[0].halo
    if halo.numel():
        hs = torch.zeros(halo.numel(), dtype=torch.float64, device=systems[0].dev)
        for y in ys:
            hs += y.index_select(0, halo)
        for y in ys:
            y.index_copy_(0, halo, hs)
    return ys


def sharded_pcg(sh: ShardedSystem, tol: float = 1e-6, max_it: int = 1000, fo: bool = False):
    """PCG (FETI-DP: identity projector) on one rank of the sharded system,
    SPEC.md:426-434 with the relative criterion eps_r(i) / eps_r(0) <= tol;
    fo adds full orthogonalization (CGS, two passes) against the stored
    F-normalised directions.  Returns (lambda, iterations, eps trace).
    Every rank runs it with its own ShardedSystem; vectors stay exact on the
    rows the rank touches, scalars come from the allreduced dot products."""
    import torch
    if sh.g.prob.method != 1:
        raise ValueError("sharded_pcg: FETI-DP only (T-FETI needs the global coarse projector)")
    d, _ = sh.g.rhs()
    dt = torch.as_tensor(d, device=sh.dev)
    lam = torch.zeros(sh.m, dtype=torch.float64, device=sh.dev)
    r = dt.clone()
    z = sh.apply(r, precond=True)
    rz = sh.dot(r, z)
    eps0 = np.sqrt(max(rz, 0.0))
    eps = [eps0]
    w = z.clone()
    Ws, Qs = [], []
    it = 0
    while eps[-1] > tol * eps0 and it < max_it:
        q = sh.apply(w)
        delta = sh.dot(w, q)
        if not delta > 0:
            break
        alpha = (sh.dot(w, r) if fo else rz) / delta
        lam += alpha * w
        r -= alpha * q
        z = sh.apply(r, precond=True)
        rz_new = sh.dot(r, z)
        it += 1
        eps.append(np.sqrt(max(rz_new, 0.0)))
        if fo:
            sd = np.sqrt(delta)
            Ws.append(w / sd)
            Qs.append(q / sd)
            w = z.clone()
            for _ in range(2):
                psi = [sh.dot(qj, w) for qj in Qs]
                for wj, p in zip(Ws, psi):
                    w -= p * wj
        else:
            w = z + (rz_new / rz) * w
        rz = rz_new
    return lam, it, np.array(eps)
