"""The algebra behind the implicit RRS direction store (solve_rrs.cuh,
solve_rrs_implicit), checked in numpy on a small synthetic dual problem.

Alg. 1 with the explicit store keeps W_j and Q_j = F W_j.
The implicit store keeps the per-iteration preconditioner blocks Z_l (column s
supported on "subdomain" s's rows only) and coefficient matrices M_j with
W_j = sum_l Z_l M_j[l]; because F is symmetric, Psi_j = Q_j^T V = W_j^T (F V),
so no Q_j is stored.  Both variants must produce the same iterates up to
rounding.  No GPU: this pins the reformulation itself.
"""
import numpy as np


def _problem(seed=0, ns=6, rows_per=5, overlap=2):
    rng = np.random.default_rng(seed)
    supports = []
    r0 = 0
    for s in range(ns):
        supports.append(np.arange(r0, r0 + rows_per))
        r0 += rows_per - overlap
    m = r0 + overlap
    A = rng.standard_normal((m, m))
    F = A @ A.T + 0.5 * np.eye(m)                       # SPD dual operator
    d = rng.standard_normal(m)
    Ms = [np.diag(rng.uniform(0.5, 2.0, len(sp))) for sp in supports]   # local preconditioners

    def precond_cols(r):
        Z = np.zeros((m, ns))
        for s, sp in enumerate(supports):
            Z[sp, s] = Ms[s] @ r[sp]
        return Z

    return F, d, precond_cols, supports


def _pivchol(D, tol=1e-12):
    """Alg. 1 line 9: symmetric pivoting by the largest remaining diagonal."""
    A = D.copy()
    n = A.shape[0]
    perm = np.arange(n)
    scale = max(np.max(np.diag(A)), 0.0)
    L = np.zeros((n, n))
    k = 0
    for k in range(n):
        j = k + int(np.argmax(np.diag(A)[k:]))
        if A[j, j] <= tol * scale:
            break
        A[[k, j]] = A[[j, k]]
        A[:, [k, j]] = A[:, [j, k]]
        L[[k, j]] = L[[j, k]]
        perm[[k, j]] = perm[[j, k]]
        L[k, k] = np.sqrt(A[k, k])
        L[k + 1:, k] = A[k + 1:, k] / L[k, k]
        A[k + 1:, k + 1:] -= np.outer(L[k + 1:, k], L[k + 1:, k])
    else:
        k = n
    return perm, L[:k, :k], k


def _rrs(F, d, precond_cols, iters, implicit, passes=2):
    m = len(d)
    lam = np.zeros(m)
    r = d - F @ lam
    V = precond_cols(r)
    Zs, Ms, CW = [V.copy()], [], np.eye(V.shape[1])       # implicit: Z blocks, M_j, coordinates of V
    Ws, Qs = [], []                                       # explicit store
    kept = []
    for _ in range(iters):
        Q = F @ V
        Delta = Q.T @ V
        perm, Lt, rank = _pivchol(Delta)
        if rank == 0:
            break
        Linv = np.linalg.inv(Lt)
        Wn = V[:, perm[:rank]] @ Linv.T
        Qn = Q[:, perm[:rank]] @ Linv.T
        if implicit:
            Ms.append(CW[:, perm[:rank]] @ Linv.T)
        else:
            Ws.append(Wn)
            Qs.append(Qn)
        kept.append(rank)
        gamma = Wn.T @ r
        lam = lam + Wn @ gamma
        r = r - Qn @ gamma
        V = precond_cols(r)
        if implicit:
            Zhat = np.hstack(Zs)
            Zs.append(V.copy())
            Ntot = np.zeros((Zhat.shape[1], V.shape[1]))
            for _ in range(passes):
                X = Zhat.T @ (F @ V)                      # W_j^T F V = Psi_j (F symmetric)
                N = sum(np.vstack([Mj, np.zeros((Zhat.shape[1] - Mj.shape[0], Mj.shape[1]))]) @
                        (Mj.T @ X[:Mj.shape[0]]) for Mj in Ms)
                V = V - Zhat @ N
                Ntot += N
            CW = np.vstack([-Ntot, np.eye(V.shape[1])])
        else:
            for _ in range(passes):
                for Wj, Qj in zip(Ws, Qs):
                    V = V - Wj @ (Qj.T @ V)
    return lam, kept


def test_implicit_store_matches_explicit_store():
    F, d, pc, _ = _problem()
    le, ke = _rrs(F, d, pc, iters=4, implicit=False)
    li, ki = _rrs(F, d, pc, iters=4, implicit=True)
    assert ke == ki
    assert np.linalg.norm(li - le) <= 1e-9 * np.linalg.norm(le)


def test_implicit_store_solves_the_dual_problem():
    F, d, pc, _ = _problem(seed=3)
    lam, kept = _rrs(F, d, pc, iters=12, implicit=True)
    assert np.linalg.norm(d - F @ lam) <= 1e-8 * np.linalg.norm(d)


def test_stored_directions_are_F_orthonormal_in_coordinates():
    """The coefficient form keeps W_all^T F W_all = I (Alg. 1 line 11)."""
    F, d, pc, supports = _problem(seed=5)
    m = len(d)
    lam = np.zeros(m)
    r = d.copy()
    V = pc(r)
    Zs, Ms, CW = [V.copy()], [], np.eye(V.shape[1])
    for _ in range(3):
        Q = F @ V
        perm, Lt, rank = _pivchol(Q.T @ V)
        Linv = np.linalg.inv(Lt)
        Ms.append(CW[:, perm[:rank]] @ Linv.T)
        Wn = V[:, perm[:rank]] @ Linv.T
        g = Wn.T @ r
        lam += Wn @ g
        r -= Q[:, perm[:rank]] @ Linv.T @ g
        V = pc(r)
        Zhat = np.hstack(Zs)
        Zs.append(V.copy())
        Ntot = 0
        for _ in range(2):
            X = Zhat.T @ (F @ V)
            N = sum(np.vstack([Mj, np.zeros((Zhat.shape[1] - Mj.shape[0], Mj.shape[1]))]) @
                    (Mj.T @ X[:Mj.shape[0]]) for Mj in Ms)
            V = V - Zhat @ N
            Ntot = Ntot + N
        CW = np.vstack([-Ntot, np.eye(V.shape[1])])
    Zall = np.hstack(Zs[:-1])
    W = np.hstack([Zall[:, :Mj.shape[0]] @ Mj for Mj in Ms])
    G = W.T @ F @ W
    assert np.abs(G - np.eye(G.shape[0])).max() <= 1e-8
    # every packed Z column lives on its subdomain's rows
    for Z in Zs:
        for s, sp in enumerate(supports):
            off = np.setdiff1d(np.arange(m), sp)
            assert np.all(Z[off, s] == 0.0)
