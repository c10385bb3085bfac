"""Restarted, right-preconditioned GMRES(m) (Saad & Schultz), the Krylov solver
the paper drives BILU with: "restarted GMRES ... with restart length 30 until the
relative residual is reduced by 10^-6 ... the vector b with all ones"
(PAPER.md:1062-1067).  BASELINE asks for 1e-8.  Readings:
right preconditioning, x0 = 0, modified Gram-Schmidt, Givens rotations, the
count is the number of inner (Arnoldi) steps, at most `max_restarts` cycles.
Convergence is declared on the true residual ||b - A x|| / ||b||.
"""
from __future__ import annotations

import numpy as np


def gmres(matvec, b, precond=None, restart=30, tol=1e-8, max_restarts=100):
    """Returns (x, iterations, converged, relres_history)."""
    b = np.asarray(b, dtype=np.float64)
    n = b.shape[0]
    M = precond if precond is not None else (lambda v: v)
    x = np.zeros(n)
    bnorm = np.linalg.norm(b)
    if bnorm == 0.0:
        return x, 0, True, [0.0]
    r = b.copy()
    beta = np.linalg.norm(r)
    hist = [beta / bnorm]
    its = 0
    for _ in range(max_restarts):
        if beta / bnorm <= tol:
            return x, its, True, hist
        V = np.zeros((restart + 1, n))
        Z = np.zeros((restart, n))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        g[0] = beta
        V[0] = r / beta
        k_used = 0
        for k in range(restart):
            Z[k] = M(V[k])
            w = matvec(Z[k])
            for i in range(k + 1):               # modified Gram-Schmidt
                H[i, k] = np.dot(w, V[i])
                w = w - H[i, k] * V[i]
            H[k + 1, k] = np.linalg.norm(w)
            hnext = H[k + 1, k]
            for i in range(k):                   # apply the previous rotations
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            den = np.hypot(H[k, k], H[k + 1, k])
            cs[k] = H[k, k] / den if den else 1.0
            sn[k] = H[k + 1, k] / den if den else 0.0
            H[k, k] = den
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            its += 1
            k_used = k + 1
            hist.append(abs(g[k + 1]) / bnorm)
            if abs(g[k + 1]) / bnorm <= tol or hnext == 0.0:
                break
            V[k + 1] = w / hnext
        y = np.zeros(k_used)
        for i in range(k_used - 1, -1, -1):      # back substitution
            y[i] = (g[i] - np.dot(H[i, i + 1:k_used], y[i + 1:k_used])) / H[i, i]
        x = x + Z[:k_used].T @ y
        r = b - matvec(x)
        beta = np.linalg.norm(r)
        hist[-1] = beta / bnorm
        if beta / bnorm <= tol:
            return x, its, True, hist
    return x, its, False, hist
