"""Iterative solve of the AIMx EFIE per frequency (oracle).  TEST INFRASTRUCTURE ONLY.

P:727-728  "The GMRES iterative solver [gmres] available in PETSc was used to
            solve (eq:EFIEAIMx) ... A relative residual norm of 10^-4 was used
            as the convergence tolerance."
P:340-359  sec:methods:aimx:pc -- diagonal preconditioning with the diagonal of
            the frequency-independent L_s instead of diag(L(k0)); P:811 names it
            "the preconditioner based on frequency-independent self-terms of
            L^A_NR and L^phi_NR".

Reading (R19): M(k0) = diag( -j w mu0 (L^A_s,NR[m,m] + k0^-2 L^phi_s,NR[m,m]) )
with L^phi = -y^rho (AMB-13), applied on the right (Z M^-1 u = b, x = M^-1 u),
so the residual GMRES minimises is the true residual of Z x = b.

GMRES(m) as in Saad & Schultz (1986) / Saad, "Iterative Methods for Sparse
Linear Systems", Algorithm 6.9 (restarted) with Arnoldi by modified
Gram-Schmidt and the Hessenberg least-squares problem solved by Givens
rotations; x0 = 0.  Plain loops, complex128.
"""
from __future__ import annotations

import numpy as np

from .aimx import AIMxOracle
from .kernels import MU0


def static_diagonal(op: AIMxOracle):
    """(L^A_s,NR[m,m], y^rho_s,NR[m,m]) -- the self terms of the static near
    matrices (every row's near list contains m itself)."""
    dA = np.empty(op.N)
    dR = np.empty(op.N)
    for m in range(op.N):
        lo, hi = op.rowptr[m], op.rowptr[m + 1]
        k = lo + int(np.nonzero(op.col[lo:hi] == m)[0][0])
        dA[m] = op.LA_NR[k]
        dR[m] = op.YR_NR[k]
    return dA, dR


def preconditioner(op: AIMxOracle, dA, dR):
    """Diagonal of M(k0) at the bound frequency."""
    return -1j * op.omega * MU0 * (dA - dR / (op.k0 * op.k0))


def gmres(matvec, b, Minv, tol=1e-4, restart=30, maxiter=1000):
    """Right-preconditioned restarted GMRES for A x = b with x0 = 0.

    matvec: x -> A x; Minv: diagonal of M^-1 (vector).  Stops when
    ||b - A x|| / ||b|| <= tol (the GMRES residual estimate, which equals the
    true residual in exact arithmetic).  Returns (x, iterations, history of
    relative residual estimates, one per iteration)."""
    b = np.asarray(b, np.complex128)
    n = b.shape[0]
    bnorm = np.linalg.norm(b)
    x = np.zeros(n, np.complex128)
    hist = []
    if bnorm == 0.0:
        return x, 0, hist
    it = 0
    while it < maxiter:
        r = b - matvec(x) if it > 0 else b.copy()
        beta = np.linalg.norm(r)
        if beta / bnorm <= tol:
            break
        V = np.zeros((restart + 1, n), np.complex128)
        H = np.zeros((restart + 1, restart), np.complex128)
        cs = np.zeros(restart, np.complex128)
        sn = np.zeros(restart, np.complex128)
        g = np.zeros(restart + 1, np.complex128)
        g[0] = beta
        V[0] = r / beta
        k_used = 0
        for j in range(restart):
            w = matvec(Minv * V[j])
            for i in range(j + 1):                      # modified Gram-Schmidt
                H[i, j] = np.vdot(V[i], w)
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] != 0.0:
                V[j + 1] = w / H[j + 1, j]
            # Givens rotation i acts on rows (i, i+1) as [[conj(c), conj(s)], [-s, c]]
            # with c = a / rho, s = b / rho, rho = sqrt(|a|^2 + |b|^2): (a, b) -> (rho, 0)
            for i in range(j):                          # previous rotations
                t = np.conj(cs[i]) * H[i, j] + np.conj(sn[i]) * H[i + 1, j]
                H[i + 1, j] = -sn[i] * H[i, j] + cs[i] * H[i + 1, j]
                H[i, j] = t
            a, c = H[j, j], H[j + 1, j]                 # new rotation zeroing H[j+1, j]
            den = np.sqrt(abs(a) ** 2 + abs(c) ** 2)
            cs[j] = a / den if den != 0 else 1.0
            sn[j] = c / den if den != 0 else 0.0
            H[j, j] = den
            H[j + 1, j] = 0.0
            g[j + 1] = -sn[j] * g[j]
            g[j] = np.conj(cs[j]) * g[j]
            it += 1
            k_used = j + 1
            hist.append(abs(g[j + 1]) / bnorm)
            if abs(g[j + 1]) / bnorm <= tol or it >= maxiter:
                break
        y = np.zeros(k_used, np.complex128)             # back substitution H y = g
        for i in range(k_used - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k_used] @ y[i + 1:k_used]) / H[i, i]
        x = x + Minv * (y @ V[:k_used])
        if hist and hist[-1] <= tol:
            break
    return x, it, hist


def solve(op: AIMxOracle, f_hz, b, tol=1e-4, restart=30, maxiter=1000):
    """Solve Z(f) x = b with the static diagonal preconditioner."""
    op.set_frequency(f_hz)
    dA, dR = static_diagonal(op)
    Minv = 1.0 / preconditioner(op, dA, dR)
    return gmres(op.matvec, b, Minv, tol, restart, maxiter)
