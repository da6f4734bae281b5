"""Oracle of the GMRES consumer of the hybrid VSIE system.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs; never by the product path.

What is computed ("Solving the hybrid-VSIE": "an iterative solver, like
the generalized minimal residual method (GMRES) [saad1986gmres], should be used"; "The
tolerance was set to 1e-5. GMRES' restarts were set to 50"):

  restarted GMRES(m) of Saad & Schultz for A x = b, x0 = 0, in the textbook order:
    r0 = b - A x0, beta = ||r0||, v1 = r0 / beta
    for j = 1..m (Arnoldi):  w = A v_j
                             h_{i,j} = v_i^H w, w -= sum_i h_{i,j} v_i     (i = 1..j)
                             (classical Gram-Schmidt, then the same once more on w and the
                              coefficients added: CGS2, reading R-G2)
                             h_{j+1,j} = ||w||, v_{j+1} = w / h_{j+1,j}
                             apply the previous Givens rotations to column j of H, form the
                             rotation that zeroes h_{j+1,j}, apply it to g = beta e1
                             |g_{j+1}| is the residual norm of the least-squares iterate
                             stop the cycle when |g_{j+1}| <= tol ||b|| or j = m
    y = H_j^{-1} g_{1..j} (upper-triangular back substitution), x += V_j y; restart from x.
  Stop: relative residual estimate |g_{j+1}| / ||b|| <= tol, or max_iter matvecs.

Pinned by tests/test_oracle_pins.py P52 (exact solve in n steps for n x n, the Arnoldi
relation A V_k = V_{k+1} H_k, the residual estimate equal to the true residual, identity and
scaled-identity operators in one step, monotone residuals within a cycle, restart behaviour).
"""
import numpy as np


def givens(a, b):
    """(c, s) with [c s; -conj(s) c] [a; b] = [r; 0], c real >= 0 (complex Givens)."""
    if b == 0:
        return 1.0, 0.0 + 0.0j
    if a == 0:
        return 0.0, np.conj(b) / abs(b)
    t = np.hypot(abs(a), abs(b))
    c = abs(a) / t
    s = (a / abs(a)) * np.conj(b) / t
    return c, s


def gmres(matvec, b, tol=1e-5, restart=50, max_iter=1000, history=None):
    """Restarted GMRES(restart) from x0 = 0 (module docstring).  Returns (x, iterations,
    relative residual estimate).  history: list receiving |g_{j+1}| / ||b|| per iteration.
    H holds the Hessenberg columns after their Givens rotations (the triangle R of the
    least-squares problem); arnoldi() gives the unrotated process."""
    b = np.asarray(b, dtype=np.complex128)
    n = b.shape[0]
    x = np.zeros(n, dtype=np.complex128)
    bn = np.linalg.norm(b)
    if bn == 0:
        return x, 0, 0.0
    its = 0
    rel = 1.0
    while its < max_iter:
        r = b - matvec(x) if its > 0 else b.copy()
        beta = np.linalg.norm(r)
        rel = beta / bn
        if rel <= tol:
            break
        m = restart
        V = np.zeros((n, m + 1), dtype=np.complex128)
        H = np.zeros((m + 1, m), dtype=np.complex128)
        cs = np.zeros(m)
        sn = np.zeros(m, dtype=np.complex128)
        g = np.zeros(m + 1, dtype=np.complex128)
        g[0] = beta
        V[:, 0] = r / beta
        j = 0
        while j < m and its < max_iter:
            w = matvec(V[:, j])
            its += 1
            h = V[:, : j + 1].conj().T @ w
            w = w - V[:, : j + 1] @ h
            h2 = V[:, : j + 1].conj().T @ w          # CGS2: one reorthogonalisation
            w = w - V[:, : j + 1] @ h2
            h = h + h2
            hn = np.linalg.norm(w)
            H[: j + 1, j] = h
            H[j + 1, j] = hn
            if hn > 0:
                V[:, j + 1] = w / hn
            # Givens rotations on the new column
            col = H[: j + 2, j].copy()
            for i in range(j):
                t = cs[i] * col[i] + sn[i] * col[i + 1]
                col[i + 1] = -np.conj(sn[i]) * col[i] + cs[i] * col[i + 1]
                col[i] = t
            c, s = givens(col[j], col[j + 1])
            cs[j], sn[j] = c, s
            col[j] = c * col[j] + s * col[j + 1]
            col[j + 1] = 0
            g[j + 1] = -np.conj(s) * g[j]
            g[j] = c * g[j]
            H[: j + 2, j] = col
            j += 1
            rel = abs(g[j]) / bn
            if history is not None:
                history.append(rel)
            if rel <= tol or hn == 0:
                break
        # y from the rotated triangle R = H[:j, :j]
        Rt = H[:j, :j]
        y = np.zeros(j, dtype=np.complex128)
        for i in range(j - 1, -1, -1):
            y[i] = (g[i] - Rt[i, i + 1: j] @ y[i + 1: j]) / Rt[i, i]
        x = x + V[:, :j] @ y
        if rel <= tol:
            break
    return x, its, rel


def arnoldi(matvec, v0, k):
    """k steps of the CGS2 Arnoldi process of gmres() from v0 (unrotated): V [n x (k+1)],
    H [(k+1) x k] with A V_k = V_{k+1} H (the relation pinned by P52)."""
    v0 = np.asarray(v0, dtype=np.complex128)
    n = v0.shape[0]
    V = np.zeros((n, k + 1), dtype=np.complex128)
    H = np.zeros((k + 1, k), dtype=np.complex128)
    V[:, 0] = v0 / np.linalg.norm(v0)
    for j in range(k):
        w = matvec(V[:, j])
        h = V[:, : j + 1].conj().T @ w
        w = w - V[:, : j + 1] @ h
        h2 = V[:, : j + 1].conj().T @ w
        w = w - V[:, : j + 1] @ h2
        H[: j + 1, j] = h + h2
        H[j + 1, j] = np.linalg.norm(w)
        V[:, j + 1] = w / H[j + 1, j]
    return V, H
