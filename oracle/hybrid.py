"""Oracle of the hybrid-VSIE system operator that the GMRES consumer applies.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs; never by the product path.

The system of Eq. 15 with unknowns x = [j_f (m_f); j_n (m_n); j_b (3 n_v)]:

    [ Z_cc^ff       V-bar U^T    (Z_cb^f)^T ] [j_f]   [v_f]
    [ U V^*         Z_cc^nn      (Z_cb^n)^T ] [j_n] = [v_n]
    [ Z_cb^f        Z_cb^n       Z_bb       ] [j_b]   [ 0 ]

(the lower-right 2 x 2 is Z^pFFT_HOSVD of P:165-167).  Blocks, each from its own oracle:
  Z_cc^ff  dense far-far Galerkin EFIE (oracle/farfar.py),
  U V^*    the far-near block Z_cc^fn (oracle/farnear.py, dense: ACA at full rank is exact),
  Z_cc^nn  the same EFIE Galerkin machinery on the near mesh ("Galerkin matrices ... of
           the m_n near ... elements"),
  Z_cb^f   the TT-compressed far coupling (oracle/ttmv.py applies of the chi TTs, Eq. 14),
  Z_cb^n   the near coupling, here also a TT of the same entry function on the near mesh (the
           paper projects it with pFFT: out of scope, reading R-G1),
  Z_bb     its local part only: the multiplication operator M_eps_r of the VIE (Eq. 2)
           tested with PWC functions, h1 h2 h3 eps_r(voxel) per unknown (a diagonal d_b); the
           nonlocal M_chi N part (FFT-based) is out of scope (reading R-G1).
Plain transposes (Eq. 15 writes V-bar U^T and [Z~^1 ... Z~^q]^T).
"""
import numpy as np

from . import ttmv


def matvec(blocks, x):
    """y = A x of the module docstring; blocks: dict with Zff [m_f x m_f], Zfn [m_n x m_f],
    Znn [m_n x m_n], tt_far / tt_near (lists of 3 chi TTs, cores per ttmv), d_body [3 n_v]."""
    mf = blocks["Zff"].shape[0]
    mn = blocks["Znn"].shape[0]
    x = np.asarray(x, dtype=np.complex128)
    jf, jn, jb = x[:mf], x[mf:mf + mn], x[mf + mn:]
    yf = blocks["Zff"] @ jf + blocks["Zfn"].T @ jn + ttmv.apply(blocks["tt_far"], jb, "T")
    yn = blocks["Zfn"] @ jf + blocks["Znn"] @ jn + ttmv.apply(blocks["tt_near"], jb, "T")
    yb = ttmv.apply(blocks["tt_far"], jf, "N") + ttmv.apply(blocks["tt_near"], jn, "N") + blocks["d_body"] * jb
    return np.concatenate([yf, yn, yb])


def body_diagonal(n, h, eps_r):
    """d_b = h1 h2 h3 eps_r(v) for the three chi blocks (chi-major, voxel index i1 fastest, the
    row order of Z_cb): the PWC Galerkin test of M_eps_r (Eq. 2)."""
    vol = float(h[0] * h[1] * h[2])
    e = np.asarray(eps_r, dtype=np.complex128).reshape(-1)
    assert e.size == n[0] * n[1] * n[2]
    return np.tile(vol * e, 3)
