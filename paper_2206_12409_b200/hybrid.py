"""Thin binding of include/vsie_hybrid.h: the hybrid-VSIE operator of Eq. 15
composed from the block handles, and restarted GMRES on it.  Argument
marshalling only: every product and every GMRES vector operation runs in the library."""
import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .coupling import _stream_ptr, _torch


class Hybrid:
    """Z = [[Z_cc^ff, Vbar U^T, Z_cb^f^T], [U V^*, Z_cc^nn, Z_cb^n^T], [Z_cb^f, Z_cb^n, diag(d_b)]].

    ff, cb_far required; fn (FarNear), nn (FarFar on the near meshes), cb_near (Coupling on the
    near meshes) all given or all None; d_body: cuda complex128 [3 n_v].  The block handles
    are referenced (kept alive by this object)."""

    def __init__(self, ff, cb_far, d_body, fn=None, nn=None, cb_near=None):
        self._refs = (ff, cb_far, fn, nn, cb_near)
        h = _lib.HANDLE()
        hv = lambda o: None if o is None else o._h   # noqa: E731
        check(lib().vsie_hybrid_create(hv(ff), hv(fn), hv(nn), hv(cb_far), hv(cb_near),
                                       C.c_void_p(d_body.data_ptr()), C.byref(h)))
        self._h = h

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().vsie_hybrid_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = _lib.vsie_hybrid_info()
        check(lib().vsie_hybrid_get_info(self._h, C.byref(i)))
        return dict(m_far=i.m_far, m_near=i.m_near, n_body=i.n_body, n=i.n, matvecs=i.matvecs)

    def matvec(self, x, out=None, stream=None):
        torch = _torch()
        y = torch.empty_like(x) if out is None else out
        check(lib().vsie_hybrid_matvec(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                       _stream_ptr(stream)))
        return y

    def gmres(self, b, restart=50, max_iter=1000, tol=1e-5, out=None, stream=None):
        """(x, info, history): restarted GMRES from x0 = 0 (vsie_hybrid_gmres)."""
        torch = _torch()
        x = torch.empty_like(b) if out is None else out
        hist = np.zeros(max_iter)
        inf = _lib.vsie_gmres_info()
        st = check(lib().vsie_hybrid_gmres(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), int(restart),
                                           int(max_iter), float(tol), hist.ctypes.data, C.byref(inf),
                                           _stream_ptr(stream)), allow_warn=True)
        info = dict(iterations=inf.iterations, restarts=inf.restarts, converged=bool(inf.converged),
                    rel_residual=inf.rel_residual, seconds=inf.seconds, matvec_seconds=inf.matvec_seconds,
                    status=st)
        return x, info, hist[: inf.iterations]
