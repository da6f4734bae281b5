"""Thin Python wrapper over include/vsie_farnear.h: ``FarNear`` = one ACA-compressed far-near
conductor block Z_cc^fn (Eq. 12; applied as in Eq. 15).

Argument marshalling only: the entries, the ACA and the low-rank products run in
libvsie_coupling.so.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from ._lib import check, lib
from .coupling import _meshes_c, _stream_ptr, _torch

STOPS = {0: "tol", 1: "max_rank", 2: "rows_exhausted"}


class FarNear:
    def __init__(self, handle, status=0):
        self._h = _lib.HANDLE(handle)
        self.status = status

    @classmethod
    def build(cls, near_meshes, far_meshes, freq: float, tol: float, max_rank=None, scale=None, device=None,
              verbose=None):
        """vsie_farnear_build: device ACA of Z_cc^fn (near rows, far columns)."""
        an, kn = _meshes_c(near_meshes)
        af, kf = _meshes_c(far_meshes)
        o = _lib.vsie_farnear_opts()
        lib().vsie_farnear_opts_default(C.byref(o))
        if max_rank is not None:
            o.max_rank = int(max_rank)
        if scale is not None:
            o.scale_re, o.scale_im = float(np.real(scale)), float(np.imag(scale))
        if device is not None:
            o.device = int(device)
        if verbose is not None:
            o.verbose = int(verbose)
        h = _lib.HANDLE()
        st = lib().vsie_farnear_build(an, len(near_meshes), af, len(far_meshes), float(freq), float(tol), C.byref(o),
                                      C.byref(h))
        check(st, allow_warn=True)
        del kn, kf
        return cls(h.value, st)

    def close(self):
        if self._h is not None and self._h.value:
            lib().vsie_farnear_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def info(self) -> dict:
        i = _lib.vsie_farnear_info()
        check(lib().vsie_farnear_get_info(self._h, C.byref(i)))
        return dict(m_near=i.m_near, m_far=i.m_far, rank=i.rank, stop=STOPS.get(i.stop, i.stop), est_err=i.est_err,
                    frob=i.frob, min_distance=i.min_distance, max_edge=i.max_edge, k0=i.k0, build_s=i.build_s,
                    entries_evaluated=i.entries_evaluated, factor_bytes=i.factor_bytes, apply_calls=i.apply_calls)

    def export(self):
        """(U [m_n, k], W [m_f, k], pivot rows [k], pivot cols [k]) on host; Z^fn ~= U W^T."""
        inf = self.info()
        k = inf["rank"]
        U = np.empty((inf["m_near"], k), dtype=np.complex128, order="F")
        W = np.empty((inf["m_far"], k), dtype=np.complex128, order="F")
        rows = np.empty(k, dtype=np.int32)
        cols = np.empty(k, dtype=np.int32)
        check(lib().vsie_farnear_export(self._h, U.ctypes.data, W.ctypes.data, rows.ctypes.data, cols.ctypes.data))
        return U, W, rows, cols

    def entries(self, rows, cols, stream=None):
        """Exact Z^fn[rows[i], cols[i]] on device (CUDA complex128 tensor)."""
        torch = _torch()
        idx = torch.stack([torch.as_tensor(rows, dtype=torch.int64), torch.as_tensor(cols, dtype=torch.int64)],
                          dim=1).contiguous().cuda()
        out = torch.empty(idx.shape[0], dtype=torch.complex128, device=idx.device)
        check(lib().vsie_farnear_entries(self._h, C.c_void_p(idx.data_ptr()), idx.shape[0], C.c_void_p(out.data_ptr()),
                                         _stream_ptr(stream)))
        return out

    def apply(self, x, op: str = "N", out=None, stream=None):
        """op N: y = U W^T x (x far [m_f(, nrhs)]); T: W U^T x; C: conj(W) U^H x (x near)."""
        torch = _torch()
        inf = self.info()
        n_out = inf["m_near"] if op == "N" else inf["m_far"]
        vec = x.dim() == 1
        X = x.reshape(-1, 1) if vec else x
        nrhs = X.shape[1]
        Xc = X.t().contiguous()
        Y = torch.empty((nrhs, n_out), dtype=torch.complex128, device=x.device) if out is None else \
            (out.reshape(-1, 1).t() if vec else out.t())
        check(lib().vsie_farnear_apply(self._h, C.c_void_p(Xc.data_ptr()), C.c_void_p(Y.data_ptr()), _lib.OPS[op],
                                       nrhs, _stream_ptr(stream)))
        return Y[0] if vec else Y.t()

    def apply_pair(self, x_far, x_near, out_near=None, out_far=None, stream=None):
        """(y_near, y_far) = (U W^T x_far, W U^T x_near): the two Eq. 15 products in one call."""
        torch = _torch()
        y_n = out_near if out_near is not None else torch.empty(x_near.shape[0], dtype=torch.complex128,
                                                                 device=x_near.device)
        y_f = out_far if out_far is not None else torch.empty(x_far.shape[0], dtype=torch.complex128,
                                                               device=x_far.device)
        self.apply_pair_raw(x_far.data_ptr(), y_n.data_ptr(), x_near.data_ptr(), y_f.data_ptr(), stream)
        return y_n, y_f

    def apply_pair_raw(self, xf_ptr: int, yn_ptr: int, xn_ptr: int, yf_ptr: int, stream=None):
        check(lib().vsie_farnear_apply_pair(self._h, C.c_void_p(xf_ptr), C.c_void_p(yn_ptr), C.c_void_p(xn_ptr),
                                            C.c_void_p(yf_ptr), _stream_ptr(stream)))


class FarFar:
    """Dense far-far block Z_cc^ff (include/vsie_farfar.h): symmetric, lower-triangle tiles."""

    def __init__(self, handle):
        self._h = _lib.HANDLE(handle)

    @classmethod
    def build(cls, far_meshes, freq: float, scale=1.0, device=-1):
        arr, keep = _meshes_c(far_meshes)
        h = _lib.HANDLE()
        check(lib().vsie_farfar_build(arr, len(far_meshes), float(freq), float(np.real(scale)), float(np.imag(scale)),
                                      int(device), C.byref(h)))
        del keep
        return cls(h.value)

    def close(self):
        if self._h is not None and self._h.value:
            lib().vsie_farfar_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def info(self) -> dict:
        i = _lib.vsie_farfar_info()
        check(lib().vsie_farfar_get_info(self._h, C.byref(i)))
        return dict(m=i.m, tile=i.tile, tiles=i.tiles, matrix_bytes=i.matrix_bytes, near_pairs=i.near_pairs,
                    build_s=i.build_s, k0=i.k0, apply_calls=i.apply_calls)

    def export(self):
        m = self.info()["m"]
        Z = np.empty((m, m), dtype=np.complex128, order="F")
        check(lib().vsie_farfar_export(self._h, Z.ctypes.data))
        return Z

    def entries(self, rows, cols, stream=None):
        torch = _torch()
        idx = torch.stack([torch.as_tensor(rows, dtype=torch.int64), torch.as_tensor(cols, dtype=torch.int64)],
                          dim=1).contiguous().cuda()
        out = torch.empty(idx.shape[0], dtype=torch.complex128, device=idx.device)
        check(lib().vsie_farfar_entries(self._h, C.c_void_p(idx.data_ptr()), idx.shape[0], C.c_void_p(out.data_ptr()),
                                        _stream_ptr(stream)))
        return out

    def apply(self, x, op: str = "N", out=None, accumulate=False, stream=None):
        torch = _torch()
        vec = x.dim() == 1
        X = x.reshape(-1, 1) if vec else x
        nrhs = X.shape[1]
        Xc = X.t().contiguous()
        if out is None:
            Y = torch.empty_like(Xc)
        else:
            Y = out.reshape(-1, 1).t() if vec else out.t()
        check(lib().vsie_farfar_apply(self._h, C.c_void_p(Xc.data_ptr()), C.c_void_p(Y.data_ptr()), _lib.OPS[op], nrhs,
                                      1 if accumulate else 0, _stream_ptr(stream)))
        return Y[0] if vec else Y.t()

    def apply_raw(self, x_ptr: int, y_ptr: int, op: str = "N", accumulate=False, stream=None):
        check(lib().vsie_farfar_apply(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), _lib.OPS[op], 1,
                                      1 if accumulate else 0, _stream_ptr(stream)))
