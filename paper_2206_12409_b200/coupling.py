"""Thin Python wrapper over the C ABI: ``Coupling`` = one Z_bc handle.

Every compute step runs inside libvsie_coupling.so; this module only converts
arguments (numpy / torch tensors -> pointers) and status codes -> exceptions.
PyTorch provides device memory and the current CUDA stream.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from fractions import Fraction

import numpy as np

from . import _lib
from ._lib import check, lib


@dataclass(frozen=True)
class Grid:
    n: tuple
    h: tuple
    origin: tuple

    def as_c(self):
        g = _lib.vsie_grid()
        for a in range(3):
            g.n[a] = int(self.n[a])
            g.h[a] = float(self.h[a])
            g.origin[a] = float(self.origin[a])
        return g


def _meshes_c(meshes):
    keep = []
    arr = (_lib.vsie_mesh * len(meshes))()
    for i, (xyz, tri) in enumerate(meshes):
        xyz = np.ascontiguousarray(xyz, dtype=np.float64)
        tri = np.ascontiguousarray(tri, dtype=np.int32)
        keep += [xyz, tri]
        arr[i].n_vertices = xyz.shape[0]
        arr[i].xyz = xyz.ctypes.data
        arr[i].n_triangles = tri.shape[0]
        arr[i].tri = tri.ctypes.data
    return arr, keep


def _opts(**kw):
    o = _lib.vsie_build_opts()
    lib().vsie_build_opts_default(C.byref(o))
    keep = None
    for k, v in kw.items():
        if v is None:
            continue
        if k == "scale":
            o.scale_re, o.scale_im = float(np.real(v)), float(np.imag(v))
        elif k == "nccl_unique_id":
            keep = C.create_string_buffer(bytes(v), 128)
            o.nccl_unique_id = C.cast(keep, C.c_void_p)
        elif k == "ipc_name":
            o.ipc_name = str(v).encode()
        else:
            setattr(o, k, v)
    return o, keep


def _torch():
    import torch
    return torch


def _stream_ptr(stream):
    torch = _torch()
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def slab_partition(n3: int, m: int, world: int, rank: int):
    """(i3 range, G4 column range) owned by `rank` (vsie_slab_partition, host only)."""
    sl = (C.c_int32 * 2)()
    cl = (C.c_int64 * 2)()
    check(lib().vsie_slab_partition(int(n3), int(m), int(world), int(rank), sl, cl))
    return (sl[0], sl[1]), (cl[0], cl[1])


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().vsie_nccl_unique_id(buf))
    return buf.raw


class Coupling:
    """A Z_bc handle (cores on device, slab partition, workspaces)."""

    def __init__(self, handle, status=0):
        self._h = _lib.HANDLE(handle)
        self.status = status

    # ------------------------------------------------------------------ construction
    @classmethod
    def build(cls, grid: Grid, meshes, freq: float, tol: float, **opts):
        """vsie_coupling_build: TT-cross over the entry kernel."""
        g = grid.as_c()
        arr, keep = _meshes_c(meshes)
        o, k2 = _opts(**opts)
        h = _lib.HANDLE()
        st = lib().vsie_coupling_build(C.byref(g), arr, len(meshes), float(freq), float(tol), C.byref(o), C.byref(h))
        check(st, allow_warn=True)
        del keep, k2
        return cls(h.value, st)

    @classmethod
    def from_cores(cls, grid: Grid, meshes, freq: float, cores, **opts):
        """vsie_coupling_import_cores; cores[chi][k] = array (r_{k-1}, n_k, r_k)."""
        g = grid.as_c()
        arr, keep = _meshes_c(meshes)
        o, k2 = _opts(**opts)
        ranks = (C.c_int32 * 9)()
        ptrs = (C.c_void_p * 12)()
        flat = []
        for chi in range(3):
            for k in range(3):
                ranks[3 * chi + k] = int(cores[chi][k].shape[2])
            for k in range(4):
                a = np.asarray(cores[chi][k], dtype=np.complex128).ravel(order="F")
                a = np.ascontiguousarray(a)
                flat.append(a)
                ptrs[4 * chi + k] = a.ctypes.data
        h = _lib.HANDLE()
        check(lib().vsie_coupling_import_cores(C.byref(g), arr, len(meshes), float(freq), ranks, ptrs, C.byref(o),
                                               C.byref(h)))
        del keep, k2, flat
        return cls(h.value)

    def close(self):
        if self._h is not None and self._h.value:
            lib().vsie_coupling_destroy(self._h)
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

    # ------------------------------------------------------------------ queries
    def info(self) -> dict:
        i = _lib.vsie_info()
        check(lib().vsie_coupling_info(self._h, C.byref(i)))
        return dict(
            n=tuple(i.n), m=i.m, ranks=[tuple(i.ranks[c]) for c in range(3)], core_bytes=i.core_bytes,
            compression=Fraction(i.compression_num, i.compression_den) if i.compression_den else None,
            entries_evaluated=i.entries_evaluated, sweeps=tuple(i.sweeps), heldout_err=tuple(i.heldout_err),
            build_s=i.build_s, build_entry_s=i.build_entry_s, build_factor_s=i.build_factor_s,
            build_maxvol_s=i.build_maxvol_s, slab=tuple(i.slab), cols=tuple(i.cols), world=i.world,
            rank=i.rank, loopback=i.loopback, k0=i.k0, apply_launches=i.apply_launches,
            apply_calls=i.apply_calls, test_moment=i.test_moment, quad_rule=i.quad_rule,
            pair_schedule={1: "g4_shared", 2: "g3_shared"}.get(i.pair_schedule))

    @property
    def m(self):
        return self.info()["m"]

    def export_cores(self):
        """[chi][k] numpy arrays (r_{k-1}, n_k, r_k) (column-major core layout, §8c-L16)."""
        inf = self.info()
        dims = list(inf["n"]) + [inf["m"]]
        out = []
        for chi in range(3):
            r = (1,) + tuple(inf["ranks"][chi]) + (1,)
            cs = []
            for k in range(4):
                ne = C.c_int64()
                buf = np.empty(r[k] * dims[k] * r[k + 1], dtype=np.complex128)
                check(lib().vsie_coupling_export_cores(self._h, chi, k, buf.ctypes.data, C.byref(ne)))
                assert ne.value == buf.size
                cs.append(buf.reshape((r[k], dims[k], r[k + 1]), order="F"))
            out.append(cs)
        return out

    def round(self, tol: float):
        """vsie_coupling_round: TT rounding of the cores in place.

        Returns the new ranks [chi][k]."""
        check(lib().vsie_coupling_round(self._h, float(tol)))
        return [tuple(r) for r in self.info()["ranks"]]

    # ------------------------------------------------------------------ compute
    def apply(self, x, op: str = "N", out=None, stream=None):
        """vsie_coupling_apply on device tensors (complex128, column-major RHS blocks).

        x: (len,) or (len, nrhs) CUDA complex128 tensor; column-major blocks are
        passed as the transpose of a contiguous (nrhs, len) tensor."""
        torch = _torch()
        inf_m = self.m
        vec = x.dim() == 1
        X = x.reshape(-1, 1) if vec else x
        nrhs = X.shape[1]
        Xc = X.t().contiguous()  # (nrhs, len): column-major (len, nrhs)
        n_out = self.out_len(op)
        if out is None:
            Y = torch.empty((nrhs, n_out), dtype=torch.complex128, device=x.device)
        else:
            Y = out.reshape(-1, 1).t() if vec else out.t()
            assert Y.is_contiguous()
        del inf_m
        check(lib().vsie_coupling_apply(self._h, C.c_void_p(Xc.data_ptr()), C.c_void_p(Y.data_ptr()), _lib.OPS[op],
                                        nrhs, _stream_ptr(stream)))
        return Y[0] if vec else Y.t()

    def apply_raw(self, x_ptr: int, y_ptr: int, op: str, nrhs: int, stream=None):
        check(lib().vsie_coupling_apply(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), _lib.OPS[op], nrhs,
                                        _stream_ptr(stream)))

    def apply_pair(self, x, u, adj: str = "T", out_y=None, out_z=None, stream=None):
        """vsie_coupling_apply_pair: (Z x, Z^T u) or (Z x, Z^H u) in one call (single RHS)."""
        torch = _torch()
        x = x.contiguous()
        u = u.contiguous()
        y = out_y if out_y is not None else torch.empty(self.out_len("N"), dtype=torch.complex128, device=x.device)
        z = out_z if out_z is not None else torch.empty(self.out_len("T"), dtype=torch.complex128, device=x.device)
        check(lib().vsie_coupling_apply_pair(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                             C.c_void_p(u.data_ptr()), C.c_void_p(z.data_ptr()), _lib.OPS[adj],
                                             _stream_ptr(stream)))
        return y, z

    def apply_pair_raw(self, x_ptr: int, y_ptr: int, u_ptr: int, z_ptr: int, adj: str = "T", stream=None):
        check(lib().vsie_coupling_apply_pair(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(u_ptr),
                                             C.c_void_p(z_ptr), _lib.OPS[adj], _stream_ptr(stream)))

    def apply_pair_host_raw(self, x_ptr: int, y_ptr: int, u_ptr: int, z_ptr: int, adj: str = "T"):
        check(lib().vsie_coupling_apply_pair_host(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(u_ptr),
                                                  C.c_void_p(z_ptr), _lib.OPS[adj]))

    def apply_pair_host(self, x: np.ndarray, u: np.ndarray, adj: str = "T"):
        """vsie_coupling_apply_pair_host: (y = Z x, z = Z^T u or Z^H u) with host buffers."""
        xc = np.ascontiguousarray(x, dtype=np.complex128)
        uc = np.ascontiguousarray(u, dtype=np.complex128)
        y = np.empty(self.out_len("N"), dtype=np.complex128)
        z = np.empty(self.out_len("T"), dtype=np.complex128)
        self.apply_pair_host_raw(xc.ctypes.data, y.ctypes.data, uc.ctypes.data, z.ctypes.data, adj)
        return y, z

    def apply_host(self, x: np.ndarray, op: str = "N") -> np.ndarray:
        """vsie_coupling_apply_host: host in, host out (H2D + apply + D2H)."""
        X = np.asarray(x, dtype=np.complex128)
        vec = X.ndim == 1
        X2 = X.reshape(-1, 1) if vec else X
        nrhs = X2.shape[1]
        Xf = np.asfortranarray(X2)
        Y = np.empty((self.out_len(op), nrhs), dtype=np.complex128, order="F")
        check(lib().vsie_coupling_apply_host(self._h, Xf.ctypes.data, Y.ctypes.data, _lib.OPS[op], nrhs))
        return Y[:, 0] if vec else Y

    def apply_host_raw(self, x_ptr: int, y_ptr: int, op: str, nrhs: int):
        check(lib().vsie_coupling_apply_host(self._h, C.c_void_p(x_ptr), C.c_void_p(y_ptr), _lib.OPS[op], nrhs))

    def out_len(self, op: str) -> int:
        inf = self.info()
        n1, n2, _ = inf["n"]
        vox = 3 * n1 * n2 * (inf["slab"][1] - inf["slab"][0]) if inf["world"] > 1 and not inf["loopback"] \
            else 3 * n1 * n2 * inf["n"][2]
        return vox if op == "N" else inf["m"]

    def _idx_call(self, fn, rows, cols, stream=None):
        torch = _torch()
        rows = torch.as_tensor(rows, dtype=torch.int64)
        cols = torch.as_tensor(cols, dtype=torch.int64)
        dev = rows.device if rows.is_cuda else torch.device("cuda")
        idx = torch.stack([rows.to(dev), cols.to(dev)], dim=1).contiguous()
        out = torch.empty(idx.shape[0], dtype=torch.complex128, device=dev)
        check(fn(self._h, C.c_void_p(idx.data_ptr()), idx.shape[0], C.c_void_p(out.data_ptr()), _stream_ptr(stream)))
        return out

    def entries(self, rows, cols, stream=None):
        """Exact quadrature entries Z[rows, cols] (vsie_coupling_entries)."""
        return self._idx_call(lib().vsie_coupling_entries, rows, cols, stream)

    def tt_eval(self, rows, cols, stream=None):
        """TT values at (rows, cols) (vsie_coupling_tt_eval)."""
        return self._idx_call(lib().vsie_coupling_tt_eval, rows, cols, stream)

    def supercore(self, chi: int, k: int, left=None, right=None, stream=None):
        """vsie_coupling_supercore: the cross's structured block M_k (column-major
        (n_left n_k) x (n_{k+1} n_right)) on the device.  left / right: int32 arrays of shape
        (n, 2) (see the header; None for k = 1 / k = 3)."""
        torch = _torch()
        inf = self.info()
        dims = list(inf["n"]) + [inf["m"]]
        dev = torch.device("cuda")
        def prep(a):
            if a is None:
                return torch.zeros((1, 2), dtype=torch.int32, device=dev)
            t = torch.as_tensor(a, dtype=torch.int32).reshape(-1, 2)
            return t.to(dev).contiguous()
        L, R = prep(left), prep(right)
        nl, nr = L.shape[0], R.shape[0]
        rows, cols = nl * dims[k - 1], dims[k] * nr
        out = torch.empty((cols, rows), dtype=torch.complex128, device=dev)   # column-major rows x cols
        check(lib().vsie_coupling_supercore(self._h, int(chi), int(k), C.c_void_p(L.data_ptr()), nl,
                                            C.c_void_p(R.data_ptr()), nr, C.c_void_p(out.data_ptr()),
                                            _stream_ptr(stream)))
        return out.t()

    # ------------------------------------------------------------------ timing
    def set_timing(self, enable):
        """0/False off, 1/True serialised per-kernel timing, 2 concurrent timeline (trace())."""
        check(lib().vsie_coupling_set_timing(self._h, int(enable)))

    PAIR_SCHEDULES = {"auto": 0, "g4_shared": 1, "g3_shared": 2}

    def configure(self, graphs=None, pair_schedule=None):
        """CUDA-graph replay and the schedule of apply_pair (None = keep): pair_schedule
        'auto' (the one moving fewer bytes), 'g4_shared' (G4 read once) or 'g3_shared'
        (G3 read once)."""
        g = -1 if graphs is None else int(bool(graphs))
        m = -1 if pair_schedule is None else self.PAIR_SCHEDULES[pair_schedule]
        check(lib().vsie_coupling_configure(self._h, g, m))

    def trace(self, max_records=4096):
        n = C.c_int32()
        arr = (_lib.vsie_trace * max_records)()
        check(lib().vsie_coupling_trace(self._h, arr, max_records, C.byref(n)))
        return [dict(name=arr[i].name.decode(), chi=arr[i].chi, call=arr[i].call, t0_ms=arr[i].t0_ms,
                     t1_ms=arr[i].t1_ms) for i in range(n.value)]

    def timers(self):
        n = C.c_int32()
        arr = (_lib.vsie_timer * 64)()
        check(lib().vsie_coupling_timers(self._h, arr, 64, C.byref(n)))
        return [dict(name=arr[i].name.decode(), launches=arr[i].launches, total_ms=arr[i].total_ms,
                     bytes_per_launch=arr[i].bytes_per_launch, flops_per_launch=arr[i].flops_per_launch)
                for i in range(min(n.value, 64))]


class PWLCoupling:
    """The PWL (q = 12) coupling: four Coupling handles built with test_moment
    l = 0..3 (PWC block and the three linear test moments), applied through
    vsie_coupling_apply_pwl.  Vectors on the voxel side stack the four 3 n_v blocks
    moment-major (include/vsie_coupling.h)."""

    def __init__(self, handles):
        assert len(handles) == 4
        self.handles = list(handles)

    @staticmethod
    def _per_moment(opts, nccl_unique_ids):
        # every moment handle of a multi-process group owns its own NCCL communicator, so
        # it needs its own unique id (rank 0 creates four and broadcasts them)
        if "nccl_unique_id" in opts and opts["nccl_unique_id"] is not None:
            raise ValueError("PWLCoupling: pass nccl_unique_ids=[four ids], one per moment handle")
        if nccl_unique_ids is None:
            return [dict(opts) for _ in range(4)]
        assert len(nccl_unique_ids) == 4
        return [dict(opts, nccl_unique_id=nccl_unique_ids[l]) for l in range(4)]

    @classmethod
    def build(cls, grid: Grid, meshes, freq: float, tol: float, nccl_unique_ids=None, **opts):
        per = cls._per_moment(opts, nccl_unique_ids)
        return cls([Coupling.build(grid, meshes, freq, tol, test_moment=l, **per[l]) for l in range(4)])

    @classmethod
    def from_cores(cls, grid: Grid, meshes, freq: float, cores4, nccl_unique_ids=None, **opts):
        """cores4[l][chi][k] as in Coupling.from_cores, one set per test moment."""
        per = cls._per_moment(opts, nccl_unique_ids)
        return cls([Coupling.from_cores(grid, meshes, freq, cores4[l], test_moment=l, **per[l]) for l in range(4)])

    def close(self):
        for h in self.handles:
            h.close()

    def round(self, tol: float):
        """vsie_coupling_round on each moment handle; returns the new ranks [l][chi][k]."""
        return [h.round(tol) for h in self.handles]

    def out_len(self, op: str) -> int:
        n = self.handles[0].out_len(op)
        return 4 * n if op == "N" else n

    def apply(self, x, op: str = "N", stream=None):
        """vsie_coupling_apply_pwl on device tensors (layouts as Coupling.apply)."""
        torch = _torch()
        vec = x.dim() == 1
        X = x.reshape(-1, 1) if vec else x
        nrhs = X.shape[1]
        n_out = self.out_len(op)
        if op == "N":
            Xc = X.t().contiguous()
        else:
            # moment-major blocks, each column-major (3 n_v, nrhs)
            nv = X.shape[0] // 4
            Xc = X.reshape(4, nv, nrhs).permute(0, 2, 1).contiguous()
        Y = torch.empty((nrhs, n_out), dtype=torch.complex128, device=x.device)
        hs = (_lib.HANDLE * 4)(*[h._h for h in self.handles])
        check(lib().vsie_coupling_apply_pwl(hs, C.c_void_p(Xc.data_ptr()), C.c_void_p(Y.data_ptr()),
                                            _lib.OPS[op], nrhs, _stream_ptr(stream)))
        if op == "N":
            nv = n_out // 4
            Y = Y.reshape(4, nrhs, nv).permute(0, 2, 1).reshape(n_out, nrhs) if nrhs > 1 else Y.t()
            return Y[:, 0] if vec else Y
        return Y[0] if vec else Y.t()

    def apply_pair(self, x, u, adj: str = "T", stream=None):
        """vsie_coupling_apply_pair_pwl: (Z_pwl x, Z_pwl^T u) or (.., Z_pwl^H u), single RHS."""
        torch = _torch()
        x = x.contiguous()
        u = u.contiguous()
        y = torch.empty(self.out_len("N"), dtype=torch.complex128, device=x.device)
        z = torch.empty(self.out_len("T"), dtype=torch.complex128, device=x.device)
        hs = (_lib.HANDLE * 4)(*[h._h for h in self.handles])
        check(lib().vsie_coupling_apply_pair_pwl(hs, C.c_void_p(x.data_ptr()), C.c_void_p(y.data_ptr()),
                                                 C.c_void_p(u.data_ptr()), C.c_void_p(z.data_ptr()), _lib.OPS[adj],
                                                 _stream_ptr(stream)))
        return y, z

    def apply_pair_raw(self, x_ptr: int, y_ptr: int, u_ptr: int, z_ptr: int, adj: str = "T", stream=None):
        hs = (_lib.HANDLE * 4)(*[h._h for h in self.handles])
        check(lib().vsie_coupling_apply_pair_pwl(hs, C.c_void_p(x_ptr), C.c_void_p(y_ptr), C.c_void_p(u_ptr),
                                                 C.c_void_p(z_ptr), _lib.OPS[adj], _stream_ptr(stream)))


_alloc_keep = []   # every hook ever installed stays callable: buffers are freed through the hook
                   # that allocated them, possibly after the hook was replaced


def use_torch_allocator(enable: bool = True):
    """Route the library's device allocations through PyTorch's caching allocator
    (vsie_set_allocator; SURVEY §8(b) allocator hook), or back to cudaMalloc / cudaFree.
    Marshalling only: the callbacks call torch.cuda.caching_allocator_alloc / _delete on the
    current device and stream."""
    if not enable:
        check(lib().vsie_set_allocator(_lib.ALLOC_FN(), _lib.FREE_FN(), None))
        return
    torch = _torch()

    def _alloc(nbytes):
        try:
            return torch.cuda.caching_allocator_alloc(int(nbytes))
        except RuntimeError:
            return None

    def _free(ptr):
        torch.cuda.caching_allocator_delete(ptr)

    set_allocator(_alloc, _free)


def set_allocator(alloc, free):
    """vsie_set_allocator with Python callables alloc(nbytes) -> device pointer (int) or None
    and free(pointer); both None restores cudaMalloc / cudaFree.  The callables are kept
    alive for the rest of the process."""
    if alloc is None and free is None:
        check(lib().vsie_set_allocator(_lib.ALLOC_FN(), _lib.FREE_FN(), None))
        return
    keep = (_lib.ALLOC_FN(lambda n, _c: alloc(n)), _lib.FREE_FN(lambda p, _c: free(p)))
    _alloc_keep.append(keep)
    check(lib().vsie_set_allocator(keep[0], keep[1], None))
