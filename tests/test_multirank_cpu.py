"""World-size-2 (gloo, CPU) tests of the N > 1 path's host logic:

* the slab partition the library uses (vsie_slab_partition) tiles the voxel
  planes and the G4 columns exactly, with equal padded column chunks;
* the design-(iii) decomposition — per-rank partial G4 products combined by an
  allreduce of 3 r3 values, per-rank slabs, partial z3 allreduce, allgather of
  the column segments of z — reproduces the single-process TT apply (oracle
  arithmetic per shard, collectives through torch.distributed/gloo);
* the NCCL unique id travels through torch.distributed.broadcast_object_list.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

WORLD = 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        import synth
        from oracle import ttmv
        from paper_2206_12409_b200 import slab_partition
        import sys
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        from gpu_common import rand_tts

        cfg = synth.get_config(1)
        n1, n2, n3 = cfg.n
        m = cfg.m
        (s0, s1), (c0, c1) = slab_partition(n3, m, world, rank)
        ranges = [None] * world
        dist.all_gather_object(ranges, ((s0, s1), (c0, c1)))
        tts = rand_tts(cfg, [(3, 5, 7), (2, 6, 4), (4, 3, 5)], 11)
        x = synth.complex_gaussian(m, 3)
        u = synth.complex_gaussian(3 * cfg.n_v, 4)
        r3max = max(t[3].shape[0] for t in tts)
        # ---- forward: partial y4 over the owned columns, allreduce, local planes
        y4 = np.zeros((3, r3max), complex)
        for chi, (G1, G2, G3, G4) in enumerate(tts):
            y4[chi, :G4.shape[0]] = G4[:, c0:c1, 0] @ x[c0:c1]
        t = torch.from_numpy(y4.view(np.float64).copy())
        dist.all_reduce(t)
        y4 = t.numpy().view(complex)
        yloc = []
        for chi, (G1, G2, G3, G4) in enumerate(tts):
            Y3 = np.einsum("bkc,c->bk", G3[:, s0:s1, :], y4[chi, :G4.shape[0]])
            Y2 = np.einsum("ajb,bk->ajk", G2, Y3)
            yloc.append(np.einsum("ia,ajk->ijk", G1[0], Y2).reshape(-1, order="F"))
        slabs = [None] * world
        dist.all_gather_object(slabs, (s0, yloc))
        # ---- transpose: local planes -> partial z3, allreduce, owned columns, allgather
        U = u.reshape(3, n1, n2, n3, order="C") if False else [u[c * cfg.n_v:(c + 1) * cfg.n_v].reshape((n1, n2, n3), order="F") for c in range(3)]
        z3 = np.zeros((3, r3max), complex)
        for chi, (G1, G2, G3, G4) in enumerate(tts):
            W1 = np.einsum("ia,ijk->ajk", G1[0], U[chi][:, :, s0:s1])
            W2 = np.einsum("ajb,ajk->bk", G2, W1)
            z3[chi, :G4.shape[0]] = np.einsum("bkc,bk->c", G3[:, s0:s1, :], W2)
        t = torch.from_numpy(z3.view(np.float64).copy())
        dist.all_reduce(t)
        z3 = t.numpy().view(complex)
        mp_ = -(-m // world)
        seg = np.zeros(mp_, complex)
        for chi, (G1, G2, G3, G4) in enumerate(tts):
            seg[:c1 - c0] += G4[:, c0:c1, 0].T @ z3[chi, :G4.shape[0]]
        recv = [torch.zeros(2 * mp_, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(recv, torch.from_numpy(seg.view(np.float64).copy()))
        z = np.concatenate([r.numpy().view(complex) for r in recv])[:m]
        # ---- unique-id broadcast (bytes through torch.distributed)
        obj = [b"\x07" * 128 if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        if rank == 0:
            yfull = [np.zeros(cfg.n_v, complex) for _ in range(3)]
            for (sb, parts) in slabs:
                for chi in range(3):
                    n12 = n1 * n2
                    k = len(parts[chi]) // n12
                    yfull[chi][n12 * sb:n12 * (sb + k)] = parts[chi]
            yref = ttmv.apply(tts, x, "N")
            zref = ttmv.apply(tts, u, "T")
            q.put(dict(ranges=ranges, yerr=float(np.linalg.norm(np.concatenate(yfull) - yref) / np.linalg.norm(yref)),
                       zerr=float(np.linalg.norm(z - zref) / np.linalg.norm(zref)), uid=obj[0]))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover
        q.put(dict(error=repr(e)))
        raise


def test_world2_slab_decomposition_gloo():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, WORLD, port, q)) for r in range(WORLD)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert "error" not in res, res
    (a0, a1), (b0, b1) = res["ranges"][0], res["ranges"][1]
    assert a0[0] == 0 and a0[1] == b0[0] and b0[1] == 12          # planes tile [0, n3)
    assert a1[0] == 0 and a1[1] == b1[0] and b1[1] == 1128        # columns tile [0, m)
    assert a1[1] - a1[0] == -(-1128 // 2)                          # equal padded chunks
    assert res["yerr"] < 1e-13 and res["zerr"] < 1e-13
    assert res["uid"] == b"\x07" * 128


@pytest.mark.parametrize("n3,m,world", [(12, 1128, 3), (110, 10080, 8), (400, 30000, 7), (8, 5, 8)])
def test_partition_tiles_exactly(n3, m, world):
    from paper_2206_12409_b200 import slab_partition
    planes, cols = [], []
    for r in range(world):
        (s0, s1), (c0, c1) = slab_partition(n3, m, world, r)
        planes.append((s0, s1))
        cols.append((c0, c1))
    assert planes[0][0] == 0 and planes[-1][1] == n3
    assert all(planes[i][1] == planes[i + 1][0] for i in range(world - 1))
    assert all(s1 > s0 for s0, s1 in planes)
    assert cols[0][0] == 0 and cols[-1][1] == m
    assert all(cols[i][1] == cols[i + 1][0] for i in range(world - 1))
    assert max(c1 - c0 for c0, c1 in cols) == -(-m // world)
