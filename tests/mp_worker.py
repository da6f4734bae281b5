"""Worker of tests/test_gpu_multiproc.py: one rank of a world-2 job whose two processes share
cuda:0 through the CUDA-IPC communicator (vsie_build_opts.ipc_name).  Every multi-process
branch of the library runs: the slab-sharded applies (y4 / z3 allreduces, z allgather), the
block applies, both pair schedules, the host-buffer pair and the TT-cross build with its
supercores split across the ranks.  Each rank compares its results with a world-1 handle
built in the same process (test infrastructure: uses oracle/ only through synth inputs).

    python tests/mp_worker.py <rank> <world> <ipc-name> <out.json>"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from gpu_common import grid_of, rand_tts  # noqa: E402
from paper_2206_12409_b200 import Coupling  # noqa: E402


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    rank, world, name, out = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3], sys.argv[4]
    torch.cuda.set_device(0)
    res = {"rank": rank}
    for ci in (1, 2):
        cfg = synth.get_config(ci)
        n1, n2, n3 = cfg.n
        r = cfg.ranks_probe
        tts = rand_tts(cfg, [r, (r[0] + 1, max(1, r[1] - 2), r[2] + 3), (max(1, r[0] - 1), r[1] + 1, r[2] - 4)],
                       600 + ci)
        h1 = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=4)
        hp = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, tts, nrhs_max=4, world=world, rank=rank,
                                 ipc_name=f"{name}_a{ci}")
        inf = hp.info()
        s0, s1 = inf["slab"]
        nv = cfg.n_v

        def slab(v):   # the rank's slab of a global voxel vector (chi-major, planes s0..s1)
            v = v.reshape((3, nv) + v.shape[1:])
            return np.ascontiguousarray(v[:, n1 * n2 * s0:n1 * n2 * s1].reshape((-1,) + v.shape[2:]))

        x = synth.complex_gaussian(cfg.m, 31)
        u = synth.complex_gaussian(3 * nv, 32)
        X = synth.complex_gaussian(cfg.m, 33, ncols=4)
        U = synth.complex_gaussian(3 * nv, 34, ncols=4)
        cu = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()
        e = {}
        y1 = h1.apply(cu(x), "N").cpu().numpy()
        e["N"] = rel(hp.apply(cu(x), "N").cpu().numpy(), slab(y1))
        for op in ("T", "C"):
            e[op] = rel(hp.apply(cu(slab(u)), op).cpu().numpy(), h1.apply(cu(u), op).cpu().numpy())
        Y1 = h1.apply(cu(X), "N").cpu().numpy()
        e["N_block"] = rel(hp.apply(cu(X), "N").cpu().numpy(), slab(Y1))
        e["T_block"] = rel(hp.apply(cu(slab(U)), "T").cpu().numpy(), h1.apply(cu(U), "T").cpu().numpy())
        z1 = h1.apply(cu(u), "T").cpu().numpy()
        for sched in ("g4_shared", "g3_shared"):
            hp.configure(pair_schedule=sched)
            yp, zp = hp.apply_pair(cu(x), cu(slab(u)), "T")
            e[f"pair_y_{sched}"] = rel(yp.cpu().numpy(), slab(y1))
            e[f"pair_z_{sched}"] = rel(zp.cpu().numpy(), z1)
        yh, zh = hp.apply_pair_host(x, slab(u), "C")
        e["pair_host_y"] = rel(yh, slab(y1))
        e["pair_host_z"] = rel(zh, h1.apply(cu(u), "C").cpu().numpy())
        res[f"cfg{ci}"] = e
        del hp, h1
    # TT-cross build with the supercore columns split over the ranks (cfg 1, tol 1e-8)
    cfg = synth.get_config(1)
    b1 = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
    bp = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1, world=world, rank=rank,
                        ipc_name=f"{name}_b")
    x = synth.complex_gaussian(cfg.m, 41)
    u = synth.complex_gaussian(3 * cfg.n_v, 42)
    s0, s1 = bp.info()["slab"]
    n12 = cfg.n[0] * cfg.n[1]
    us = np.ascontiguousarray(u.reshape(3, -1)[:, n12 * s0:n12 * s1].reshape(-1))
    y1 = b1.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy().reshape(3, -1)[:, n12 * s0:n12 * s1].reshape(-1)
    # diagnostics: the replicated cores G1 / G2 of both builds, and a digest of b1's cores
    c1 = b1.export_cores()
    try:
        cp = bp.export_cores()
        g12 = max(float(np.max(np.abs(c1[c][k] - cp[c][k]))) for c in range(3) for k in (0, 1))
    except Exception as ex:  # noqa: BLE001 (diagnostic only)
        g12 = str(ex)
    digest = float(sum(np.sum(np.abs(c1[c][k]) * (1 + np.arange(c1[c][k].size).reshape(c1[c][k].shape) % 7))
                       for c in range(3) for k in range(4)))
    res["build_diag"] = {"g12_diff": g12, "b1_digest": digest, "sweeps1": b1.info()["sweeps"],
                         "sweepsp": bp.info()["sweeps"], "held1": list(b1.info()["heldout_err"]),
                         "heldp": list(bp.info()["heldout_err"])}
    res["build"] = {"ranks_equal": bp.info()["ranks"] == b1.info()["ranks"],
                    "status": bp.status,
                    "N": rel(bp.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy(), y1),
                    "T": rel(bp.apply(torch.from_numpy(us).cuda(), "T").cpu().numpy(),
                             b1.apply(torch.from_numpy(u).cuda(), "T").cpu().numpy())}
    # cfg 2: the randomized range finder on row-split supercores (k = 2, 3: min dim > 384);
    # the sums over the ranks' row blocks round differently, so the TT is an equally valid
    # approximation, compared through its applies (both within ~1e-6 of Z)
    cfg = synth.get_config(2)
    b1 = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
    bp = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1, world=world, rank=rank,
                        ipc_name=f"{name}_c")
    x = synth.complex_gaussian(cfg.m, 43)
    s0, s1 = bp.info()["slab"]
    n12 = cfg.n[0] * cfg.n[1]
    y1 = b1.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy().reshape(3, -1)[:, n12 * s0:n12 * s1].reshape(-1)
    i1, ip = b1.info(), bp.info()
    res["build_rowsplit"] = {"status": bp.status, "heldout": list(ip["heldout_err"]),
                             "ranks1": i1["ranks"], "ranksp": ip["ranks"],
                             "N": rel(bp.apply(torch.from_numpy(x).cuda(), "N").cpu().numpy(), y1)}
    with open(out, "w") as f:
        json.dump(res, f)
    print("worker ok", rank)


if __name__ == "__main__":
    main()
