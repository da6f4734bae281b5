"""Benchmark of the Z_bc hot path (BASELINE.json metric):
  "Z_bc TT matvec+adjoint ms & HBM GB/s per GMRES step; Z_bc entries/sec (FP64)".

One step = one GMRES iteration's use of the block: a forward apply y = Z x
(Eq. 17) plus a transpose apply z = Z^T u (Eqs. 18-19) through the C
ABI, on TT cores built by vsie_coupling_build (TT-cross) for
BASELINE config 4 (head 1 mm: 200x240x220 voxels, shield + bore 39890 RWG, tol 1e-6),
the largest single-GPU configuration whose build fits the bench (config 3 / 5 use seeded
cores at the ranks of the recorded cfg 3 build).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

N > 1 runs under torchrun, one process per GPU: the voxel grid is slab-sharded
along i3 and G4 along its columns (SURVEY §8e design iii); partials are
combined with NCCL inside the library (strong scaling: fixed total work).
Rank 0 prints ONE JSON line.  --impl reference times the CPU oracle (NumPy) on
the host cores instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import synth  # noqa: E402

METRIC = "Z_bc TT matvec+adjoint ms & HBM GB/s per GMRES step; Z_bc entries/sec (FP64)"


def step_bytes_flops(n, m, ranks, k=1):
    """B_fwd = 16 [sum_chi (n1 r1 + r1 n2 r2 + r2 n3 r3 + r3 m) + k (m + 3 n_v)], B_adj = B_fwd;
    F = 8 k sum_chi (r3 m + r2 n3 r3 + r1 n2 r2 n3 + n_v r1) per direction (block: cores once, vectors x k)."""
    n1, n2, n3 = n
    nv = n1 * n2 * n3
    cores = sum(n1 * r1 + r1 * n2 * r2 + r2 * n3 * r3 + r3 * m for (r1, r2, r3) in ranks)
    b_fwd = 16 * (cores + k * (m + 3 * nv))
    f_fwd = 8 * k * sum(r3 * m + r2 * n3 * r3 + r1 * n2 * r2 * n3 + nv * r1 for (r1, r2, r3) in ranks)
    return 2 * b_fwd, 2 * f_fwd


def moved_bytes(n, m, ranks, schedule, k=1):
    """Bytes one GMRES pair step of the library must move through HBM with the schedule it
    runs: every core once per direction, except the core streamed once for
    both (G4 for schedule 'g4_shared', G3 for 'g3_shared'), plus x, y, u, z (the separate
    applies, schedule None, read every core twice).  Whole job: G3 / G4 / the voxel vectors
    are split over the ranks (G1 / G2, replicated, are < 0.5% of the bytes)."""
    n1, n2, n3 = n
    nv = n1 * n2 * n3
    g12 = sum(n1 * r1 + r1 * n2 * r2 for (r1, r2, r3) in ranks)
    g3 = sum(r2 * n3 * r3 for (r1, r2, r3) in ranks)
    g4 = sum(r3 * m for (r1, r2, r3) in ranks)
    reads = {"g4_shared": 2 * g3 + g4, "g3_shared": g3 + 2 * g4}.get(schedule, 2 * (g3 + g4))
    return 16 * (2 * g12 + reads + 2 * k * (m + 3 * nv))


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "200"],
                                      stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.p is not None:
            time.sleep(0.25)
            self.p.terminate()
            try:
                out, _ = self.p.communicate(timeout=5)
            except Exception:
                self.p.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], None, set()
        for l in getattr(self, "lines", []):
            f = [x.strip() for x in l.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for k, nm in enumerate(names):
                if f[3 + k].lower().startswith("active"):
                    reasons.add(nm)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


def cpu_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def oracle_step_rate(cfg, ranks, steps=2, seed=5):
    """The CPU oracle (oracle/ttmv.py, as it stands) timed on the host cores on the
    same workload: cores with the GPU build's ranks (matvec cost does not depend on the
    core values).  Large configs (n_v > 5e6) time chi 0 only (forward +
    transpose of one chi TT, constant-valued cores) and scale by 3 -- the three chi
    components are identical work -- to bound the sample to ~10-30 s."""
    from oracle import ttmv
    big = cfg.n_v > 5_000_000
    if big:
        dims = tuple(cfg.n) + (cfg.m,)
        rr = (1,) + tuple(ranks[0]) + (1,)
        tts = [[np.full((rr[k], dims[k], rr[k + 1]), 0.5 + 0.25j) / np.sqrt(rr[k]) for k in range(4)]]
        x = np.full(cfg.m, 1.0 + 0.5j)
        u = np.full(cfg.n_v, 0.5 - 1.0j)
        scale = 3.0
    else:
        sys.path.insert(0, os.path.join(ROOT, "tests"))
        from gpu_common import rand_tts
        tts = rand_tts(cfg, ranks, seed)
        x = synth.complex_gaussian(cfg.m, synth.SEEDS["x"])
        u = synth.complex_gaussian(3 * cfg.n_v, synth.SEEDS["u"])
        scale = 1.0
    ts = []
    for _ in range(steps):
        t0 = time.perf_counter()
        ttmv.apply(tts, x, "N")
        ttmv.apply(tts, u, "T")
        ts.append((time.perf_counter() - t0) * scale)
    return statistics.median(ts), ts


def oracle_entry_rate(cfg, count=20000):
    from oracle import entries as oent
    prob = oent.problem_from_config(cfg)
    idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), count, 777)
    t0 = time.perf_counter()
    oent.entries(prob, idx[:, 0], idx[:, 1])
    return count / (time.perf_counter() - t0)


def ranks_hint(cfg):
    """Ranks of the last GPU build of this config (committed under profiles/; the block
    workload cfg 5 has the geometry of cfg 3), else the probe ranks."""
    p = os.path.join(ROOT, "profiles", f"ranks_cfg{3 if cfg.idx == 5 else cfg.idx}.json")
    if os.path.exists(p):
        with open(p) as f:
            return [tuple(r) for r in json.load(f)["ranks"]]
    return [tuple(cfg.ranks_probe)] * 3


def workload_name(cfg, k):
    """The config.workload string of both arms (identical for the driver's ratio)."""
    return (f"cfg{cfg.idx} {cfg.name}: grid {cfg.n}, h {cfg.h[0]*1e3:.0f} mm, m={cfg.m} RWG "
            f"({' + '.join(f'{s.name} {s.n_az}x{s.n_ax}' for s in cfg.surfaces)}), "
            f"f=298.2 MHz, tol {cfg.tol}, nrhs {k}")


def run_reference(args):
    """--impl reference: the CPU oracle on the host cores (rank 0 only)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    cfg = synth.get_config(args.config)
    ranks = ranks_hint(cfg)
    B, F = step_bytes_flops(cfg.n, cfg.m, ranks)
    from threadpoolctl import threadpool_info
    for _ in range(max(0, min(args.warmup, 1))):
        oracle_step_rate(cfg, ranks, steps=1)
    t, ts = oracle_step_rate(cfg, ranks, steps=args.steps)
    cores = cpu_cores()
    blas = [d.get("num_threads") for d in threadpool_info()]
    val = B / t / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": "GB/s", "n_gpus": 0, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": workload_name(cfg, cfg.nrhs), "grid": list(cfg.n), "m": cfg.m, "tol": cfg.tol,
                   "ranks": ranks, "step": "TT forward + transpose apply (oracle/ttmv.py, NumPy einsum)"},
        "cpu_baseline": {"value": val, "unit": "GB/s", "cores": cores, "kind": "oracle",
                         "sample": f"{args.steps} full GMRES steps of cfg{cfg.idx} with random cores at the GPU ranks",
                         "blas_threads": blas},
        "e2e": {"value": val, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def device_cores(cfg, ranks, seed, dev, m=None):
    """Seeded random complex TT cores at the given ranks, drawn on the device (the core
    values do not change the matvec cost) and returned as host arrays."""
    import torch
    g = torch.Generator(device=dev)
    dims = tuple(cfg.n) + (cfg.m if m is None else m,)
    out = []
    for c in range(3):
        rr = (1,) + tuple(ranks[c]) + (1,)
        g.manual_seed(seed + 101 * c)
        cores = []
        for k in range(4):
            shp = (rr[k], dims[k], rr[k + 1])
            a = torch.randn(shp + (2,), generator=g, device=dev, dtype=torch.float64) / np.sqrt(2 * rr[k])
            cores.append(torch.view_as_complex(a).cpu().numpy())
        out.append(cores)
    return out


def device_gaussian(n, k, seed, dev):
    """(a + ib)/sqrt 2 complex Gaussian (n x k, column-major) drawn on the device with a
    seeded generator -- used for the block-RHS workload whose 30 GB voxel block is not
    built on the host (SURVEY §8d recipe, torch generator instead of PCG64)."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(seed)
    a = torch.randn((k, n, 2), generator=g, device=dev, dtype=torch.float64) / np.sqrt(2.0)
    return torch.view_as_complex(a).reshape(-1)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cores", default="auto", choices=["auto", "build", "random"],
                    help="build = TT-cross build (default for configs 1, 2, 4 on one GPU); random = seeded cores "
                         "at the ranks of the recorded build (configs 3, 5: the build takes minutes; all N > 1 runs)")
    ap.add_argument("--round", type=float, default=None, metavar="TOL",
                    help="TT-round the cores (vsie_coupling_round, SURVEY 8f NEXT-1) at TOL before timing "
                         "(single process only)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-farnear", action="store_true", help="skip the far-near ACA block sub-measurement")
    ap.add_argument("--no-gmres", action="store_true", help="skip the GMRES consumer sub-measurement")
    ap.add_argument("--no-paper-setting", action="store_true",
                    help="skip the paper-setting build (tol 1e-3, 1 x 1 quadrature) sub-measurement")
    ap.add_argument("--separate", action="store_true",
                    help="time the step as two vsie_coupling_apply calls instead of vsie_coupling_apply_pair")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2206_12409_b200 import Coupling, grid_of, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    assert world == args.gpus or world == 1, "launch N > 1 with torchrun --nproc-per-node N"
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    uid = None
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        uid = obj[0]
    cfg = synth.get_config(args.config)
    k = cfg.nrhs
    # auto: the TT-cross build on one GPU (configs 1, 2, 4); seeded cores at the recorded
    # build ranks for configs 3 / 5 (their builds take minutes) and for every multi-GPU run
    # (the metric is the apply step; the multi-rank build is timed separately, not here)
    mode = args.cores if args.cores != "auto" else ("build" if cfg.idx in (1, 2, 4) and world == 1 else "random")
    t0 = time.perf_counter()
    if mode == "build":
        h = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=k, rank=rank, world=world,
                           nccl_unique_id=uid, device=local)
    else:
        ranks0 = ranks_hint(cfg)
        h = Coupling.from_cores(grid_of(cfg), cfg.meshes(), cfg.freq, device_cores(cfg, ranks0, 7, dev), nrhs_max=k,
                                rank=rank, world=world, nccl_unique_id=uid, device=local)
    build_s = time.perf_counter() - t0
    round_info = None
    if args.round is not None:
        assert world == 1, "--round needs a single-process handle"
        r_before = h.info()["ranks"]
        t1 = time.perf_counter()
        h.round(args.round)
        round_info = {"tol": args.round, "ranks_before": r_before, "round_s": time.perf_counter() - t1}
    inf = h.info()
    ranks = inf["ranks"]
    if rank == 0:
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    B, F = step_bytes_flops(cfg.n, cfg.m, ranks, k)
    n1, n2, n3 = cfg.n
    n3loc = inf["slab"][1] - inf["slab"][0]
    vox_loc = 3 * n1 * n2 * n3loc
    if k == 1:
        x = torch.from_numpy(synth.complex_gaussian(cfg.m, synth.SEEDS["x"])).to(dev)
        u_full = synth.complex_gaussian(3 * cfg.n_v, synth.SEEDS["u"]).reshape(3, -1)
        u_np = np.ascontiguousarray(u_full[:, n1 * n2 * inf["slab"][0]:n1 * n2 * inf["slab"][1]].reshape(-1))
        u = torch.from_numpy(u_np).to(dev)
    else:
        x = device_gaussian(cfg.m, k, synth.SEEDS["X"], dev)
        u = device_gaussian(vox_loc, k, synth.SEEDS["U"], dev)
        u_np = None
    y = torch.empty(vox_loc * k, dtype=torch.complex128, device=dev)
    z = torch.empty(cfg.m * k, dtype=torch.complex128, device=dev)
    flush = torch.empty(512 * 2 ** 20, dtype=torch.uint8, device=dev)   # > 126 MB L2
    stream = torch.cuda.current_stream()

    def step_separate():
        h.apply_raw(x.data_ptr(), y.data_ptr(), "N", k, stream)
        h.apply_raw(u.data_ptr(), z.data_ptr(), "T", k, stream)

    def step_pair():
        # one GMRES coupling matvec: y = Z x and z = Z^T u in one call (G4 streamed once)
        h.apply_pair_raw(x.data_ptr(), y.data_ptr(), u.data_ptr(), z.data_ptr(), "T", stream)

    use_pair = k == 1 and not args.separate
    step = step_pair if use_pair else step_separate

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        # keep the GPU under the same load for >= 0.6 s so that the 200 ms clock
        # samples see it (untimed), then the timed region
        t_end = time.perf_counter() + 0.6
        while time.perf_counter() < t_end:
            for _ in range(20 if k == 1 else 1):
                flush.fill_(1)
                step()
            torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        launches0 = h.info()["apply_launches"]
        for i in range(args.steps):
            flush.fill_(i & 0xFF)                     # evict L2 between timed steps
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    launches = h.info()["apply_launches"] - launches0
    per = [a.elapsed_time(b) for a, b in ev]
    ms = float(np.mean(per))
    sep_ms = None
    if use_pair:
        # the same step as two separate applies (context for the fused pair)
        for _ in range(3):
            step_separate()
        ev2 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev2[i][0].record(stream)
            step_separate()
            ev2[i][1].record(stream)
        torch.cuda.synchronize()
        sep_ms = float(np.mean([a.elapsed_time(b) for a, b in ev2]))
    # per-kernel CUDA-event timing: a second pass of the same K steps (same stream,
    # same inputs, L2 flushed) directly after the timed region, so the headline is
    # not perturbed by the event records between kernels
    h.set_timing(True)
    for i in range(args.steps):
        flush.fill_(i & 0xFF)
        step()
    torch.cuda.synchronize()
    timers = h.timers()
    h.set_timing(False)
    if world > 1:
        tt = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    value = B / (ms * 1e-3) / 1e9
    sched = inf.get("pair_schedule") if use_pair else None
    moved = moved_bytes(cfg.n, cfg.m, ranks, sched, k)

    # ---- end to end: host buffers through the C ABI (H2D + apply + D2H inside)
    e2e = None
    if vox_loc * k * 16 <= (4 << 30):
        xh = (torch.from_numpy(synth.complex_gaussian(cfg.m, synth.SEEDS["x"])) if k == 1 else x.cpu()).pin_memory()
        uh = (torch.from_numpy(u_np) if k == 1 else u.cpu()).pin_memory()
        yh = torch.empty(vox_loc * k, dtype=torch.complex128).pin_memory()
        zh = torch.empty(cfg.m * k, dtype=torch.complex128).pin_memory()
        def host_step():
            if use_pair:
                h.apply_pair_host_raw(xh.data_ptr(), yh.data_ptr(), uh.data_ptr(), zh.data_ptr(), "T")
            else:
                h.apply_host_raw(xh.data_ptr(), yh.data_ptr(), "N", k)
                h.apply_host_raw(uh.data_ptr(), zh.data_ptr(), "T", k)

        for _ in range(2):
            host_step()
        tl = []
        for _ in range(max(3, min(args.steps, 20))):
            if world > 1:
                dist.barrier()
            t1 = time.perf_counter()
            host_step()
            tl.append(time.perf_counter() - t1)
        e2e_s = float(np.mean(tl))
        if world > 1:
            tt = torch.tensor([e2e_s], device=dev, dtype=torch.float64)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        h2d = 16 * (cfg.m + vox_loc) * k
        e2e = {"value": B / e2e_s / 1e9, "unit": "GB/s", "ms_per_step": e2e_s * 1e3,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": h2d}
    else:
        e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": 16 * (cfg.m + vox_loc) * k,
               "d2h_bytes_per_step": 16 * (cfg.m + vox_loc) * k,
               "note": "not run: the pinned host copies of this block workload exceed 4 GiB"}

    # ---- entries/s (FP64): 1e6 uniform random (row, col) through vsie_coupling_entries
    ne = 1_000_000
    idx = synth.uniform_indices((3 * cfg.n_v, cfg.m), ne, 424242)
    rows_t = torch.from_numpy(idx[:, 0]).to(dev)
    cols_t = torch.from_numpy(idx[:, 1]).to(dev)
    h.entries(rows_t, cols_t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        h.entries(rows_t, cols_t)
    e1.record()
    torch.cuda.synchronize()
    ent_s = ne * 5 / (e0.elapsed_time(e1) * 1e-3)
    # block mode (the TT-cross's structured supercores): a k = 2 block of 16 x 64 index sets
    brng = np.random.default_rng(5)
    bl = np.stack([brng.integers(0, cfg.n[0], 16), np.zeros(16, int)], axis=1)
    br = np.stack([brng.integers(0, cfg.m, 64), np.zeros(64, int)], axis=1)
    Mb = h.supercore(1, 2, bl, br)
    nblk = Mb.numel()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3):
        Mb = None                     # the caching allocator reuses the block (no cudaMalloc timed)
        Mb = h.supercore(1, 2, bl, br)
    e1.record()
    torch.cuda.synchronize()
    blk_s = 3 * nblk / (e0.elapsed_time(e1) * 1e-3)
    del Mb

    if world > 1:
        dist.barrier()
    if rank != 0:
        dist.destroy_process_group()
        return 0

    # ---- far-near block: device ACA of Z_cc^fn against the synthetic near
    # coil, then the Eq. 15 pair y_n = U W^T j_f, y_f = W U^T j_n (two launches), L2 flushed
    farnear = None
    gm = None
    if not args.no_farnear:
        from paper_2206_12409_b200 import FarFar, FarNear
        tol_fn = 1e-3   # the hybrid method's ACA tolerance
        fn = FarNear.build([synth.near_mesh(cfg.idx)], cfg.meshes(), cfg.freq, tol_fn)
        fi = fn.info()
        xf = device_gaussian(fi["m_far"], 1, 7101, dev)
        xn = device_gaussian(fi["m_near"], 1, 7102, dev)
        yn = torch.empty_like(xn)
        yf = torch.empty_like(xf)
        for _ in range(3):
            fn.apply_pair_raw(xf.data_ptr(), yn.data_ptr(), xn.data_ptr(), yf.data_ptr())
        ts = []
        for i in range(20):
            flush.fill_(i & 255)
            e0.record()
            fn.apply_pair_raw(xf.data_ptr(), yn.data_ptr(), xn.data_ptr(), yf.data_ptr())
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        fms = float(np.median(ts))
        fbytes = 2 * fi["factor_bytes"] + 32 * (fi["m_far"] + fi["m_near"])
        # dense far-far block Z_cc^ff: symmetric lower-triangle tiles, one read per apply
        ff = FarFar.build(cfg.meshes(), cfg.freq)
        ffi = ff.info()
        for _ in range(3):
            ff.apply_raw(xf.data_ptr(), yf.data_ptr())
        ts2 = []
        for i in range(20):
            flush.fill_(i & 255)
            e0.record()
            ff.apply_raw(xf.data_ptr(), yf.data_ptr())
            e1.record()
            torch.cuda.synchronize()
            ts2.append(e0.elapsed_time(e1))
        ffms = float(np.median(ts2))
        # ---- GMRES consumer (include/vsie_hybrid.h): the Eq. 15 system with
        # this handle as Z_cb^f, the two blocks above, Z_cc^nn on the near coil, a near coupling
        # TT (seeded cores at this handle's ranks) and the PWC body diagonal h1 h2 h3 eps_r of the
        # synthetic phantom; restarted GMRES(50) for a fixed 60 iterations (tol out of reach)
        gm = None
        cbn = None
        if world == 1 and k == 1 and not args.no_gmres:
            from paper_2206_12409_b200 import Hybrid, VsieError
            near = [synth.near_mesh(cfg.idx)]
            try:
                cbn = Coupling.from_cores(grid_of(cfg), near, cfg.freq,
                                          device_cores(cfg, ranks, 8, dev, m=fi["m_near"]), nrhs_max=1)
            except VsieError as ex:   # the near coil too close to this grid for the coupling's rule
                gm = {"skipped": f"near coupling not buildable on this grid: {ex}"}
        if cbn is not None:
            nn = FarFar.build(near, cfg.freq)
            eps = synth.phantom_eps(cfg.n, cfg.h, cfg.origin, cfg.freq)
            d_b = torch.from_numpy(np.tile(cfg.h[0] * cfg.h[1] * cfg.h[2] * eps, 3)).to(dev)
            hy = Hybrid(ff, h, d_b, fn=fn, nn=nn, cb_near=cbn)
            hn = hy.info()["n"]
            bvec = torch.zeros(hn, dtype=torch.complex128, device=dev)
            bvec[: fi["m_far"]] = device_gaussian(fi["m_far"], 1, 7103, dev)
            hy.gmres(bvec, restart=50, max_iter=3, tol=1e-30)            # warm-up (graph captures)
            xg, gi, ghist = hy.gmres(bvec, restart=50, max_iter=60, tol=1e-30)
            mv0 = hy.info()["matvecs"]
            t_mv = []
            for i in range(5):
                flush.fill_(i & 255)
                e0.record()
                hy.matvec(bvec, out=xg)
                e1.record()
                torch.cuda.synchronize()
                t_mv.append(e0.elapsed_time(e1))
            gm = {"n": hn, "m_far": fi["m_far"], "m_near": fi["m_near"], "n_body": 3 * cfg.n_v,
                  "restart": 50, "iterations": gi["iterations"], "restarts": gi["restarts"],
                  "rel_residual_after": gi["rel_residual"], "solve_s": gi["seconds"],
                  "ms_per_iteration": 1e3 * gi["seconds"] / gi["iterations"],
                  "matvec_share": gi["matvec_seconds"] / gi["seconds"],
                  "matvec_ms": float(np.median(t_mv)), "matvecs_counted": mv0,
                  "krylov_basis_gb": 16 * hn * 51 / 1e9,
                  "note": ("Eq. 15 operator: Z_cc^ff + ACA (tol 1e-3) + Z_cc^nn + the TT coupling pair of "
                           "this handle + a near TT pair (seeded cores) + body diagonal; Z_bb's nonlocal "
                           "FFT part and pFFT are out of scope (DESIGN.md R-G1); 60 iterations of "
                           "GMRES(50) incl. one restart, host wall time; matvec_ms: staged matvec, "
                           "median of 5, L2 flushed")}
            hy.close()
            nn.close()
            cbn.close()
        ff.close()
        farnear = {"m_near": fi["m_near"], "m_far": fi["m_far"], "aca_tol": tol_fn, "rank": fi["rank"],
                   "stop": fi["stop"], "aca_est_err": fi["est_err"], "build_s": fi["build_s"],
                   "aca_entries": fi["entries_evaluated"], "pair_ms": fms, "pair_bytes": fbytes,
                   "pair_gbs": fbytes / (fms * 1e-3) / 1e9,
                   "pair_frac": fbytes / (fms * 1e-3) / 1e9 / load_peaks()[0],
                   "note": ("near surface = synthetic open cylinder (synth.NEAR_COILS); pair = both Eq. 15 "
                            "products, each factor read twice (dot + expand), median of 20, L2 flushed"),
                   "farfar": {"m": ffi["m"], "build_s": ffi["build_s"], "matrix_bytes": ffi["matrix_bytes"],
                              "near_pairs": ffi["near_pairs"], "apply_ms": ffms,
                              "apply_gbs": ffi["matrix_bytes"] / (ffms * 1e-3) / 1e9,
                              "apply_frac": ffi["matrix_bytes"] / (ffms * 1e-3) / 1e9 / load_peaks()[0],
                              "dense_equivalent_gbs": 16 * ffi["m"] ** 2 / (ffms * 1e-3) / 1e9,
                              "note": "Z_cc^ff y = Z x from the symmetric half (128 x 128 lower tiles, read once)"}}
        fn.close()

    # ---- the paper's own setting: TT-cross tol 1e-3 on the 1 x 1 far rule (quad_rule 1):
    # build time, ranks, held-out error, and the GMRES coupling pair on those cores (L2 flushed)
    paper = None
    if world == 1 and k == 1 and not args.no_paper_setting:
        t1 = time.perf_counter()
        hp = Coupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, 1e-3, nrhs_max=1, quad_rule=1)
        pb = time.perf_counter() - t1
        pi = hp.info()
        for _ in range(3):
            hp.apply_pair(x, u, "T", out_y=y, out_z=z)
        tp = []
        for i in range(20):
            flush.fill_(i & 255)
            e0.record()
            hp.apply_pair(x, u, "T", out_y=y, out_z=z)
            e1.record()
            torch.cuda.synchronize()
            tp.append(e0.elapsed_time(e1))
        pms = float(np.median(tp))
        pbytes = moved_bytes(cfg.n, cfg.m, pi["ranks"], pi["pair_schedule"])
        paper = {"tol": 1e-3, "quad_rule": 1, "ranks": pi["ranks"], "build_s": pb, "heldout_err": pi["heldout_err"],
                 "pair_ms": pms, "pair_moved_gbs": pbytes / (pms * 1e-3) / 1e9,
                 "note": "P:287: TT-cross tolerance 1e-3, 1 volume x 1 surface integration point for Z_bc^f"}
        hp.close()

    # ---- FP64 roofline of the entry kernel: measured FP64 instructions per entry x entries/s
    # over the measured DFMA issue rate (one FP64-pipe thread instruction per FMA)
    fp64_ops = None
    ep = os.path.join(ROOT, "profiles", "r02", "ncu_entries.json")
    if os.path.exists(ep):
        with open(ep) as f:
            fp64_ops = float(json.load(f)["captures"][0]["fp64_ops_per_entry"])
    with open(os.path.join(ROOT, "profiles", "r01", "fp64_peaks.json")) as f:
        fp64_peak_ops = float(json.load(f)["dfma_tflops"]) * 1e12 / 2.0

    # ---- roofline of the dominant kernel (largest share of the step)
    peak, peak_kind = load_peaks()
    kern = [t for t in timers if t["bytes_per_launch"] > 0 and t["launches"] > 0]
    dom = max(kern, key=lambda t: t["total_ms"]) if kern else None
    roof = None
    with open(os.path.join(ROOT, "profiles", "r01", "fp64_peaks.json")) as f:
        dmma_peak = float(json.load(f)["dmma_f64_tflops"])
    if dom:
        avg_ms = dom["total_ms"] / dom["launches"]
        ach = dom["bytes_per_launch"] / (avg_ms * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            with open(tp) as f:
                traffic = json.load(f).get(f"cfg{cfg.idx}", {}).get(dom["name"])
        roof = {"bound": "hbm", "kernel": dom["name"], "achieved": ach, "peak": peak, "unit": "GB/s",
                "frac": ach / peak, "traffic": traffic, "peak_source": peak_kind,
                "share_of_step": dom["total_ms"] / max(1e-9, sum(t["total_ms"] for t in timers)),
                "bytes_per_launch": dom["bytes_per_launch"], "avg_us": avg_ms * 1e3,
                "step_frac": moved / (ms * 1e-3) / 1e9 / peak,
                "step_frac_basis": "bytes the step's schedule moves (moved_bytes_per_step) / time / peak",
                "step_frac_formula": value / peak}
        ai = dom.get("flops_per_launch", 0) / max(1, dom["bytes_per_launch"])
        if dom.get("flops_per_launch"):
            # the G1 / G2 steps stream HBM and issue FP64 tensor work from the same warps: report the
            # FP64 side too (nominal 8 flop per complex multiply-add against the measured DMMA rate;
            # the 3M form issues 6 of them, plus K padding -- DESIGN.md §7)
            tf0 = dom["flops_per_launch"] / (avg_ms * 1e-3) / 1e12
            roof["co_bound"] = {"fp64_tflops": tf0, "fp64_peak_tflops": dmma_peak, "fp64_frac": tf0 / dmma_peak,
                                "hbm_frac": ach / peak, "flop_per_byte": ai,
                                "ridge_flop_per_byte": dmma_peak * 1e12 / (peak * 1e9)}
        if k > 1 or ai > dmma_peak * 1e12 / (peak * 1e9):
            # above the FP64 ridge (block RHS, SURVEY §8d AI ~ 15; the G2 contractions, AI ~ 20):
            # a tensor-core bound kernel, against the DMMA rate measured on this pool
            # (tools/microbench/fp64_peaks.cu -> profiles/r01/fp64_peaks.json)
            dmma = dmma_peak
            tf = dom["flops_per_launch"] / (avg_ms * 1e-3) / 1e12
            roof.update({"bound": "tensor", "achieved": tf, "peak": dmma, "unit": "TFLOP/s", "frac": tf / dmma,
                         "peak_source": "measured FP64 DMMA (profiles/r01/fp64_peaks.json)",
                         "flops_per_launch": dom["flops_per_launch"],
                         "step_frac": (F / (ms * 1e-3) / 1e12 / dmma) if k > 1 else moved / (ms * 1e-3) / 1e9 / peak})
    kern_table = {t["name"]: {"avg_us": 1e3 * t["total_ms"] / max(1, t["launches"]),
                              "launches_per_step": t["launches"] / max(1, args.steps),
                              "gbs": (t["bytes_per_launch"] / (t["total_ms"] / t["launches"] * 1e-3) / 1e9)
                              if t["bytes_per_launch"] else None,
                              "tflops": (t["flops_per_launch"] / (t["total_ms"] / t["launches"] * 1e-3) / 1e12)
                              if t.get("flops_per_launch") else None} for t in timers}
    cpu = None
    if not args.no_cpu_baseline and world == 1:
        # a bounded sample of ~10 s of host work: as many oracle steps as fit (>= 1)
        t1, _ = oracle_step_rate(cfg, ranks, steps=1)
        nsteps = int(max(1, min(50, 10.0 / max(t1, 1e-3))))
        t_cpu, ts = oracle_step_rate(cfg, ranks, steps=nsteps) if nsteps > 1 else (t1, [t1])
        B1, _ = step_bytes_flops(cfg.n, cfg.m, ranks, 1)
        cpu = {"value": B1 / t_cpu / 1e9, "unit": "GB/s", "cores": cpu_cores(), "kind": "oracle",
               "steps_timed": len(ts),
               "sample": (f"{len(ts) + 1} single-RHS GMRES step(s) (oracle TT fwd + transpose, NumPy) of the same cfg and ranks"
                          + (", chi 0 timed and x3" if cfg.n_v > 5_000_000 else ", random cores")
                          + (" (per RHS column of the block workload)" if k > 1 else "")),
               "ms_per_step": t_cpu * 1e3, "entries_per_s": oracle_entry_rate(cfg)}
    line = {
        "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "c128", "data": "synthetic",
        "config": {"workload": workload_name(cfg, k),
                   "step": (f"1 forward (y = Z x) + 1 transpose (z = Z^T u) TT apply as ONE vsie_coupling_apply_pair "
                            f"call (the coupling pair of a GMRES matvec; one large core streamed once for both)"
                            if use_pair else f"1 forward (Y = Z X) + 1 transpose (Z^T U) TT apply, {k} RHS"),
                   "bytes_per_step_note": ("value = SURVEY 8d formula bytes (B_fwd + B_adj: every core counted in both "
                                           "directions) / time, the normalised metric both arms report; the HBM "
                                           "bytes the step actually moves are moved_bytes_per_step (one large core "
                                           "streamed once for both directions), moved_gbs = those / time"),
                   "pair_schedule": sched,
                   "moved_bytes_per_step": moved,
                   "moved_gbs": moved / (ms * 1e-3) / 1e9,
                   "separate_applies": ({"ms_per_step": sep_ms, "gbs": B / (sep_ms * 1e-3) / 1e9} if sep_ms else None),
                   "cores": ("TT-cross build on this GPU" if mode == "build"
                             else "seeded random cores at the ranks of the recorded B200 build (profiles/)"),
                   "ranks": ranks,
                   "rounded": round_info,
                   "parallelism": f"slab{world} (i3 planes + G4 columns, NCCL)" if world > 1 else "1 GPU",
                   "l2": "flushed between timed steps (512 MiB write)",
                   "bytes_per_step": B, "flops_per_step": F, "build_s": build_s,
                   "build_breakdown_s": {"entries": inf["build_entry_s"], "factor": inf["build_factor_s"],
                                         "maxvol": inf["build_maxvol_s"]} if mode == "build" else None,
                   "heldout_err": inf["heldout_err"] if mode == "build" else None,
                   "sweeps": inf["sweeps"] if mode == "build" else None,
                   "compression": float(inf["compression"]) if inf["compression"] else None},
        "entries": {"value": ent_s, "unit": "entries/s", "pair_interactions_per_s": 48 * ent_s,
                    "sample": "1e6 uniform random (row, col), 5 reps",
                    "block_entries_per_s": blk_s,
                    "block_sample": "k = 2 supercore, 16 x 64 index sets (vsie_coupling_supercore), 3 reps",
                    "fp64_ops_per_entry": fp64_ops,
                    "fp64_ops_source": "ncu DFMA + DMUL + DADD thread instructions per entry (profiles/r02/ncu_entries.json)",
                    "fp64_peak_ops_per_s": fp64_peak_ops,
                    "fp64_peak_source": "measured DFMA rate / 2 (profiles/r01/fp64_peaks.json, tools/microbench/fp64_peaks.cu)",
                    "fp64_frac": ent_s * fp64_ops / fp64_peak_ops if fp64_ops else None,
                    "fp64_frac_block": blk_s * fp64_ops / fp64_peak_ops if fp64_ops else None,
                    "structured_blocks_per_s": (inf["entries_evaluated"] / inf["build_entry_s"])
                    if mode == "build" and inf["build_entry_s"] > 0 else None,
                    "structured_note": "supercore blocks evaluated by the TT-cross build (entries / entry-kernel time)"},
        "roofline": roof,
        "farnear": farnear,
        "gmres": gm if not args.no_farnear else None,
        "paper_setting": paper,
        "kernels": kern_table,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(launches),
        "gpu_launches_note": "kernel launches of this library inside the K timed steps (count from the library's launch counter; includes split-K sum kernels)",
        "clocks": clk.summary(),
    }
    print(json.dumps(line))
    with open(os.path.join(ROOT, "gpurun_out", f"bench_cfg{cfg.idx}_n{world}.json"), "w") as f:
        json.dump(line, f, indent=1)
    if mode == "build":
        with open(os.path.join(ROOT, "gpurun_out", f"ranks_cfg{cfg.idx}.json"), "w") as f:
            json.dump({"ranks": ranks, "source": "vsie_coupling_build on B200"}, f)
    if world > 1:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
