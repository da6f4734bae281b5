"""Time the PWL (q = 12) GMRES coupling pair (vsie_coupling_apply_pair_pwl) on one GPU.

Builds the four moment handles by TT-cross (config 2 by default), then times K steps of
y = Z_pwl x, z = Z_pwl^T u with CUDA events on the launching stream, L2 flushed between
steps, and reports GB/s by the SURVEY §8d byte formula summed over the four handles'
ranks (one JSON line)."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--round", type=float, default=None, metavar="TOL",
                    help="TT-round each moment handle (vsie_coupling_round) at TOL before timing")
    args = ap.parse_args()
    import torch
    import synth
    from bench import step_bytes_flops
    from paper_2206_12409_b200 import PWLCoupling, grid_of
    cfg = synth.get_config(args.config)
    t0 = time.perf_counter()
    P = PWLCoupling.build(grid_of(cfg), cfg.meshes(), cfg.freq, cfg.tol, nrhs_max=1)
    build_s = time.perf_counter() - t0
    ranks_before = None
    if args.round is not None:
        ranks_before = [h.info()["ranks"] for h in P.handles]
        P.round(args.round)
    infos = [h.info() for h in P.handles]
    B = sum(step_bytes_flops(cfg.n, cfg.m, inf["ranks"], 1)[0] for inf in infos)
    dev = torch.device("cuda")
    x = torch.from_numpy(synth.complex_gaussian(cfg.m, 9100)).to(dev)
    u = torch.from_numpy(synth.complex_gaussian(4 * 3 * cfg.n_v, 9101)).to(dev)
    y = torch.empty(4 * 3 * cfg.n_v, dtype=torch.complex128, device=dev)
    z = torch.empty(cfg.m, dtype=torch.complex128, device=dev)
    flush = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        for i in range(args.steps):
            flush.fill_(i & 0xFF)
            ev[i][0].record(st)
            fn()
            ev[i][1].record(st)
        torch.cuda.synchronize()
        return float(np.mean([a.elapsed_time(b) for a, b in ev]))

    ms_pair = timed(lambda: P.apply_pair_raw(x.data_ptr(), y.data_ptr(), u.data_ptr(), z.data_ptr(), "T", st))

    def sep():
        P.apply(x, "N", stream=st)
        P.apply(u, "T", stream=st)

    ms_sep = timed(sep)
    print(json.dumps({
        "metric": "PWL (q = 12) Z_bc TT GMRES coupling pair, HBM GB/s (SURVEY 8d bytes over 4 moment TTs)",
        "value": B / (ms_pair * 1e-3) / 1e9, "unit": "GB/s", "ms_per_step": ms_pair,
        "ms_separate_applies": ms_sep, "bytes_per_step": B, "workload": f"cfg{cfg.idx} PWL",
        "ranks": [inf["ranks"] for inf in infos], "heldout_err": [inf["heldout_err"] for inf in infos],
        "compression": [float(inf["compression"]) for inf in infos], "build_s": build_s, "steps": args.steps,
        "round": None if args.round is None else {"tol": args.round, "ranks_before": ranks_before},
        "l2_flush": "512 MiB fill between steps"}))


if __name__ == "__main__":
    main()
