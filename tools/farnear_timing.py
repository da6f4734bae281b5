"""Far-near block (NEXT-3): ACA build time / rank and the Eq. 15 pair time per config.

    python tools/farnear_timing.py [cfg ...] [--tol T]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2206_12409_b200 import FarNear  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfgs", nargs="*", type=int, default=[1, 2, 4])
    ap.add_argument("--tol", type=float, default=None)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--ff", action="store_true", help="also build Z_cc^ff and time its apply")
    a = ap.parse_args()
    for ci in a.cfgs:
        cfg = synth.get_config(ci)
        tol = a.tol if a.tol else max(cfg.tol, 1e-6)
        h = FarNear.build([synth.near_mesh(ci)], cfg.meshes(), cfg.freq, tol)
        inf = h.info()
        mn, mf, k = inf["m_near"], inf["m_far"], inf["rank"]
        xf = torch.from_numpy(synth.complex_gaussian(mf, 1)).cuda()
        xn = torch.from_numpy(synth.complex_gaussian(mn, 2)).cuda()
        yn = torch.empty(mn, dtype=torch.complex128, device="cuda")
        yf = torch.empty(mf, dtype=torch.complex128, device="cuda")
        flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
        res = {}
        for mode in ("pair", "N", "T"):
            def run():
                if mode == "pair":
                    h.apply_pair_raw(xf.data_ptr(), yn.data_ptr(), xn.data_ptr(), yf.data_ptr())
                elif mode == "N":
                    h.apply(xf, "N", out=yn)
                else:
                    h.apply(xn, "T", out=yf)
            for _ in range(5):
                run()
            ts = []
            for it in range(a.iters):
                flush.fill_(it & 255)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run()
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            factor = 16 * k * (mn + mf)
            moved = 2 * factor if mode == "pair" else factor
            res[mode] = dict(ms=ms, factor_bytes=factor, moved_bytes=moved, gbs=moved / ms / 1e6)
        if a.ff:
            from paper_2206_12409_b200 import FarFar
            ff = FarFar.build(cfg.meshes(), cfg.freq)
            fi = ff.info()
            for _ in range(3):
                ff.apply_raw(xf.data_ptr(), yf.data_ptr())
            ts = []
            for it in range(min(a.iters, 50)):
                flush.fill_(it & 255)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ff.apply_raw(xf.data_ptr(), yf.data_ptr())
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            res["ff"] = dict(build_s=fi["build_s"], matrix_bytes=fi["matrix_bytes"], near_pairs=fi["near_pairs"],
                             ms=ms, gbs=fi["matrix_bytes"] / ms / 1e6)
            ff.close()
        print(json.dumps(dict(cfg=ci, tol=tol, m_near=mn, m_far=mf, rank=k, stop=inf["stop"],
                              est_err=inf["est_err"], build_s=inf["build_s"], min_distance=inf["min_distance"],
                              max_edge=inf["max_edge"], **res)), flush=True)
        h.close()


if __name__ == "__main__":
    main()
