"""Write tests/golden/cfg1_dense_summary.json (pin P17, regression).

Calls only oracle/ and synth/.  Run after the P1-P16 pins pass:
    python tools/make_golden.py
"""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import entries  # noqa: E402

SEED = 12409017


def main():
    cfg = synth.get_config(1)
    prob = entries.problem_from_config(cfg)
    Z = entries.dense(prob)
    nv = cfg.n_v
    fro = [float(np.linalg.norm(Z[c * nv:(c + 1) * nv])) for c in range(3)]
    W = synth.complex_gaussian(Z.size, SEED).reshape(Z.shape)
    cs = complex(np.sum(W * Z))
    out = dict(
        source="oracle/entries.dense on synth config 1 (SURVEY §8c-E, §8d cfg 1); written by tools/make_golden.py",
        shape=list(Z.shape), fro=fro, checksum_seed=SEED, checksum=[cs.real, cs.imag])
    path = os.path.join(ROOT, "tests", "golden", "cfg1_dense_summary.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(path, out)


if __name__ == "__main__":
    main()
