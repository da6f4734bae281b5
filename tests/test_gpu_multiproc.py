"""World-2 multi-process path on ONE GPU: two processes share cuda:0
through the CUDA-IPC communicator (host barrier, no kernel waits on another process), so every
`h->comm` branch of the apply and of the cross build runs; each rank's applies equal the
world-1 handle's to 1e-13, the row-split build of cfg 1 (direct factorisations) reproduces the
world-1 build exactly, and the row-split build of cfg 2 (randomized range finder on the ranks'
row blocks) is an equally valid TT (tests/mp_worker.py)."""
import json
import os
import subprocess
import sys
import uuid

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_world2_ipc_equals_world1(tmp_path):
    name = "t" + uuid.uuid4().hex[:12]
    outs = [str(tmp_path / f"r{r}.json") for r in range(2)]
    procs = [subprocess.Popen([sys.executable, os.path.join(ROOT, "tests", "mp_worker.py"), str(r), "2", name, outs[r]],
                              stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True, cwd=ROOT) for r in range(2)]
    logs = [p.communicate(timeout=900) for p in procs]
    for p, (so, se) in zip(procs, logs):
        assert p.returncode == 0, se[-3000:]
    for o in outs:
        res = json.load(open(o))
        for ci in (1, 2):
            for k, v in res[f"cfg{ci}"].items():
                assert v <= 1e-13, (res["rank"], ci, k, v)
        b = res["build"]
        assert b["ranks_equal"] and b["status"] == 0, b
        assert b["N"] <= 1e-13 and b["T"] <= 1e-13, (b, res.get("build_diag"))
        # cfg 2 built with row-split supercores (SURVEY §8e cross step)
        c = res["build_rowsplit"]
        assert c["status"] == 0 and max(c["heldout"]) <= 1e-5, c
        for r1, rp in zip(c["ranks1"], c["ranksp"]):
            for a, b_ in zip(r1, rp):
                assert abs(a - b_) <= max(1, 0.05 * a), c
        assert c["N"] <= 2e-5, c
