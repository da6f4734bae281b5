"""SASS opcode summary of the library's kernels (cuobjdump -sass): per kernel the count of the
instructions that show which hardware paths a kernel uses -- DMMA (FP64 tensor cores,
mma.sync.m8n8k4.f64; tcgen05 has no f64 kind), UBLKCP / UTMALDG (1-D bulk / tensor TMA),
SYNCS (mbarrier), DFMA / DMUL / DADD (FP64 pipe), LDGSTS (cp.async), MUFU (special functions).

    python tools/sass_summary.py [out.json]"""
import collections, json, os, re, subprocess, sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2206_12409_b200", "libvsie_coupling.so")
OPS = ("DMMA", "UBLKCP", "UTMALDG", "SYNCS", "DFMA", "DMUL", "DADD", "LDGSTS", "MUFU", "HMMA", "UTCHMMA")


def main():
    sass = subprocess.run(["cuobjdump", "-sass", LIB], capture_output=True, text=True, check=True).stdout
    out = collections.OrderedDict()
    cur = None
    for line in sass.splitlines():
        m = re.search(r"Function : (\S+)", line)
        if m:
            cur = m.group(1)
            dm = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip()
            cur = re.sub(r"\(.*", "", dm.replace("vsie::(anonymous namespace)::", ""))
            out.setdefault(cur, collections.Counter())
            continue
        if cur is None:
            continue
        for op in OPS:
            if re.search(r"\b" + op + r"\b", line):
                out[cur][op] += 1
    tot = collections.Counter()
    for c in out.values():
        tot.update(c)
    res = {"library": os.path.relpath(LIB, ROOT), "arch": "sm_100a",
           "totals": dict(tot), "kernels": {k: dict(v) for k, v in out.items() if v}}
    path = sys.argv[1] if len(sys.argv) > 1 else None
    if path:
        json.dump(res, open(path, "w"), indent=1)
    print(json.dumps(res["totals"]))


if __name__ == "__main__":
    main()
