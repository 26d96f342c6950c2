"""Per-kernel SASS opcode histograms of the built engine (cuobjdump -sass of
the sm_100a objects): the instructions that prove the data-movement path --
UTMALDG (TMA tensor-map loads), UBLKCP (cp.async.bulk), LDGSTS (Ampere-style
cp.async), SYNCS (mbarrier waits) -- plus DFMA/DADD/DMUL (FP64 work),
LDG/STG/LDS/STS, SHFL and total instruction counts.

    python tools/sass_histogram.py [--out profiles/r2_sass_histogram.txt]
"""

import argparse
import collections
import glob
import os
import re
import subprocess

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ["UTMALDG", "UBLKCP", "LDGSTS", "SYNCS", "DFMA", "DADD", "DMUL", "LDG", "STG", "LDS",
        "STS", "SHFL", "BAR", "ATOMG", "RED"]


def demangle(names):
    try:
        out = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True,
                             text=True, check=True).stdout.split("\n")
        return dict(zip(names, out))
    except Exception:
        return {n: n for n in names}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--filter", default="k_cgs|k_jacobi|k_block_op|k_residual|k_newton|k_mg|"
                                        "k_band|k_ara|k_dae|k_gmres")
    args = ap.parse_args()
    objs = sorted(glob.glob(os.path.join(ROOT, "paper_2101_01776_b200", "csrc", "*.o")))
    rows = []
    for obj in objs:
        sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
        cur, hist = None, None
        funcs = []
        for line in sass.split("\n"):
            m = re.match(r"\s*Function : (\S+)", line)
            if m:
                cur = m.group(1)
                hist = collections.Counter()
                funcs.append((cur, hist))
                continue
            m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(@!?U?P\w+\s+)?([A-Z][A-Z0-9_]*)(\.[\w.]*)?", line)
            if m and hist is not None:
                op = m.group(2)
                hist["total"] += 1
                for k in KEYS:
                    if op == k or op.startswith(k):
                        hist[k] += 1
        names = demangle([f for f, _ in funcs])
        for f, h in funcs:
            nm = names.get(f, f)
            if re.search(args.filter, nm):
                rows.append((os.path.basename(obj), nm, h))
    lines = ["object | kernel | total | " + " | ".join(KEYS), "---|---|---|" + "---|" * len(KEYS)]
    for obj, nm, h in rows:
        short = nm if len(nm) < 110 else nm[:107] + "..."
        lines.append(f"{obj} | {short} | {h['total']} | " + " | ".join(str(h[k]) for k in KEYS))
    text = "\n".join(lines)
    print(text)
    if args.out:
        with open(args.out, "w") as fh:
            fh.write("# SASS opcode histograms (cuobjdump -sass, sm_100a objects of this build)\n\n")
            fh.write(text + "\n")


if __name__ == "__main__":
    main()
