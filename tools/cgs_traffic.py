"""Per-launch DRAM traffic of the CGS2 sweeps in the REAL bench step (warm
L2, --cache-control none) against their algorithmic bytes, from an ncu
launch list of tools/one_step.py and the engine counters of the same step.

  IRKG_GRAPHS=0 ncu --nvtx --nvtx-include "step/" --cache-control none \\
      --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,\\
      dram__bytes_write.sum --csv --log-file launches.csv \\
      python tools/one_step.py --out counters.json
  python tools/cgs_traffic.py launches.csv counters.json --out profiles/r2_cgs_traffic.json
"""
import argparse
import collections
import csv
import json
import re


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("launches")
    ap.add_argument("counters")
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    rows = [r for r in csv.reader(open(args.launches)) if len(r) > 10]
    hdr = rows[0]
    ik, im, iv, iid = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in rows[1:]:
        if r[iid].isdigit():
            per[int(r[iid])][r[im]] = float(r[iv].replace(",", ""))
            names[int(r[iid])] = re.sub(r"\(.*", "", r[ik]).replace("void ", "").strip()
    kinds = collections.defaultdict(lambda: [0, 0.0, 0.0, 0.0])
    for i, m in per.items():
        k = kinds[names[i]]
        k[0] += 1
        k[1] += m.get("gpu__time_duration.sum", 0.0)
        k[2] += m.get("dram__bytes_read.sum", 0.0)
        k[3] += m.get("dram__bytes_write.sum", 0.0)
    cnt = json.load(open(args.counters))
    cgs = [v for n, v in kinds.items() if n.startswith("k_cgs")]
    launches = sum(v[0] for v in cgs)
    traffic = sum(v[2] + v[3] for v in cgs) / max(1, launches)
    alg = cnt["cgs_bytes"] / max(1, cnt["cgs_launches"])
    tot_t = sum(v[1] for v in kinds.values())
    doc = {
        "what": f"CGS2 sweeps of one configs[1] step ({launches} launches, "
                f"{cnt['arnoldi_iterations']} Arnoldi steps)",
        "cache": "warm L2 (ncu --cache-control none, the bench step's own L2 state)",
        "traffic_per_launch": traffic, "algorithmic_per_launch": alg, "ratio": traffic / alg,
        "ncu_launches": launches, "engine_cgs_launches": cnt["cgs_launches"],
        "kernels": {n: {"launches": v[0], "time_share": v[1] / tot_t,
                        "avg_us": v[1] / v[0] / 1e3, "dram_read_mb": v[2] / v[0] / 1e6,
                        "dram_write_mb": v[3] / v[0] / 1e6}
                    for n, v in sorted(kinds.items(), key=lambda kv: -kv[1][1])},
    }
    print(json.dumps({k: doc[k] for k in ("what", "traffic_per_launch",
                                          "algorithmic_per_launch", "ratio")}, indent=1))
    if args.out:
        with open(args.out, "w") as fh:
            json.dump(doc, fh, indent=1)


if __name__ == "__main__":
    main()
