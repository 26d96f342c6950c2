"""Key metrics of an ncu --set full report, one line per launch (CSV).

usage: python tools/ncu_summary.py REPORT.ncu-rep [--algo-bytes JSON]
Columns: kernel, duration_us, dram_read_MB, dram_write_MB, dram_GBps,
L2_hit_pct, warps_active_pct, registers, grid, top-3 stall reasons.
"""
import csv
import subprocess
import sys


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h = rows[0]

    def g(r, k):
        try:
            return float(r[h.index(k)].replace(",", ""))
        except (ValueError, IndexError):
            return float("nan")

    w = csv.writer(sys.stdout)
    w.writerow(["kernel", "duration_us", "dram_read_MB", "dram_write_MB", "dram_GBps",
                "L2_hit_pct", "warps_active_pct", "registers", "grid", "stalls"])
    for r in rows[2:]:
        name = r[h.index("Kernel Name")].split("(")[0].replace("void ", "")
        dur = g(r, "gpu__time_duration.sum")
        rd, wr = g(r, "dram__bytes_read.sum"), g(r, "dram__bytes_write.sum")
        stalls = []
        for i, k in enumerate(h):
            if "smsp__pcsamp_warps_issue_stalled" in k and not k.endswith("_not_issued"):
                try:
                    stalls.append((float(r[i]), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        top = " ".join(f"{k}:{100 * v / tot:.0f}%" for v, k in sorted(stalls, reverse=True)[:3])
        w.writerow([name, f"{dur:.2f}", f"{rd:.2f}", f"{wr:.2f}", f"{(rd + wr) / dur * 1e3:.0f}",
                    f"{g(r, 'lts__t_sector_hit_rate.pct'):.1f}",
                    f"{g(r, 'sm__warps_active.avg.pct_of_peak_sustained_active'):.1f}",
                    f"{g(r, 'launch__registers_per_thread'):.0f}", f"{g(r, 'launch__grid_size'):.0f}",
                    top])


if __name__ == "__main__":
    main(sys.argv[1])
