"""Summaries of one profiling pass (scripts_profile.sh output dir): kernel
shares from the ncu launch lists and per-launch duration / DRAM traffic /
issue rate from the --set full captures. Usage: prof_summary.py DIR."""
import csv
import io
import statistics
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr = rows[0]
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    per = defaultdict(list)
    for r in rows[1:]:
        if len(r) > vi and r[hdr.index("Metric Name")] == "gpu__time_duration.sum":
            v = float(r[vi].replace(",", ""))
            unit = r[hdr.index("Metric Unit")]
            us = v / 1e3 if unit in ("ns", "nsecond") else (v * 1e3 if unit in ("ms", "msecond") else v)
            per[r[ki].split("(")[0]].append(us)
    return per


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                          "gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,"
                          "sm__inst_executed.avg.per_cycle_active,launch__registers_per_thread,"
                          "lts__t_sector_hit_rate.pct"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    per = defaultdict(list)
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        per[d["Kernel Name"].split("(")[0]].append(d)
    return per, dict(zip(hdr, units))


if __name__ == "__main__":
    base = sys.argv[1]
    for cfg in ("cfg2", "cfg4"):
        per = launches(f"{base}/launches_{cfg}.csv")
        tot = sum(sum(v) for k, v in per.items() if "Fill" not in k and "fill" not in k)
        print(f"## launch list {cfg} (us per launch, share of the quantize; the L2-flush fill excluded)")
        for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
            sh = "" if "ill" in k else f"{100 * sum(v) / tot:5.1f}%"
            print(f"  {k[:60]:60s} n={len(v):4d} mean={statistics.mean(v):9.1f} {sh}")
    for rep in ("small_cfg2", "large_cfg4"):
        per, units = full(f"{base}/{rep}.ncu-rep")
        print(f"## ncu --set full {rep} (mean per launch; units {units.get('dram__bytes_read.sum')}, "
              f"{units.get('gpu__time_duration.sum')})")
        for k, ds in per.items():
            f = lambda m: statistics.mean(float(d[m].replace(",", "")) for d in ds)  # noqa: E731
            rd, wr, t = f("dram__bytes_read.sum"), f("dram__bytes_write.sum"), f("gpu__time_duration.sum")
            print(f"  {k[:50]:50s} n={len(ds)} t={t:.4f} dram_r+w={rd + wr:.2f} ipc={f('sm__inst_executed.avg.per_cycle_active'):.2f} "
                  f"regs={f('launch__registers_per_thread'):.0f} l2hit={f('lts__t_sector_hit_rate.pct'):.1f}")
