"""Per-launch ncu counters of the integrator (and, for csv names containing "contract", of the window
contraction) per config -> profiles/ncu_counters.json (read by bench.py).

usage: python tools/ncu_counters.py OUT.json LIB_SHA16 cfg0.csv cfg1.csv ...   (one csv per config, from
  ncu --metrics smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,
      sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,
      sm__inst_issued.avg.pct_of_peak_sustained_active --csv -k regex:integrate ...)
The csv name must contain cfgN.  Values are the mean over the captured launches.
"""
import collections
import csv
import json
import re
import sys

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
         "second": 1.0, "inst": 1, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9, "hz": 1, "Khz": 1e3, "Mhz": 1e6,
         "Ghz": 1e9, "%": 1, "cycle/second": 1, "cycle/nsecond": 1e9, "cycle/usecond": 1e6}

out, sha = sys.argv[1], sys.argv[2]
try:
    res = json.load(open(out))
except Exception:
    res = {}
for path in sys.argv[3:]:
    cfg = re.search(r"cfg(\d)", path).group(1)
    rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
    h = rows[0]
    ni, mi, vi, ui, ki = (h.index(k) for k in ("ID", "Metric Name", "Metric Value", "Metric Unit", "Kernel Name"))
    per = collections.defaultdict(dict)
    kname = {}
    for r in rows[1:]:
        v = float(r[vi].replace(",", "")) * UNITS.get(r[ui], 1)
        per[r[ni]][r[mi]] = v
        kname[r[ni]] = r[ki]
    n = len(per)
    mean = lambda m: sum(d.get(m, 0.0) for d in per.values()) / max(1, n)
    key = f"config{cfg}_contract" if "contract" in path.split("/")[-1] else f"config{cfg}"
    res[key] = {
        "lib_sha16": sha, "launches": n, "kernel": next(iter(kname.values()))[:80] if kname else None,
        "inst_executed": mean("smsp__inst_executed.sum"), "dram_read": mean("dram__bytes_read.sum"),
        "dram_write": mean("dram__bytes_write.sum"), "duration_s": mean("gpu__time_duration.sum"),
        "sm_hz": mean("sm__cycles_elapsed.avg.per_second"),
        "hmma_active_pct": mean("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "issue_active_pct": mean("sm__inst_issued.avg.pct_of_peak_sustained_active"),
        "source": f"ncu --metrics (cold cache, serialised) on bench.py --config {cfg}, {path.split('/')[-1]}",
    }
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))
