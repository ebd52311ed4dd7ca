"""Summarise an ncu report: headline metrics + stall-sample regions of the SASS (by execution count)."""
import collections, csv, io, subprocess, sys

rep = sys.argv[1]
def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout
det = ncu("--page", "details")
for key in ["Duration", "Executed Ipc Active", "Issue Slots Busy", "Eligible Warps Per Scheduler", "Active Warps Per Scheduler",
            "Registers Per Thread", "Block Size", "Grid Size", "Achieved Occupancy"]:
    for line in det.splitlines():
        if line.strip().startswith(key):
            print("  ", " ".join(line.split())); break
raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
h, v = raw[0], raw[2]
want = ["sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]
for name in want:
    if name in h: print("  ", name, v[h.index(name)], raw[1][h.index(name)])
rows = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "sass"))))
hh, data = rows[1], rows[2:]
ia, src, st, ad = hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Address")
reasons = [x for x in hh if x.startswith("stall_") and "Not Issued" not in x]
ri = [hh.index(x) for x in reasons]
tot = sum(int(r[st] or 0) for r in data)
regions, cur = [], None
for r in data:
    n, s = int(r[ia] or 0), int(r[st] or 0)
    if cur and abs(cur["n"] - n) <= max(0.05 * n, 20000):
        cur["s"] += s; cur["cnt"] += 1; cur["end"] = r[ad]
    else:
        cur = {"n": n, "s": s, "cnt": 1, "start": r[ad], "end": r[ad], "first": r[src].strip()[:48], "r": collections.Counter()}
        regions.append(cur)
    for name, i in zip(reasons, ri): cur["r"][name] += int(r[i] or 0)
for g in sorted(regions, key=lambda g: -g["s"])[:int(sys.argv[2]) if len(sys.argv) > 2 else 14]:
    top = ", ".join(f"{k[6:]}:{v2 / max(g['s'], 1):.2f}" for k, v2 in g["r"].most_common(3))
    print(f"{g['s'] / tot:6.3f} exec={g['n'] / 1e6:7.2f}M n={g['cnt']:4d} {g['start'][-5:]}-{g['end'][-5:]} {g['first']:48s} {top}")
