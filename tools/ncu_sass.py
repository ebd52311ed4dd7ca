"""Per-instruction stall samples of an ncu report between two SASS offsets (hex, last 5 hex digits as ncu_regions.py prints, inclusive)."""
import csv, io, subprocess, sys

rep, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hh, data = rows[1], rows[2:]
ia, src, st, ad = (hh.index("Instructions Executed"), hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"),
                   hh.index("Address"))
reasons = [x for x in hh if x.startswith("stall_") and "Not Issued" not in x]
ri = [hh.index(x) for x in reasons]
tot = sum(int(r[st] or 0) for r in data)
base = int(data[0][ad], 16)
for r in data:
    a = int(r[ad], 16) & 0xFFFFF  # the last 5 hex digits, as ncu_regions.py prints them
    if lo <= a <= hi:
        s = int(r[st] or 0)
        top = sorted(((int(r[i] or 0), n[6:]) for n, i in zip(reasons, ri)), reverse=True)[:2]
        print(f"{a:6x} {s / tot * 100:5.2f}% {int(r[ia] or 0) / 1e6:7.2f}M {r[src].strip()[:60]:60s} "
              + " ".join(f"{n}:{v}" for v, n in top if v))
