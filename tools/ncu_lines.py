"""Stall samples of an ncu report aggregated by CUDA source line (needs -lineinfo and --import-source on).

usage: python tools/ncu_lines.py REPORT.ncu-rep [TOP]
Inlined helpers are charged to their own lines; prints share of all samples, instructions executed
and the top stall reasons per line.
"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = next(r for r in rows if r and r[0] == "Line No")
si, ie = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
reasons = [(i, h) for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows:
    if len(r) != len(hdr) or r[0] == "Line No" or r[2] != "-":
        continue
    try:
        s = int(r[si] or 0)
    except ValueError:
        continue
    if s:
        rs = sorted(((int(r[i] or 0), h[6:]) for i, h in reasons), reverse=True)[:3]
        lines.append((s, int(r[ie] or 0), int(r[0]), r[1].strip()[:70], rs))
tot = sum(l[0] for l in lines)
for s, n, ln, src, rs in sorted(lines, reverse=True)[:top]:
    why = ", ".join(f"{h}:{v / s:.2f}" for v, h in rs if v)
    print(f"{s / tot:6.3f} {n / 1e6:8.2f}M L{ln:<5d} {src:70s} {why}")
