"""Registers / spills / barriers per integrate_kernel instance from `python -m paper_1305_6861_b200.build --force -v`
output on stdin (the -Xptxas -v log), one line per instance."""
import re
import subprocess
import sys

cur = None
rows = []
spill = ""
for line in sys.stdin:
    m = re.search(r"Compiling entry function '(_Z\S+)'", line)
    if m:
        cur = subprocess.run(["c++filt", m.group(1)], capture_output=True, text=True).stdout.strip()
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m and cur:
        spill = f"stack {m.group(1)} spill st {m.group(2)} ld {m.group(3)}"
        continue
    m = re.search(r"Used (\d+) registers", line)
    if m and cur:
        if "integrate_kernel" in cur:
            name = cur.replace("void bloch::integrate_kernel", "integrate").replace("(bloch::KParams)", "")
            rows.append(f"{name:45s} regs {m.group(1):>4s}  {spill}")
        cur = None
print("\n".join(sorted(rows)))
