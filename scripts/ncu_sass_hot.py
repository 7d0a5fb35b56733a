"""Top SASS lines of an ncu report by stall samples and by executed instructions."""
import csv
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
h = rows[hi]
ai, si = h.index("Address"), h.index("Source")
wi, ii = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    try:
        data.append((int(r[wi]), int(r[ii]), r[ai][-5:], r[si].strip()[:95]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
toti = sum(d[1] for d in data) or 1
print(f"samples={tot} instructions={toti} sass_lines={len(data)}")
print("-- by stall samples")
for d in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{d[0]:8d} {100 * d[0] / tot:5.1f}% inst={d[1]:11d} {d[2]} {d[3]}")
print("-- by instructions executed")
for d in sorted(data, key=lambda x: -x[1])[:n]:
    print(f"{d[1]:11d} {100 * d[1] / toti:5.1f}% {d[2]} {d[3]}")
