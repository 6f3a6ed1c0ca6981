"""Summarise an ncu source page (SASS) by stall samples: top instructions."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source=sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ii = h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) <= si:
        continue
    try:
        data.append((int(r[si] or 0), int(r[ii] or 0), r[0], r[1]))
    except ValueError:
        pass
tot = sum(d[0] for d in data) or 1
print("total samples", tot, "instructions", sum(d[1] for d in data))
for idx, d in enumerate(data):
    pass
order = sorted(range(len(data)), key=lambda i: -data[i][0])[:top]
for i in sorted(order):
    s, n, a, src = data[i]
    print("%5d %5.1f%% %10d  %s" % (i, 100.0 * s / tot, n, src.strip()[:90]))
