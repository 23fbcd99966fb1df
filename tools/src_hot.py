"""Per-CUDA-source-line summary of an ncu --set full report (kernel compiled with -lineinfo):
python tools/src_hot.py report.ncu-rep [source.cu] [N]  -> share of warp instructions, of stall samples, active lanes."""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
srcf = sys.argv[2] if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))


def num(x):
    try:
        return int(x)
    except ValueError:
        return 0


m = defaultdict(lambda: [0, 0, 0, "", 0])
cur = None
for r in rows[3:]:
    if len(r) < 10:
        continue
    if r[0] != "":
        try:
            cur = int(r[0])
        except ValueError:
            cur = None
            continue
        m[cur][0] += num(r[4])
        m[cur][1] += num(r[7])
        m[cur][2] += num(r[8])
        m[cur][3] = r[1]
    elif cur:
        m[cur][4] = max(m[cur][4], num(r[7]))
ti = sum(v[1] for v in m.values())
ts = sum(v[0] for v in m.values())
print(f"warp instructions {ti}, stall samples {ts}")
print(" line  %inst  %samples  lanes  max-exec  source")
for l, (sa, i, t, s, mx) in sorted(m.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{l:5d} {100 * i / ti:5.1f}% {100 * sa / ts:5.1f}%  {t / max(i, 1):5.1f} {mx:10.3g}  {s.strip()[:100]}")
if len(sys.argv) > 4:  # line ranges "a-b,c-d": region totals
    for rg in sys.argv[4].split(","):
        a, b = map(int, rg.split("-"))
        i = sum(v[1] for l, v in m.items() if a <= l <= b)
        sa = sum(v[0] for l, v in m.items() if a <= l <= b)
        print(f"lines {a}-{b}: {100 * i / ti:.1f}% inst, {100 * sa / ts:.1f}% samples")
