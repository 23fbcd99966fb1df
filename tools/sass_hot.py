"""Top SASS instructions of an ncu report by warp-stall samples:
python tools/sass_hot.py report.ncu-rep [N]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr = rows[1]
data = [r for r in rows[2:] if len(r) == len(hdr)]
iS, iI, iSrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
tot = sum(int(r[iS]) for r in data)
print("samples", tot, "warp instructions", sum(int(r[iI]) for r in data))
for s, k in sorted(((int(r[iS]), k) for k, r in enumerate(data)), reverse=True)[:top]:
    print(f"{k:5d} {s:8d} {100 * s / tot:5.1f}% {int(data[k][iI]):12d}  {data[k][iSrc].strip()[:80]}")
