# summarise a gpu_quick.sh run
D=gpurun_out/${1:-quick}
tail -1 $D/pytest_parity.log; tail -1 $D/pytest_c3.log
python - "$D" <<'PY'
import json, re, sys
D = sys.argv[1]
d = json.load(open(f"{D}/bench_c3.json"))
print("ms/step", round(d["ms_per_step"], 1), "combine ms", round(d["roofline"]["kernel_ms_avg"], 1), "walk ms/launch", round(d["roofline"]["walk"]["kernel_ms_avg"], 2))
tot = None
for l in open(f"{D}/prof_c3.err"):
    if l.startswith("[unit-prof]"):
        nums = [float(x) for x in re.findall(r"(?<![\w.])[-+]?\d+\.?\d*(?:e[+-]?\d+)?", l)]
        tot = nums if tot is None else [a + b for a, b in zip(tot, nums)]
names = "units visits queued emissions support cycbuild cycpairs serial serialids pieces pullids pushtests".split()
if tot: print("; ".join(f"{n} {v:.3g}" for n, v in zip(names, tot)))
PY
