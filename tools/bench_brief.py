import json,sys
for l in sys.stdin.read().strip().splitlines():
    if not l.startswith("{"): continue
    d=json.loads(l); e=d.get("e2e") or {}
    print(round(d["value"]/1e9,2), round(d["ms_per_step"],4), round(d["roofline"]["kernel_ms_avg"],4), round((e.get("value") or 0)/1e9,3), round(e.get("ms_per_step") or 0,3), d["gpu_launches"], d["clocks"]["sm_mhz"])
