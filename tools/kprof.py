"""Per-K breakdown of [unit-prof] lines: python tools/kprof.py prof.err"""
import sys
keys = ["cols by K:", "cycles by K:", "build cycles by K:", "pull ids by K:", "push tests by K:"]
acc = {k: [0.0] * 8 for k in keys}
for l in open(sys.argv[1]):
    if not l.startswith("[unit-prof]"):
        continue
    for k in keys:
        if k in l:
            v = [float(x) for x in l.split(k)[1].split("|")[0].split()]
            acc[k] = [a + b for a, b in zip(acc[k], v)]
T = sum(acc["cycles by K:"])
for i in range(8):
    c = acc["cycles by K:"][i]
    print(f"K={1 << i:4d} cols {acc['cols by K:'][i]:9.0f} cycles {c:.3g} ({100 * c / T:4.1f}%) build {acc['build cycles by K:'][i]:.3g}"
          f" pull {acc['pull ids by K:'][i]:.3g} push {acc['push tests by K:'][i]:.3g}"
          + (f" cyc/id {c / max(1, acc['pull ids by K:'][i] + acc['push tests by K:'][i]):.2f}"))
