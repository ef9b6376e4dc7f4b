#!/bin/bash
# Full C5 cross product: N = 64, C_in = C_out in {64,128,256,512} x
# H = W in {56,28,14,7}, families proposed / t4 / t2_linear, bf16 fwd+bwd. One bench
# line per point into gpurun_out/<tag>_c5_grid.jsonl (run under gpurun from the repo root).
tag=${1:-rx}
out=gpurun_out/${tag}_c5_grid.jsonl
rm -f $out
for fam in ${FAMS:-proposed t4 t2lin}; do for c in 64 128 256 512; do for hw in 56 28 14 7; do
  python - "c5_${fam}_${c}x${hw}" <<'PY' >> $out 2>/dev/null
import sys, bench
w = sys.argv[1]
if w not in bench.WORKLOADS:
    fam, s = w[3:].rsplit("_", 1)
    c, hw = map(int, s.split("x"))
    bench.WORKLOADS[w] = ({"t2lin": "t2_linear"}.get(fam, fam), "conv", 64, c, c, hw, hw, 3, 1, 1, "bf16")
sys.argv = ["bench.py", "--workload", w, "--steps", "10", "--warmup", "3", "--no-cpu", "--nets", ""]
bench.main()
PY
done; done; done
python - $out <<'PY'
import json, sys
rows = {}
for l in open(sys.argv[1]):
    l = l.strip()
    if not l.startswith("{"):
        continue
    d = json.loads(l)
    w = d["config"]["workload"].split(":")[0]
    _, fam, s = w.split("_", 2)
    rows.setdefault(fam, {})[s] = d
for fam, r in rows.items():
    print(f"{fam}: TFLOP/s (ms/step), rows C = 64..512, columns HW = 56, 28, 14, 7")
    for c in (64, 128, 256, 512):
        print("  C=%3d " % c + "  ".join(
            "%7.1f (%6.3f)" % (r[f"{c}x{hw}"]["value"], r[f"{c}x{hw}"]["ms_per_step"]) if f"{c}x{hw}" in r else "   --   "
            for hw in (56, 28, 14, 7)))
PY
