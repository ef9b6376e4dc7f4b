#!/bin/bash
# A/B of the squared-input backward schedule: serial (QD_SQ_SERIAL=1), side-stream
# wgrad chain (default), and the SM partition (QD_SQ_PART=<pct of pairs for wgrad3>)
# usage: tools/sq_ab.sh  (under gpurun, from the repo root)
run() {
  python - "$1" <<'PY' 2>/dev/null
import sys, json, io, contextlib, bench
w = sys.argv[1]
if w not in bench.WORKLOADS:
    fam, s = w[3:].rsplit("_", 1)
    c, hw = map(int, s.split("x"))
    bench.WORKLOADS[w] = ({"t2lin": "t2_linear"}.get(fam, fam), "conv", 64, c, c, hw, hw, 3, 1, 1, "bf16")
sys.argv = ["bench.py", "--workload", w, "--steps", "20", "--warmup", "5", "--no-cpu", "--nets", ""]
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
d = json.loads(buf.getvalue().strip().splitlines()[-1])
print(w, round(d["value"], 1), "TFLOP/s", round(d["ms_per_step"] * 1e3, 1), "us")
PY
}
for w in c5_t2lin_64x56 c5_t2lin_128x28 c5_t2lin_256x14 c5_t2_64x56 c5_t2_128x28 c5_t2and4_64x56; do
  echo "serial  $(QD_SQ_SERIAL=1 run $w)"
  echo "side    $(run $w)"
  for pct in 40 50 60; do echo "part$pct  $(QD_SQ_PART=$pct run $w)"; done
done
