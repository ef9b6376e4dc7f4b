#!/bin/bash
# fc GEMMs with the 512@7 conv's GEMM shapes (M = 6272 pixels): do 2-D TMA boxes
# run the v1 kernel faster than the conv's 4-D (7 x 7 x 2 pixel) boxes?
for spec in "fc_fprop_like:proposed:fc:6272:4608:512" "fc_small:proposed:fc:6272:512:512"; do
  IFS=: read name fam kind n c f <<< "$spec"
  python - "$name" "$fam" "$kind" "$n" "$c" "$f" <<'PY'
import sys, bench
name, fam, kind, n, c, f = sys.argv[1:7]
bench.WORKLOADS[name] = (fam, kind, int(n), int(c), int(f), 1, 1, 1, 1, 0, "bf16")
sys.argv = ["bench.py", "--workload", name, "--steps", "10", "--warmup", "3", "--no-cpu", "--nets", ""]
import io, contextlib, json
buf = io.StringIO()
with contextlib.redirect_stdout(buf):
    bench.main()
d = json.loads(buf.getvalue().strip().splitlines()[-1])
print(name, round(d["value"], 1), {k: round(v["ms"] * 1000, 1) for k, v in d["roofline"]["kernels"].items()})
PY
done
