#!/bin/bash
# C2-fp32 (split path): wgrad3 pairs (QD_X3_PART) beside the persistent dgrad; gpurun_out/<tag>_x3_part_${wl}.txt
tag=${1:-rx}
wl=${2:-c2_fp32}
out=gpurun_out/${tag}_x3_part_${wl}.txt
: > $out
for p in ${3:-20 24 26 28 30 32 34 36 38 40 44 48}; do
  v=$(QD_X3_PART=$p python bench.py --workload $wl --steps 10 --warmup 3 --no-cpu --nets "" 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.1f TFLOP/s %.4f ms' % (d['value'], d['ms_per_step']))")
  echo "QD_X3_PART=$p $v" | tee -a $out
done
