#!/bin/bash
for k in "$@"; do
  v=$(QD_X3_PART=$k python bench.py --workload c2_fp32 --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1000,1))")
  echo "QD_X3_PART=$k $v"
done
