#!/bin/bash
# usage: tools/part_sweep.sh K1 K2 ...   (C2 bench at QD_PART=K pairs for the wgrad3)
for k in "$@"; do
  v=$(QD_PART=$k python bench.py --steps 20 --warmup 5 --no-cpu --nets "" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1000,1))")
  echo "QD_PART=$k $v"
done
