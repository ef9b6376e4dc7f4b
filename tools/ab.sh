#!/bin/bash
# A/B of env settings over layer workloads (run under gpurun from the repo root):
# tools/ab.sh "<workloads>" "<env settings, QD_X=0 = baseline>" [nets]
for w in $1; do
  for v in $2; do
    echo -n "$w $v: "; env $v python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --nets "" 2>/dev/null | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); k=d['roofline'].get('kernels',{})
print(round(d['value'],1), round(d['ms_per_step']*1000,1), ' '.join(f'{n}={v[\"ms\"]*1000:.1f}' for n,v in k.items()))"
  done
done
for n in $3; do for v in $2; do
  echo -n "$n $v: "; env $v python bench.py --workload $n --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step'],3))"
done; done
