#!/bin/bash
# A/B of the conv2 B-ring depth cap (QD_C2_BSLOTS=8 = the old cap) on the workloads whose
# conv2 kernels stream B. Run under gpurun from the repo root; output gpurun_out/<tag>_bslots_ab.txt
tag=${1:-rx}
out=gpurun_out/${tag}_bslots_ab.txt
: > $out
one() {  # label, env, workload
  local v=$(env $2 python bench.py --workload $3 --steps 10 --warmup 3 --no-cpu --nets "" 2>/dev/null | python -c "
import sys, json
d = json.loads(sys.stdin.read().strip().splitlines()[-1])
k = d['roofline']['kernels']
print('%8.1f TFLOP/s %8.4f ms  ' % (d['value'], d['ms_per_step']) + ' '.join('%s=%.1f' % (n, v['ms'] * 1e3) for n, v in k.items() if 'conv' in n))")
  echo "$3 [$1] $v" | tee -a $out
}
for w in c5_proposed_128x28 c5_proposed_256x14 r18_128x28 r18_256x14 c5_proposed_512x7; do
  for c in 3 4 6 8 12; do one cap$c QD_C2_BSLOTS=$c $w; done
done
for c in 4 6 8; do
  echo "qresnet18 [cap$c] $(QD_C2_BSLOTS=$c python bench.py --workload qresnet18 --steps 20 --warmup 5 --no-cpu 2>/dev/null | python -c "import sys,json; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])")" | tee -a $out
done
