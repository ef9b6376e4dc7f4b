#!/bin/bash
# A/B of the conv2 streamed-B ring: per-tap slots (QD_C2_BGROUP=0) vs one slot per channel block
# (all r*r taps on one barrier); QD_C2_BSLOTS caps the per-tap ring depth on the workloads whose
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
for w in c2_fp32 c5_proposed_128x28 c5_proposed_256x14 r18_128x28 r18_256x14 c5_t4_64x56; do
  one pertap QD_C2_BGROUP=0 $w
  one default QD_NOOP=1 $w
  one grouped QD_C2_BGROUP=1 $w
done
