for w in c5_proposed_64x56 c5_proposed_128x28 c5_proposed_256x14 c5_t4_64x56 c5_t2lin_64x56 r18_64x56 r18_128x28 c2_fp32; do
  for v in "QD_X=0" "QD_ASLOTS=2" "QD_ASLOTS=3"; do
    echo -n "$w $v: "; env $v python bench.py --workload $w --steps 10 --warmup 3 --no-cpu --nets "" 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1), round(d['ms_per_step']*1000,1))"
  done
done
for v in "QD_X=0" "QD_ASLOTS=2"; do
  echo -n "r18net $v: "; env $v python bench.py --workload qresnet18 --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))"
  echo -n "vgg $v: "; env $v python bench.py --workload qvgg16 --steps 10 --warmup 3 --no-cpu 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['value'],1))"
done
