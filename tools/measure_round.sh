#!/bin/bash
# Round measurement set (run under gpurun from the repo root): bench lines, sweep,
# launch list and one ncu --set full capture of the C2 step kernels. Outputs: gpurun_out/<tag>_*.
tag=${1:-rx}
o=gpurun_out/${tag}
python bench.py --steps 20 --warmup 5 > ${o}_bench_c2.json 2> ${o}_bench_c2.err
python bench.py --impl reference --steps 3 --warmup 1 > ${o}_bench_c2_ref.json 2>&1
python bench.py --workload qvgg16 --steps 20 --warmup 5 > ${o}_bench_qvgg16.json 2>&1
python bench.py --workload qresnet18 --impl reference --steps 2 --warmup 0 > ${o}_bench_qresnet18_ref.json 2>&1
python bench.py --workload c2_fp32 --steps 10 --warmup 3 > ${o}_bench_c2_fp32.json 2>&1
python bench.py --workload c1 --steps 20 --warmup 5 > ${o}_bench_c1.json 2>&1
python bench.py --workload dw_proposed_256x28 --steps 10 --warmup 3 --no-cpu > ${o}_bench_dw.json 2>&1
rm -f ${o}_sweep.jsonl
for fam in proposed t4 t2lin; do for s in 64x56 128x28 256x14 512x7; do
  w=c5_${fam}_${s}
  python - "$w" <<'PY' >> ${o}_sweep.jsonl 2>/dev/null
import sys, bench
w = sys.argv[1]
if w not in bench.WORKLOADS:
    fam, s = w[3:].rsplit("_", 1)
    c, hw = map(int, s.split("x"))
    bench.WORKLOADS[w] = ({"t2lin": "t2_linear"}.get(fam, fam), "conv", 64, c, c, hw, hw, 3, 1, 1, "bf16")
sys.argv = ["bench.py", "--workload", w, "--steps", "10", "--warmup", "3", "--no-cpu"]
bench.main()
PY
done; done
QD_NO_PART=1 QD_FOLD_MAIN=1 python tools/prof_step.py 3 > ${o}_prof_plain.log 2>&1 && \
  QD_NO_PART=1 QD_FOLD_MAIN=1 ncu --set full --clock-control none --import-source on -k regex:"conv2|wgrad3|prologue|pack|wsum|wfinish" -s 7 -c 7 \
      -o ${o}_c2_full python tools/prof_step.py 3 > ${o}_ncu_full.log 2>&1
python bench.py --steps 2 --warmup 3 --nets "" --no-cpu > ${o}_plain_launch.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${o}_launches.csv \
      python bench.py --steps 2 --warmup 3 --nets "" --no-cpu > ${o}_ncu_launch.log 2>&1
echo measure done
# single-rank torchrun with every collective on (NCCL process group, graph-captured all-reduces)
QD_DIST_FORCE=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29531 \
    bench.py --gpus 1 --steps 20 --warmup 5 --no-cpu > ${o}_bench_dist1.json 2> ${o}_bench_dist1.err
python tools/gaps.py qresnet18 10 > ${o}_resnet_kernels.txt 2>&1
echo measure2 done
