#!/bin/bash
# usage: tools/gpu.sh <tag> <timeout_s> '<command>'   (runs from the repo root, logs gpurun_out/call_<tag>.txt)
cd /root/repo || exit 1
mkdir -p gpurun_out
timeout $(( $2 + 1200 )) /usr/local/graft/bin/gpurun --timeout "$2" -- "$3" > "gpurun_out/call_$1.txt" 2>&1
