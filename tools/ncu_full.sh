#!/bin/bash
# ncu --set full of each tensor-core kernel on one fwd+bwd (B=1 H=8 N=32768 d=128).  Usage: tools/ncu_full.sh TAG [regex] [args]
TAG=${1:-run}; RX=${2:-tc_|sparse_}; shift 2; ARGS=${@:-1 8 32768 128}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:${RX} -c 9 \
  -o gpurun_out/${TAG}_full python tools/prof_step.py $ARGS > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
tail -3 gpurun_out/${TAG}_ncu.log
