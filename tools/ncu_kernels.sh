#!/bin/bash
# ncu --set full of the launches matching a kernel-name regex in one config-2
# pipeline call, for the given library (default: the in-tree build).
#   bash tools/ncu_kernels.sh <regex> <tag> [lib.so] [count]
set -e
RX=$1; TAG=$2; LIB=${3:-}; CNT=${4:-16}
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --set full --clock-control none --import-source on -k regex:$RX -c $CNT \
  -o gpurun_out/ncu_$TAG -f python tools/prof_batch.py --batch 256 --iters 1 ${LIB:+--lib $LIB} > gpurun_out/ncu_$TAG.log 2>&1
python tools/ncu_summary.py gpurun_out/ncu_$TAG.ncu-rep --out gpurun_out/ncu_$TAG.json --note "ncu --set full -k regex:$RX -c $CNT, tools/prof_batch.py --batch 256 --iters 1 ($LIB)" > /dev/null
rm -f gpurun_out/ncu_$TAG.ncu-rep
