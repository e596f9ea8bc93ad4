#!/bin/bash
# ncu evidence for the config-2 pipeline (run on the GPU box from the repo root):
# 1) launch list of the bench command, 2) launch list of two prof_batch calls
# (-> launches per call), 3) --set full capture of the second call only.
set -e
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum --clock-control none -c 1500 --csv --log-file gpurun_out/launches_bench.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cfg5 --e2e-steps 2 > gpurun_out/ncu_bench.log 2>&1
$NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_call.csv \
  python tools/prof_batch.py --batch 256 --iters 1 > gpurun_out/ncu_call.log 2>&1
# torch's own launches (the input copies) precede the two calls
ALL=$(grep -c '"gpu__time_duration.sum"' gpurun_out/launches_call.csv)
NAT=$(grep '"gpu__time_duration.sum"' gpurun_out/launches_call.csv | grep -c 'at::' || true)
PER=$(( (ALL - NAT) / 2 ))
SKIP=$(( NAT + PER ))
echo "launches per call: $PER (skip $SKIP)" | tee gpurun_out/per_call.txt
$NCU --set full --clock-control none --import-source on -s $SKIP -c $PER -o gpurun_out/full_cfg2 -f \
  python tools/prof_batch.py --batch 256 --iters 1 > gpurun_out/ncu_full.log 2>&1
# summaries travel back; the raw report (> 64 MiB) does not
python tools/ncu_summary.py gpurun_out/full_cfg2.ncu-rep --out gpurun_out/ncu_full_cfg2.json \
  --note "ncu --set full --clock-control none --import-source on -s $SKIP -c $PER python tools/prof_batch.py --batch 256 --iters 1: the second of two config-2 calls (256 graphs N=1024)" > /dev/null
python tools/launch_shares.py gpurun_out/launches_bench.csv --out gpurun_out/launch_shares_cfg2.json \
  --note "ncu --metrics gpu__time_duration.sum --clock-control none -c 1500 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-cfg5 --e2e-steps 2 (cold-cache, serialised: compare shares)" > /dev/null
rm -f gpurun_out/full_cfg2.ncu-rep
