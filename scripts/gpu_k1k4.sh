#!/bin/bash
# Per-kernel times of the sweep rows (cfg5, bf16) and, after a clean plain run, one ncu
# capture of K1 + K4 for the named algorithm.
set -u
mkdir -p gpurun_out
prof=${1:-lin8}; shift
: > gpurun_out/kt.jsonl
for a in ${*:-lin4 lin5 lin6 lin7 lin8}; do
  timeout 120 python scripts/kernel_times.py $a bf16 >> gpurun_out/kt.jsonl 2>> gpurun_out/kt.err; echo "kt $a rc=$?"
done
cut -c1-330 gpurun_out/kt.jsonl
if [ "$prof" != none ]; then
  python scripts/kernel_times.py $prof bf16 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:"input_transform|output_transform" -s 2 -c 2 \
      -o /tmp/prof_$prof python scripts/kernel_times.py $prof bf16 > gpurun_out/ncu_$prof.log 2>&1
  ncu -i /tmp/prof_$prof.ncu-rep --page details > gpurun_out/ncu_details_large_$prof.txt 2>/dev/null
  ncu -i /tmp/prof_$prof.ncu-rep --page source --csv > gpurun_out/ncu_source_large_$prof.csv 2>/dev/null
  echo "ncu $prof rc=$?"
fi
