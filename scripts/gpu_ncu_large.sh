#!/bin/bash
# ncu captures (one call) of the slow large-tile kernels: K4 and K1 for lin7, K1 for
# lin8 and sup1_6 (cfg5 shapes, bf16), exported to text on the box.
set -u
mkdir -p gpurun_out
for a in ${*:-lin7 lin8}; do
  ncu --set full --clock-control none --import-source on -k regex:"input_transform|output_transform" -s 2 -c 2 \
      -o /tmp/prof_$a python scripts/kernel_times.py $a bf16 > gpurun_out/ncu_$a.log 2>&1
  ncu -i /tmp/prof_$a.ncu-rep --page details > gpurun_out/ncu_details_large_$a.txt 2>/dev/null
  ncu -i /tmp/prof_$a.ncu-rep --page source --csv > gpurun_out/ncu_source_large_$a.csv 2>/dev/null
  echo "$a rc=$?"
done
