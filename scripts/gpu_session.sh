#!/bin/bash
# One gpurun call: GPU tests (optional), smoke, and per-kernel times of the large-tile
# sweep rows (cfg5 shapes), for A/B work on K1 / K4.
#   bash scripts/gpu_session.sh [tests|notests] [algos...]
set -u
mkdir -p gpurun_out
mode=${1:-tests}; shift || true
algos=${*:-"lin4 lin5 lin6 sup1_6 lin7 lin8"}
if [ "$mode" = tests ]; then
  timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
  tail -3 gpurun_out/gpu_tests.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
fi
: > gpurun_out/kt.jsonl
for a in $algos; do
  for d in bf16; do
    timeout 120 python scripts/kernel_times.py $a $d >> gpurun_out/kt.jsonl 2>> gpurun_out/kt.err; echo "kt $a $d rc=$?"
  done
done
cat gpurun_out/kt.jsonl
