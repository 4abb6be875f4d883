#!/bin/bash
# Round-2 evidence on one B200 (run through gpurun from the repo root).
#   part 1: GPU tests, the default bench line, the other configs, the error study
#   part 2: the ncu launch list of the bench command and full captures of the top
#           kernels (bf16 lin4 / fp32 lin4 / bf16 lin8), exported to text on the box
#           (gpurun returns at most 64 MiB).  compute-sanitizer is closed on this pool.
set -u
mkdir -p gpurun_out
part=${1:-all}
if [ "$part" = 1 ] || [ "$part" = all ]; then
  python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "tests rc=$?"
  python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?"
  python scripts/configs_timing.py > gpurun_out/configs_r02.json 2> gpurun_out/configs.err; echo "configs rc=$?"
  python scripts/error_study.py > gpurun_out/error_study_r02.json 2> gpurun_out/es.err; echo "error study rc=$?"
fi
if [ "$part" = 2 ] || [ "$part" = all ]; then
  B="python bench.py --steps 2 --warmup 3 --no-extras --graph off"
  $B > gpurun_out/plain.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1
  for tag in bf16_lin4 fp32_lin4 bf16_lin8; do
    case $tag in
      bf16_lin4) X="";;
      fp32_lin4) X="--dtype fp32";;
      bf16_lin8) X="--algo lin8";;
    esac
    $B $X > gpurun_out/plain_$tag.log 2>&1 && \
      ncu --set full --clock-control none -k regex:"domain_gemm|input_transform|output_transform|weight_transform" -s 4 -c 4 \
          -o /tmp/prof_$tag $B $X > gpurun_out/ncu_$tag.log 2>&1 && \
      ncu -i /tmp/prof_$tag.ncu-rep --page raw --csv > gpurun_out/ncu_raw_$tag.csv 2>/dev/null && \
      ncu -i /tmp/prof_$tag.ncu-rep --page details > gpurun_out/ncu_details_$tag.txt 2>/dev/null
    echo "$tag rc=$?"
  done
fi
echo done
