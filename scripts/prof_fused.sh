B="python bench.py --steps 3 --warmup 3 --no-extras"
timeout 300 $B > gpurun_out/p_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused -s 2 -c 1 -o gpurun_out/prof_fused1 $B > gpurun_out/ncu_fused1.log 2>&1
