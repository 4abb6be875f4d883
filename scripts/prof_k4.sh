B="python bench.py --steps 3 --warmup 3 --no-extras --algo lin6"
timeout 300 $B > gpurun_out/p_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:output_transform -s 2 -c 1 -o gpurun_out/prof_k4lin6 $B > gpurun_out/ncu_k4.log 2>&1
