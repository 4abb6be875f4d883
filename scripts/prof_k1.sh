python scripts/time_k1.py > gpurun_out/p_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:input_transform -s 3 -c 1 -o gpurun_out/prof_k1w python scripts/time_k1.py > gpurun_out/ncu_k1w.log 2>&1
