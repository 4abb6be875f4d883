set -x
B="python bench.py --steps 3 --warmup 3 --no-extras"
$B > gpurun_out/p_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r01.csv $B > gpurun_out/ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:domain_gemm -s 2 -c 1 -o gpurun_out/prof_gemm $B > gpurun_out/ncu_gemm.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:input_transform -s 2 -c 1 -o gpurun_out/prof_in $B > gpurun_out/ncu_in.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:output_transform -s 2 -c 1 -o gpurun_out/prof_out $B > gpurun_out/ncu_out.log 2>&1
python scripts/l2bw.py > gpurun_out/l2bw.txt 2>&1
