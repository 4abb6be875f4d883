set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
B="python bench.py --steps 3 --warmup 3 --no-extras"
timeout 300 $B > gpurun_out/p_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r01b.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in input_transform domain_gemm output_transform weight_transform; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/profb_$k $B > gpurun_out/ncub_$k.log 2>&1
done
