set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "input_transform or layer" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --sweep off > gpurun_out/bench_k1t.json 2> gpurun_out/bench_k1t.err; echo "rc=$?" >> gpurun_out/bench_k1t.err
B="python bench.py --steps 3 --warmup 3 --no-extras"
timeout 300 $B > gpurun_out/p_plain.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:input_transform -s 2 -c 1 -o gpurun_out/prof_k1t $B > gpurun_out/ncu_k1t.log 2>&1
