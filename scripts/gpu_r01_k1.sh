set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench_ffma scripts/ubench_ffma.cu && /tmp/ubench_ffma > gpurun_out/ubench_ffma.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --sweep on > gpurun_out/bench_k1.json 2> gpurun_out/bench_k1.err; echo "rc=$?" >> gpurun_out/bench_k1.err
