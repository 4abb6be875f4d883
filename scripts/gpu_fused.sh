set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "full_size or layer or vgg or ranking" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for L in 2 3 4 6 100; do WINO_FUSED_LAG=$L timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras > gpurun_out/bench_fused_L$L.json 2> gpurun_out/bench_fused_L$L.err; done
WINO_UNFUSED=1 timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err
