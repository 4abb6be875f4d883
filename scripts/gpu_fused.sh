set -x
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "fused" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for L in 4 6 8 10 14; do WINO_FUSED=1 WINO_FUSED_LAG=$L timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras > gpurun_out/bench_fused_L$L.json 2> gpurun_out/bench_fused_L$L.err; done
timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras > gpurun_out/bench_unfused.json 2> gpurun_out/bench_unfused.err
