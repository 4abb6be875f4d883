set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "nhwc or layer" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --layout nhwc > gpurun_out/bench_nhwc.json 2> gpurun_out/bench_nhwc.err; echo "rc=$?" >> gpurun_out/bench_nhwc.err
