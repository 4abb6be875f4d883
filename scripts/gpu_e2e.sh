timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_io or full_size" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python bench.py --steps 30 --warmup 3 --sweep off > gpurun_out/bench_e2e.json 2> gpurun_out/bench_e2e.err; echo "rc=$?" >> gpurun_out/bench_e2e.err
