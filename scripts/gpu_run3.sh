set -x
timeout 900 python -m pytest tests -m gpu -q -x -k "input_transform or layer or smoke" > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --sweep off > gpurun_out/bench3.json 2> gpurun_out/bench3.err; echo "rc=$?" >> gpurun_out/bench3.err
