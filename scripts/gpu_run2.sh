set -x
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 100 --warmup 5 --sweep off > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo "rc=$?" >> gpurun_out/bench2.err
