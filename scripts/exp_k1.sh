timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "input_transform" > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for i in 1 2; do python scripts/time_k1.py; done
python scripts/time_k1.py lin3 bf16; python scripts/time_k1.py lin2 bf16
