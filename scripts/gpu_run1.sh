set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 180 python -m pytest tests/test_gpu_parity.py -x -q -k "domain_gemm_isolated and lin2" > gpurun_out/t1.log 2>&1; echo "rc=$?" >> gpurun_out/t1.log
grep -q "passed" gpurun_out/t1.log || exit 1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 600 python bench.py --steps 50 --warmup 5 --sweep off > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo "rc=$?" >> gpurun_out/bench1.err
