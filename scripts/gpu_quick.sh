# parity suite + K1 timing + one bench line
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for a in lin4 lin3 lin6 sup1_4 lin2; do timeout 120 python scripts/time_k1.py $a bf16 2>&1 | tail -1; done
timeout 300 python bench.py --steps 30 --warmup 5 --sweep off --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'])"
