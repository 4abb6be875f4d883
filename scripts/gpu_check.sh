# full GPU suite + K1 timing + bench line; md5 of the library that ran
md5sum paper_1905_05233_b200/libwino.so
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log; tail -3 gpurun_out/gpu_tests.log
for a in lin4 lin6 sup1_6 sup1_10 sup1_12; do timeout 120 python scripts/time_k1.py $a bf16 2>&1 | tail -1; done
timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['ms_per_step'], d['value'], d['gpu_launches'], d['clocks'])"
