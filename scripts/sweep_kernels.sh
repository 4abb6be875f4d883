timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "output_transform or layer" > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for a in lin4 sup1_4 lin6 sup1_6 lin8 sup1_8; do timeout 300 python bench.py --steps 20 --warmup 3 --sweep off --algo $a > gpurun_out/bench_$a.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_$a.json'));print('$a', round(d['value']),round(d['ms_per_step'],3), {k:round(v['us'],1) for k,v in d['kernels'].items()})"; done
