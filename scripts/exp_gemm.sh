for s in 0 1; do WINO_GEMM_EXP=$s timeout 300 python bench.py --steps 50 --warmup 5 --sweep off > gpurun_out/bench_s$s.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_s$s.json'));print('exp $s', d['value'],d['ms_per_step'], {k:round(v['us'],1) for k,v in d['kernels'].items()})"; done
