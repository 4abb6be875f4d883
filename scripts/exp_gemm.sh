for s in 4 3; do WINO_GEMM_STAGES=$s timeout 300 python bench.py --steps 50 --warmup 5 --sweep off > gpurun_out/bench_s$s.json 2> /dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_s$s.json'));print('stages $s', d['value'],d['ms_per_step'], {k:round(v['us'],1) for k,v in d['kernels'].items()})"; done
