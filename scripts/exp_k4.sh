for e in tma plain; do for a in sup1_4 lin6 sup1_6 lin8; do if [ $e = plain ]; then export WINO_K4_PLAIN=1; fi; timeout 300 python bench.py --steps 20 --warmup 3 --sweep off --algo $a > gpurun_out/bench_$a.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_$a.json'));print('$e $a', round(d['ms_per_step'],3), round(d['kernels']['output_transform']['us'],1))"; done; done
