set -x
for D in 0 1 2 4 6 7 15; do WINO_FUSED=1 WINO_FUSED_LAG=8 WINO_FUSED_DBG=$D timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras > gpurun_out/bench_fdbg_$D.json 2> gpurun_out/bench_fdbg_$D.err; done
