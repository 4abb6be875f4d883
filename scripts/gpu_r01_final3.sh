# final evidence for the round (one gpurun call)
set -x
md5sum paper_1905_05233_b200/libwino.so
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 300 python bench.py --layout nhwc --steps 50 --warmup 5 --sweep off > gpurun_out/bench_nhwc.json 2> gpurun_out/bench_nhwc.err
B="python bench.py --steps 3 --warmup 3 --no-extras"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r01b.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in input_transform domain_gemm output_transform weight_transform; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/profb_$k $B > gpurun_out/ncub_$k.log 2>&1
  ncu -i /tmp/profb_$k.ncu-rep --page raw --csv > gpurun_out/profb_$k.raw.csv 2>/dev/null
  ncu -i /tmp/profb_$k.ncu-rep --page details > gpurun_out/profb_$k.details.txt 2>/dev/null
done
