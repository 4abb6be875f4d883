# evidence refresh with the current library + Table 2/3 network proxy
set -x
md5sum paper_1905_05233_b200/libwino.so
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
B="python bench.py --steps 3 --warmup 3 --no-extras"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r01b.csv $B > gpurun_out/ncu_launch.log 2>&1
for k in input_transform domain_gemm output_transform weight_transform; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o /tmp/profb_$k $B > gpurun_out/ncub_$k.log 2>&1
  ncu -i /tmp/profb_$k.ncu-rep --page raw --csv > gpurun_out/profb_$k.raw.csv 2>/dev/null
  ncu -i /tmp/profb_$k.ncu-rep --page details > gpurun_out/profb_$k.details.txt 2>/dev/null
done
timeout 1500 python scripts/vgg16_stack.py --n 32 --proxy 32 --reps 3 --dtype bf16 --algos lin4,lin6,lin8,sup1_6,sup1_8,sup1_10,sup1_12 > gpurun_out/vgg16_proxy_bf16.json 2> gpurun_out/vgg16_bf16.err
timeout 1200 python scripts/vgg16_stack.py --n 32 --proxy 32 --reps 3 --dtype fp16 --algos lin4,lin6,sup1_6,sup1_8,sup1_12 > gpurun_out/vgg16_proxy_fp16.json 2> gpurun_out/vgg16_fp16.err
