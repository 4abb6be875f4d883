# chunked K3 -> K4 (L2-resident M slices): parity test + bench per slice size
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "chunked or fused or layer" > gpurun_out/gpu_tests.log 2>&1; tail -1 gpurun_out/gpu_tests.log
for c in none 2 3 4 6 8 12; do
  if [ $c = none ]; then unset WINO_CHUNK_TB; else export WINO_CHUNK_TB=$c; fi
  echo "chunk=$c $(timeout 300 python bench.py --steps 50 --warmup 5 --sweep off --no-extras 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['value'], d['gpu_launches'])")"
done
unset WINO_CHUNK_TB
