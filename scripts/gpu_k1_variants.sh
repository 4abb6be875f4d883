# time K1 for each scripts/variants/libwino_*.so (swapped in place), then restore;
# parity subset with the first variant
cp paper_1905_05233_b200/libwino.so /tmp/libwino_orig.so
for v in "$@"; do
  cp scripts/variants/libwino_$v.so paper_1905_05233_b200/libwino.so
  for a in lin4 lin3 lin2 sup1_4; do echo "$v $(timeout 120 python scripts/time_k1.py $a bf16 2>&1 | tail -1)"; done
done
cp scripts/variants/libwino_$1.so paper_1905_05233_b200/libwino.so
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "input_transform or layer" 2>&1 | tail -1
cp /tmp/libwino_orig.so paper_1905_05233_b200/libwino.so
