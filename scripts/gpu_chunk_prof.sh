# per-launch duration and DRAM bytes of a chunked layer (L2 state kept between launches)
export WINO_CHUNK_TB=4
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 120 -c 60 --csv --log-file gpurun_out/chunk_launches.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/chunk_ncu.log 2>&1
unset WINO_CHUNK_TB
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --cache-control none --clock-control none -s 12 -c 8 --csv --log-file gpurun_out/nochunk_launches.csv python bench.py --steps 3 --warmup 3 --no-extras > gpurun_out/nochunk_ncu.log 2>&1
