timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_io" 2>&1 | tail -1
for c in ramp 8; do if [ $c = ramp ]; then unset WINO_HOSTIO_CHUNKS; else export WINO_HOSTIO_CHUNKS=$c; fi; timeout 300 python scripts/time_e2e.py; timeout 300 python scripts/time_e2e.py; done
