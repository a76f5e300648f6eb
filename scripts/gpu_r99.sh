set -x; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "wide_levels or ring_schedule" > gpurun_out/r99_tests.log 2>&1
echo done
