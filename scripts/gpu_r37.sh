set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r37_sweep.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "ring or example or int64_zeta or full_size" 2>&1 | tail -5 > gpurun_out/r37_gpu_tests.log
echo done
