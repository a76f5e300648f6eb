set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ringdf.py C5w 0.0625 > gpurun_out/r50_sweep.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r50_gpu_tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r50_bench.log 2>&1
echo done
