set -x; mkdir -p gpurun_out
timeout 120 python scripts/cl_smoke.py > gpurun_out/r95_smoke.log 2>&1 || exit 1
timeout 300 python scripts/sweep_ringdf.py C5w 0.0625 > gpurun_out/r95_sweep.log 2>&1
echo done
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r95_bench.log 2>&1
