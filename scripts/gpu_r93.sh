set -x; mkdir -p gpurun_out
timeout 120 python scripts/cl_smoke.py > gpurun_out/r93_smoke.log 2>&1 || exit 1
timeout 300 python scripts/sweep_ringdf.py C5w 0.0625 > gpurun_out/r93_sweep.log 2>&1
echo done
