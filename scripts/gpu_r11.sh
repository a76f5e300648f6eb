set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r11_sweep.log 2>&1
echo done
