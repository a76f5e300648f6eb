set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r9_sweep.log 2>&1
S="python bench.py --config C5w --steps 2 --warmup 1 --scale 0.0625 --no-cpu-baseline --no-e2e"
timeout 300 $S > gpurun_out/r9_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_r4" -c 1 -o gpurun_out/r9_prof $S > gpurun_out/r9_ncu.log 2>&1
echo done
