set -x; mkdir -p gpurun_out
S="python bench.py --config C5w --steps 2 --warmup 1 --scale 0.0625 --no-cpu-baseline --no-e2e"
timeout 300 $S > gpurun_out/r3b_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_cols|k_moeb_ring" -c 2 -o gpurun_out/r3_prof $S > gpurun_out/r3b_ncu.log 2>&1
echo done
