set -x; mkdir -p gpurun_out
S="python bench.py --config C5w --scale 0.0625 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --moebius-kernel ringcl"
timeout 300 $S > gpurun_out/r97_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_moeb_ringcl" -c 1 -o gpurun_out/r97_prof $S > gpurun_out/r97_ncu.log 2>&1
echo done
