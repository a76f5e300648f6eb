mkdir -p gpurun_out
for rd in 8 40 72 104; do
timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-provenance --dtype i64 --moebius-kernel ringcw --ring-debug $rd --scale 0.0625 > gpurun_out/cw2_rd$rd.log 2>&1
done
