set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r12_sweep.log 2>&1
for c in C4w C3w C2; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r12_bench_$c.log 2>&1
done
echo done
