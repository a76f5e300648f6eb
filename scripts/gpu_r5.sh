set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r5_sweep.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r5_gpu_tests.log
for c in C5w C4w C3w C2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r5_bench_$c.log 2>&1
done
echo done
