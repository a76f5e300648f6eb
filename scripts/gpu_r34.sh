set -x; mkdir -p gpurun_out
for c in C3w C4w C2; do
  timeout 300 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r34_bench_$c.log 2>&1
done
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r34_gpu_tests.log
echo done
