set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r8_sweep.log 2>&1
for v in 0 1 2; do
timeout 300 python bench.py --config C5w --steps 3 --warmup 3 --scale 0.25 --no-cpu-baseline --no-e2e --gather-variant $v > gpurun_out/r8_bench_gv$v.log 2>&1
done
timeout 300 python bench.py --config C4w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r8_bench_C4w.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r8_gpu_tests.log
echo done
