set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/r1_gpu_tests.log
timeout 600 python bench.py --steps 3 --warmup 3 --scale 0.0625 --no-cpu-baseline > gpurun_out/r1_bench_small.log 2>&1
timeout 1200 python bench.py --steps 5 --warmup 3 > gpurun_out/r1_bench.log 2>&1
echo done
