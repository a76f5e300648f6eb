set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r70_gpu_tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r70_bench.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --moebius-kernel ringcl > gpurun_out/r70_bench_cl.log 2>&1
echo done
