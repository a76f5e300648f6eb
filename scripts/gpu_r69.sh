set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r69_gpu_tests.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/r69_bench.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --moebius-kernel ringcl > gpurun_out/r69_bench_cl.log 2>&1
echo done
