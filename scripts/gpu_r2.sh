set -x; mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r2_gpu_tests.log
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2_bench.log 2>&1
tail -c 600 gpurun_out/r2_bench.log
S="python bench.py --steps 2 --warmup 1 --scale 0.0625 --no-cpu-baseline --no-e2e"
timeout 300 $S > gpurun_out/r2_plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches.csv $S > gpurun_out/r2_ncu.log 2>&1
echo done
