set -x; mkdir -p gpurun_out
for v in 0 3; do
timeout 300 python bench.py --config C5w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --gather-variant $v > gpurun_out/r39_bench_gv$v.log 2>&1
timeout 300 python bench.py --config C4w --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --gather-variant $v > gpurun_out/r39_bench_C4w_gv$v.log 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "gather" 2>&1 | tail -3 > gpurun_out/r39_gpu_tests.log
echo done
