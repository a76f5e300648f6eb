set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ring.py C5w 0.0625 > gpurun_out/r6_sweep.log 2>&1
for c in C5w C4w C3w C2; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r6_bench_$c.log 2>&1
done
S="python bench.py --config C5w --steps 2 --warmup 1 --scale 0.0625 --no-cpu-baseline --no-e2e"
timeout 300 $S > gpurun_out/r6_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gather_cols|k_moeb_ring" -c 2 -o gpurun_out/r6_prof $S > gpurun_out/r6_ncu.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/r6_gpu_tests.log
echo done
