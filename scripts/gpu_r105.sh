set -x; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r105_gpu.txt
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r105_gpu_tests.log 2>&1
timeout 900 python bench.py > gpurun_out/r105_bench_default.log 2>&1
for c in C1 C2 C3w C4w; do
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r105_bench_$c.log 2>&1
done
timeout 400 python bench.py --config C5w --dtype i64 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r105_bench_C5w_i64.log 2>&1
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r105_bench_reference.log 2>&1
S="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e"
timeout 600 $S > gpurun_out/r105_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r105_launches.csv $S > gpurun_out/r105_ncu_launch.log 2>&1 && \
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"k_moeb_ringcl|k_gather_r4|k_scan_tiles|k_to_rank_major" -c 5 -o gpurun_out/r105_full $S > gpurun_out/r105_ncu_full.log 2>&1
echo done
