mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ring_schedule or wide_levels or random_shapes" > gpurun_out/cw_tests.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline --no-provenance --dtype i64 --moebius-kernel ringcw --ring-debug 8 --scale 0.0625 > gpurun_out/cw2_ringcw.log 2>&1
for dt in i64 f64; do
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-provenance --dtype $dt --moebius-kernel ringcw > gpurun_out/cw2_full_$dt.log 2>&1
done
