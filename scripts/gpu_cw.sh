# RINGCW bring-up: parity on the ring tests, then C5w Möbius times (CW vs CL)
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ring_schedule or wide_levels or int64_zeta or example" > gpurun_out/cw_tests.log 2>&1
for k in ringcw ringcl; do
  for dt in i64 f64; do
    echo "== $k $dt"
    timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --no-provenance --dtype $dt --moebius-kernel $k 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']['moebius_solve']; print('moebius ms %.3f  step %.3f cyc/level %.1f' % (k['ms_per_call'], d['ms_per_step'], d['roofline'].get('latency',{}).get('cycles_per_level',0)))
    elif 'Error' in l or 'error' in l: print(l.strip())"
  done
done > gpurun_out/cw_bench.log 2>&1
