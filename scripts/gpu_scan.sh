mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "scan_modes" > gpurun_out/scan_tests.log 2>&1
for c in "C5w --dtype f64" "C5w --dtype i64" "C4w" "C3w"; do for m in 2 1; do
timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-provenance --scan-mode $m 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$c mode=$m scan %.3f frac %.3f step %.3f' % (k['scan']['ms_per_call'], k['scan']['frac'], d['ms_per_step']))
    elif 'rror' in l: print('$c $m', l.strip()[:200])"
done; done > gpurun_out/scan.log 2>&1
