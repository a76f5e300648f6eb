mkdir -p gpurun_out
for dt in f64 i64; do for nh in 2 3 2 3; do
timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-provenance --dtype $dt --ringcl-helpers $nh 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']['moebius_solve']; print('$dt nh=$nh moebius ms %.3f step %.3f' % (k['ms_per_call'], d['ms_per_step']))"
done; done > gpurun_out/nh.log 2>&1
