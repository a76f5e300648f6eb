# Möbius schedule sweep (gpurun): Möbius ms and cycles/level per schedule / helper count
for m in ${MOEBS:-ringcl ringsq}; do
  for nh in ${NHS:-0}; do
    echo "== $m helpers=$nh ${EXTRA}"
    timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --moebius-kernel $m ${EXTRA} \
        --ringcl-helpers $nh 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']['moebius_solve']; r=d['roofline']
        print('moebius ms %.3f  step ms %.3f  cycles/level %s  exact %s' % (k['ms_per_call'], d['ms_per_step'], (r.get('latency') or {}).get('cycles_per_level'), d['round_trip_exact']))
    elif 'ring_debug' in l or 'rror' in l: print(l.rstrip()[:300])"
  done
done
