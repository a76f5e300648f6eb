# per-config bench lines (gpurun): step / Möbius / gather ms per config
for c in ${CONFIGS:-C2 C3w C4w}; do
  echo "== $c ${EXTRA}"
  timeout 400 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline --no-e2e ${EXTRA} 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']
        print('step ms %.3f  ' % d['ms_per_step'] + '  '.join('%s %.3f ms (%.3f)' % (p, v['ms_per_call'], v['frac']) for p, v in k.items()) + '  moebius=%s exact=%s' % (d['config']['moebius_kernel'], d['round_trip_exact']))
    elif 'rror' in l: print(l.rstrip()[:300])"
done
