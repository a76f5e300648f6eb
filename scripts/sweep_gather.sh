# gather kernel sweep (gpurun): one bench line per configuration, gather ms only.
# SWEEP: tokens pi<N> (--gather-pi-cfg N) or var<N> (--gather-variant N)
for tok in ${SWEEP:-var4 pi0 pi1 pi2 pi3}; do
  case $tok in pi*) a="--gather-pi-cfg ${tok#pi}";; var*) a="--gather-variant ${tok#var}";; esac
  for dt in ${DTYPES:-f64 i64}; do
    echo "== $a $dt ${EXTRA}"
    timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --dtype $dt $a ${EXTRA} | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']['gather']; print('gather ms %.3f frac %.3f' % (k['ms_per_call'], k['frac']))"
  done
done
