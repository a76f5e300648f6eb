mkdir -p gpurun_out
for c in C3w C4w C2 ER4 ER6; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-provenance 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$c moeb %.3f gather %.3f step %.3f rt %s' % (k['moebius_solve']['ms_per_call'], k['gather']['ms_per_call'], d['ms_per_step'], d['round_trip_exact']))"
done

