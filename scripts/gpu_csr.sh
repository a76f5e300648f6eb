mkdir -p gpurun_out
for c in C3w C4w C2 ER4 ER6; do
  timeout 300 python bench.py --config $c --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-provenance 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']; print('$c moeb %.3f gather %.3f step %.3f rt %s' % (k['moebius_solve']['ms_per_call'], k['gather']['ms_per_call'], d['ms_per_step'], d['round_trip_exact']))"
done
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "C2 or sparse or boolean or int64_zeta or fp64 or edge or ragged or full_size" > gpurun_out/csr_tests.log 2>&1
