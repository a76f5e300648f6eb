mkdir -p gpurun_out
python - <<'PY' > gpurun_out/chunk_plan.log 2>&1
import workloads as W, paper_2211_13706_b200 as pz
wl=W.make_workload("C5w", scale=0.0625); P=pz.Poset(wl.n, wl.src, wl.dst); print(P.info())
PY
for dt in f64 i64; do for ch in 0 32 64 128 256; do
timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --no-provenance --dtype $dt --ringcl-chunk $ch 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); k=d['kernels']['moebius_solve']; print('$dt ch=$ch moebius ms %.3f step %.3f rt %s' % (k['ms_per_call'], d['ms_per_step'], d['round_trip_exact']))
    elif 'rror' in l: print('$dt ch=$ch', l.strip()[:200])"
done; done > gpurun_out/chunk.log 2>&1
