set -x; mkdir -p gpurun_out
timeout 300 python scripts/sweep_ringdf.py C5w 0.0625 > gpurun_out/r104_sweep.log 2>&1
for h in 1 2 3; do
python - <<PY > gpurun_out/r104_full_h$h.log 2>&1
import sys, json, torch
sys.path.insert(0, '.')
import paper_2211_13706_b200 as pz, workloads as W
wl = W.make_workload("C5w", 1.0)
P = pz.Poset(wl.n, wl.src, wl.dst)
x = torch.from_numpy(wl.values(seed=1)).cuda(); g = P.zeta(x); y = torch.empty_like(x)
P.set_option("ringcl_helpers", $h)
P.moebius(g, out=y); torch.cuda.synchronize()
P.set_option("profile", 1); P.profile_read()
for _ in range(3): P.moebius(g, out=y)
prof, _ = P.profile_read()
print(json.dumps({"h": $h, "moebius_ms": prof["moebius_solve"][0] / 3, "info_ell": P.info()["ell"], "wmax": P.info()["max_level_width"]}))
PY
done
echo done
