"""Tuning sweep (not a test): RING Möbius lanes-per-element on a workload."""
import sys, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2211_13706_b200 as pz
import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5w"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0625
wl = W.make_workload(cfg, scale)
P = pz.Poset(wl.n, wl.src, wl.dst)
info = P.info()
x = torch.from_numpy(wl.values(seed=1)).cuda()
g = P.zeta(x)
y = torch.empty_like(x)
res = {"cfg": cfg, "n": wl.n, "k": info["k"], "ell": info["ell"], "reach": info["reach"]}
for lpe in (1, 2, 4, 8, 16):
    try:
        P.set_option("ring_lpe", lpe)
    except pz.PosetError as e:
        continue
    P.moebius(g, out=y); torch.cuda.synchronize()
    P.set_option("profile", 1); P.profile_read()
    for _ in range(3):
        P.moebius(g, out=y)
    prof, _ = P.profile_read(); P.set_option("profile", 0)
    ms = prof["moebius_solve"][0] / 3
    res[f"lpe{lpe}_ms"] = ms
    res[f"lpe{lpe}_clk_per_level"] = ms * 1e-3 * 1.965e9 / info["ell"]
print(json.dumps(res))
