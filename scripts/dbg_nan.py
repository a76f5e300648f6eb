import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np
import paper_2211_13706_b200 as pz
import workloads as W
wl = W.make_workload("C5w", 0.0625)
P = pz.Poset(wl.n, wl.src, wl.dst)
x = torch.from_numpy(wl.values(seed=1)).cuda()
g = P.zeta(x)
out = {"g_nan": int(torch.isnan(g).sum())}
for kern, name in ((pz.MOEB_RINGDF, "ringdf"), (pz.MOEB_RING, "ring"), (pz.MOEB_RINGWS, "ringws")):
    P.set_option("moebius_kernel", kern)
    y = torch.full_like(x, float("nan"))
    P.moebius(g, out=y); torch.cuda.synchronize()
    bad = torch.isnan(y) | ((y - x).abs() > 1e-6)
    rows = torch.nonzero(bad.any(1)).flatten()
    cols = torch.nonzero(bad.any(0)).flatten()
    out[name] = {"bad": int(bad.sum()), "nan": int(torch.isnan(y).sum()), "rows": rows[:20].tolist(), "nrows": int(rows.numel()),
                 "cols": cols.tolist(), "maxerr": float((y - x).abs().nan_to_num(1e300).max())}
    y2 = P.moebius(g); torch.cuda.synchronize()
    out[name]["alloc_out_bad"] = int((torch.isnan(y2) | ((y2 - x).abs() > 1e-6)).sum())
# int64 B=32
xi = torch.from_numpy(W.int_values(wl.n, 32, -1000, 1000, seed=3)).cuda()
P.set_option("moebius_kernel", pz.MOEB_AUTO)
gi = P.zeta(xi)
out["i64_B32_bad"] = int((P.moebius(gi) != xi).sum())
print(json.dumps(out))
