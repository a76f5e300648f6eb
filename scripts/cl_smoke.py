"""RINGCL first light: small posets, int64 round trip against AUTO (tuning aid)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_13706_b200 as pz
import workloads as W
out = {}
for n, B in ((2000, 1), (20000, 3), (200000, 32)):
    src, dst = W.window_dag(n, 2, 64, 3, forced=True)
    P = pz.Poset(n, src, dst)
    info = P.info()
    x = torch.from_numpy(W.int_values(n, B, -1000, 1000, seed=1)).cuda()
    g = P.zeta(x)
    P.set_option("moebius_kernel", pz.MOEB_RINGDF)
    y0 = P.moebius(g)
    P.set_option("moebius_kernel", pz.MOEB_RINGCL)
    y1 = P.moebius(g); torch.cuda.synchronize()
    out[f"{n}x{B}"] = {"ringdf": info["ringdf"], "df_ok": bool((y0 == x).all()), "cl_ok": bool((y1 == x).all()),
                       "cl_bad": int((y1 != x).sum())}
    print(json.dumps(out), flush=True)
