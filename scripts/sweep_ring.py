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
P.set_option("moebius_kernel", pz.MOEB_RING)
for lpe in (1, 2, 4, 8):
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
for kern, name in ((pz.MOEB_RINGDF, "ringdf"), (pz.MOEB_RINGWS, "ringws"), (pz.MOEB_RING, "ring_lpe8")):
    if (kern == pz.MOEB_RINGWS and not info["ringws"]) or (kern == pz.MOEB_RINGDF and not info["ringdf"] & 1) \
            or (kern == pz.MOEB_RINGCL and not info["ringdf"] & 2):
        continue
    P.set_option("ring_lpe", 8)
    P.set_option("moebius_kernel", kern)
    P.moebius(g, out=y); torch.cuda.synchronize()
    P.set_option("profile", 1); P.profile_read()
    for _ in range(3):
        P.moebius(g, out=y)
    prof, _ = P.profile_read(); P.set_option("profile", 0)
    ms = prof["moebius_solve"][0] / 3
    res[f"{name}_ms"] = ms
    res[f"{name}_clk_per_level"] = ms * 1e-3 * 1.965e9 / info["ell"]
    if wl.dtype == "i64" or True:
        xb = x if wl.dtype == "i64" else None
if info["ringws"]:
    P.set_option("moebius_kernel", pz.MOEB_RINGWS)
    for nwo in (4, 8, 12):
        for lpeo in (4, 8):
            try:
                P.set_option("ringws_nwo", nwo); P.set_option("ringws_lpeo", lpeo)
            except pz.PosetError:
                continue
            P.moebius(g, out=y); torch.cuda.synchronize()
            P.set_option("profile", 1); P.profile_read()
            for _ in range(3):
                P.moebius(g, out=y)
            prof, _ = P.profile_read(); P.set_option("profile", 0)
            ms = prof["moebius_solve"][0] / 3
            res[f"ws_nwo{nwo}_lpeo{lpeo}_clk"] = ms * 1e-3 * 1.965e9 / info["ell"]
    P.set_option("ringws_nwo", 8); P.set_option("ringws_lpeo", 8)
# experiment: RING lpe 8 without the global store of f (output invalid)
P.set_option("moebius_kernel", pz.MOEB_RING); P.set_option("ring_lpe", 8); P.set_option("ring_debug", 1)
P.moebius(g, out=y); torch.cuda.synchronize()
P.set_option("profile", 1); P.profile_read()
for _ in range(3):
    P.moebius(g, out=y)
prof, _ = P.profile_read(); P.set_option("profile", 0)
res["ring8_nostore_clk"] = prof["moebius_solve"][0] / 3 * 1e-3 * 1.965e9 / info["ell"]
P.set_option("ring_debug", 0)
# int64 data, RING lpe 8
xi = torch.from_numpy(W.int_values(wl.n, wl.batch, -1000, 1000, seed=3)).cuda()
gi = P.zeta(xi); yi = torch.empty_like(gi)
P.moebius(gi, out=yi); torch.cuda.synchronize()
P.set_option("profile", 1); P.profile_read()
for _ in range(3):
    P.moebius(gi, out=yi)
prof, _ = P.profile_read(); P.set_option("profile", 0)
res["ring8_i64_clk"] = prof["moebius_solve"][0] / 3 * 1e-3 * 1.965e9 / info["ell"]
if info["ringdf"]:
    P.set_option("moebius_kernel", pz.MOEB_RINGDF)
    P.set_option("ring_debug", 8)
    P.moebius(g, out=y); torch.cuda.synchronize()
    d = P.debug_read()
    lv = max(1, int(d[4]))
    res["ringdf_prof"] = {"ready_to_publish": d[0] / lv, "publish_to_ready_when_waiting": d[1] / max(1, lv - d[3]),
                          "late_levels_frac": d[3] / lv, "lateness_when_late": d[2] / max(1, d[3]), "levels": lv,
                          "ready_to_before_arrive": d[5] / lv, "avg_passes": d[6] / lv, "ready_to_near_sum": d[7] / lv}
    for bits, name in ((16, "nofar"), (48, "nofar_nomid"), (112, "nofar_nomid_nonear")):
        P.set_option("ring_debug", bits)
        P.moebius(g, out=y); torch.cuda.synchronize()
        P.set_option("profile", 1); P.profile_read()
        for _ in range(3):
            P.moebius(g, out=y)
        prof, _ = P.profile_read(); P.set_option("profile", 0)
        res[f"ringdf_{name}_clk"] = prof["moebius_solve"][0] / 3 * 1e-3 * 1.965e9 / info["ell"]
    P.set_option("ring_debug", 0)
res["ok_roundtrip_i64"] = None
xi = torch.from_numpy(W.int_values(wl.n, 4, -1000, 1000, seed=3)).cuda()
gi = P.zeta(xi)
P.set_option("moebius_kernel", pz.MOEB_AUTO)
res["ok_roundtrip_i64"] = bool(torch.equal(P.moebius(gi), xi))
print(json.dumps(res))
