"""Tuning aid (not a test): RINGDF cycles per level on C5w (scaled), its
instrumented breakdown and the sum-skipping timing experiments, plus an int64
round-trip check of the default schedule."""
import sys, json, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2211_13706_b200 as pz
import workloads as W

cfg = sys.argv[1] if len(sys.argv) > 1 else "C5w"
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0625
wl = W.make_workload(cfg, scale)
P = pz.Poset(wl.n, wl.src, wl.dst)
info = P.info()
res = {"cfg": cfg, "n": wl.n, "k": info["k"], "ell": info["ell"], "reach": info["reach"],
       "moebius_kernel": info["moebius_kernel"]}
x = torch.from_numpy(wl.values(seed=1)).cuda()
g = P.zeta(x)
y = torch.empty_like(x)


def clk(kern):
    P.set_option("moebius_kernel", kern)
    P.moebius(g, out=y); torch.cuda.synchronize()
    P.set_option("profile", 1); P.profile_read()
    for _ in range(3):
        P.moebius(g, out=y)
    prof, _ = P.profile_read(); P.set_option("profile", 0)
    return prof["moebius_solve"][0] / 3 * 1e-3 * 1.965e9 / info["ell"]


res["ringdf_clk"] = clk(pz.MOEB_RINGDF)
if info["ringdf"] & 2:
    res["ringcl_clk"] = clk(pz.MOEB_RINGCL)
    for nh in (1, 2, 3):
        P.set_option("ringcl_helpers", nh)
        res[f"ringcl_h{nh}_clk"] = clk(pz.MOEB_RINGCL)
    P.set_option("ringcl_helpers", 0)
    P.set_option("ring_debug", 8)
    P.moebius(g, out=y); torch.cuda.synchronize()
    d = P.debug_read()
    lv, hl = max(1, int(d[3])), max(1, int(d[6]))
    res["ringcl_prof"] = {"owner_farbar_wait": d[0] / lv, "owner_near_wait": d[1] / lv, "owner_L7pub_to_far_ready": d[2] / lv,
                          "helper_lvl_waits": d[4] / hl, "helper_far_sum_send": d[5] / hl, "helper_far_sum_only": d[7] / hl, "levels": lv}
    P.set_option("ring_debug", 8 + 32)   # bit 5 (skip_far & 2): rows awaited before the waits
    P.moebius(g, out=y); torch.cuda.synchronize()
    d = P.debug_read()
    lv, hl = max(1, int(d[3])), max(1, int(d[6]))
    res["ringcl_prof_rowsfirst"] = {"helper_lvl_waits": d[4] / hl, "helper_far_sum_send": d[5] / hl,
                                    "helper_far_sum_only": d[7] / hl}
    P.set_option("ring_debug", 8 + 64)   # bit 6 (skip_far & 4): time a second far sum
    P.moebius(g, out=y); torch.cuda.synchronize()
    d = P.debug_read()
    hl = max(1, int(d[6]))
    res["ringcl_prof_second_sum"] = {"helper_far_sum_only": d[7] / hl}
    P.set_option("ring_debug", 16)
    res["ringcl_nofar_clk"] = clk(pz.MOEB_RINGCL)
    P.set_option("ring_debug", 24)
    P.moebius(g, out=y); torch.cuda.synchronize()
    d = P.debug_read()
    lv, hl = max(1, int(d[3])), max(1, int(d[6]))
    res["ringcl_nofar_prof"] = {"owner_farbar_wait": d[0] / lv, "owner_near_wait": d[1] / lv, "owner_L7pub_to_far_ready": d[2] / lv,
                          "helper_lvl_waits": d[4] / hl, "helper_far_sum_send": d[5] / hl}
    P.set_option("ring_debug", 0)
    xi = torch.from_numpy(W.int_values(wl.n, 4, -1000, 1000, seed=5)).cuda()
    P.set_option("moebius_kernel", pz.MOEB_RINGCL)
    res["ok_roundtrip_i64_ringcl"] = bool((P.moebius(P.zeta(xi)) == xi).all())
res["ringdf_fp64_maxerr_vs_input"] = float((y - x).abs().max())
P.set_option("ring_debug", 8)
P.moebius(g, out=y); torch.cuda.synchronize()
d = P.debug_read()
lv = max(1, int(d[4]))
res["ringdf_prof"] = {"ready_to_publish": d[0] / lv, "publish_to_ready_when_waiting": d[1] / max(1, lv - d[3]),
                      "late_levels_frac": d[3] / lv, "lateness_when_late": d[2] / max(1, d[3]),
                      "ready_to_before_arrive": d[5] / lv, "avg_passes": d[6] / lv, "ready_to_near_sum": d[7] / lv}
for bits, name in ((16, "nofar"), (48, "nofar_nomid"), (112, "nofar_nomid_nonear")):
    P.set_option("ring_debug", bits)
    res[f"ringdf_{name}_clk"] = clk(pz.MOEB_RINGDF)
P.set_option("ring_debug", 0)
res["ring_lpe8_clk"] = clk(pz.MOEB_RING)
xi = torch.from_numpy(W.int_values(wl.n, 4, -1000, 1000, seed=3)).cuda()
P.set_option("moebius_kernel", pz.MOEB_AUTO)
res["ok_roundtrip_i64"] = bool((P.moebius(P.zeta(xi)) == xi).all())
print(json.dumps(res))
