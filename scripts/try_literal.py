"""Literal C3 / C4 through the sparse-rows path (N1): setup time, nnz, one
zeta + Möbius round trip at B=1 (int64), sampled zeta rows vs the DFS
checker.  Used for the round-2 measurements (gpurun)."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import paper_2211_13706_b200 as pz  # noqa: E402
import workloads as W  # noqa: E402
from oracle.chain import zeta_sampled_edges  # noqa: E402

name = sys.argv[1]
scale = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
wl = W.make_workload(name, scale, dtype="i64", batch=1)
t0 = time.time()
try:
    P = pz.Poset(wl.n, wl.src, wl.dst)
except pz.PosetError as e:
    print(f"{name} n={wl.n}: {e.code} after {time.time() - t0:.1f} s: {e}", flush=True)
    sys.exit(0)
t1 = time.time()
info = P.info()
print(f"{name} n={wl.n} k={info['k']} ell={info['ell']} nnz={info['nnz']} csr_bytes={info['csr_bytes'] / 1e9:.2f} GB "
      f"zeta_sparse={info['zeta_sparse']} setup {t1 - t0:.1f} s (rows {info['t_mtable']:.1f} s)", flush=True)
import torch  # noqa: E402
f = wl.values(seed=1)
x = torch.from_numpy(f).cuda()
torch.cuda.synchronize()
t2 = time.time()
g = P.zeta(x)
torch.cuda.synchronize()
t3 = time.time()
back = P.moebius(g)
torch.cuda.synchronize()
t4 = time.time()
print(f"zeta {1e3 * (t3 - t2):.1f} ms  moebius {1e3 * (t4 - t3):.1f} ms  round trip exact: "
      f"{bool(torch.equal(back, x))}", flush=True)
rng = np.random.default_rng(0)
xs = np.unique(rng.integers(0, wl.n, 8))
want, _ = zeta_sampled_edges(wl.n, wl.src, wl.dst, f, xs)
print("sampled zeta rows match:", bool((g.cpu().numpy()[xs] == want).all()), flush=True)
