"""Multi-GPU (NCCL, one process per GPU) runs of the sharded paths through
the real library: row-sharded single-function zeta
(dist.row_sharded_zeta: split-phase kernels + NCCL all-gathers of the scan
tails, F and g) and column-sharded batched zeta / Möbius, each compared with
O2 element by element on every rank.  Skipped with fewer than 2 GPUs (the
round-end GPU box has one); the same choreography runs on CPU in
test_dist_gloo.py."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available() or torch.cuda.device_count() < 2:   # pragma: no cover
    pytest.skip("needs >= 2 CUDA devices", allow_module_level=True)

import workloads as W  # noqa: E402


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import paper_2211_13706_b200 as pz
    from paper_2211_13706_b200 import dist as pdist
    from oracle.chain import ChainOracle
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
        n = 30000
        src, dst = W.window_dag(n, 2, 1000, 0, forced=True)
        P = pz.Poset(n, src, dst, device=rank)
        O = ChainOracle(n, src, dst)
        ok = True
        # single function: rows sharded, NCCL all-gathers
        for f in (W.int_values(n, 1, -10**15, 10**15, seed=3), W.int_values(n, 3, -1000, 1000, seed=4)):
            g = pdist.row_sharded_zeta(P, torch.from_numpy(f).cuda())
            torch.cuda.synchronize()
            ok &= bool((g.cpu().numpy() == O.zeta(f)).all())
        # batched: columns sharded, no collective on the data path
        B = 64
        f = W.int_values(n, B, -10**15, 10**15, seed=5)
        lo, hi = pdist.column_shard(B, world, rank)
        x = torch.from_numpy(np.ascontiguousarray(f[:, lo:hi])).cuda()
        g = P.zeta(x)
        back = P.moebius(g)
        torch.cuda.synchronize()
        ok &= bool((g.cpu().numpy() == O.zeta(f)[:, lo:hi]).all()) and bool(torch.equal(back, x))
        # the row-sharded index: each rank keeps only its rows, same result
        pdist.shard_index(P)
        f = W.int_values(n, 2, -10**15, 10**15, seed=6)
        g = pdist.row_sharded_zeta(P, torch.from_numpy(f).cuda())
        torch.cuda.synchronize()
        ok &= bool((g.cpu().numpy() == O.zeta(f)).all())
        dist.destroy_process_group()
        q.put((rank, ok, ""))
    except Exception as e:   # pragma: no cover
        q.put((rank, False, repr(e)))


def test_nccl_row_and_column_sharding():
    import torch.multiprocessing as mp
    world = min(torch.cuda.device_count(), 4)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert all(ok for _, ok, _ in res), res
