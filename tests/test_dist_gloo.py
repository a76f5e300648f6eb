"""Multi-process (world size 2, gloo, CPU) coverage of the sharded paths of
``paper_2211_13706_b200/dist.py``.

There is no GPU here, so the per-rank compute calls go to a CPU stand-in
with the same interface as ``Poset``'s split-phase methods.  The stand-in
takes the library's own host-side layout (``poset_analyze``: chains,
bottom-up positions, levels -> ranks and slots) and implements each phase's
contract from ``include/poset.h`` literally with down-sets from oracle O1.
What is under test is the distributed choreography: range splitting, the
all-gather of scan tails and their combination into carries, the all-gather
of F, the row-range gathers and the final all-gather + scatter -- it must
reproduce g = Z f exactly (int64) on every rank.  The kernels behind the same
calls are parity-tested on the GPU (test_gpu_parity.py, split-phase test).
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import workloads as W  # noqa: E402

try:
    import paper_2211_13706_b200 as pz
    from paper_2211_13706_b200 import dist as pdist
except ImportError:   # pragma: no cover - the library must be built
    pz = None


class HostSplitPhases:
    """CPU stand-in for the split-phase calls of one rank (contract of
    poset_scan_slots / poset_combine_tails / poset_scan_carry /
    poset_gather_rows / poset_rank_to_user in include/poset.h)."""

    def __init__(self, n, src, dst):
        from oracle import brute
        info, chain, pos, level = pz.analyze(n, src, dst, want_chains=True)
        self.n = n
        k = info["k"]
        rank_user = np.lexsort((np.arange(n), level))          # level order, ties by id
        self.rank_user = rank_user
        lens = np.bincount(chain, minlength=k)
        off = np.concatenate([[0], np.cumsum(lens)])
        slot = off[chain] + pos                                  # per user vertex
        self.slot_user = np.empty(n, np.int64)
        self.slot_user[slot] = np.arange(n)
        self.start = np.zeros(n, bool)
        self.start[slot[pos == 0]] = True
        down = brute.downsets(n, src, dst)
        # m(x, j) as a global slot (or -1): highest chain-j member of ↓x
        self.m = np.full((n, k), -1, np.int64)
        for x in range(n):
            mem = brute._bits(down[x], n)
            for y in mem:
                j = chain[y]
                self.m[x, j] = max(self.m[x, j], slot[y])

    def scan_slots(self, f, F, tail, lo, hi):
        f, F, tail = f.numpy(), F.numpy(), tail.numpy()
        run = np.zeros(f.shape[1], f.dtype)
        flag = 0
        for s in range(lo, hi):
            if self.start[s]:
                run = np.zeros_like(run)
                flag = 1
            run = run + f[self.slot_user[s]]
            F[s] = run
        tail[0] = flag
        tail[1] = run

    def combine_tails(self, tails, world, rank, carry):
        tails, carry = tails.numpy(), carry.numpy()
        run = np.zeros_like(carry)
        for p in range(rank):
            run = tails[p, 1] if tails[p, 0, 0] else run + tails[p, 1]
        carry[:] = run

    def scan_carry(self, F, carry, lo, hi):
        F, carry = F.numpy(), carry.numpy()
        for s in range(lo, hi):
            if self.start[s]:
                break
            F[s] += carry

    def gather_rows(self, F, g_part, lo, hi):
        F, g_part = F.numpy(), g_part.numpy()
        for r in range(lo, hi):
            x = self.rank_user[r]
            acc = np.zeros(F.shape[1], F.dtype)
            for s in self.m[x]:
                if s >= 0:
                    acc = acc + F[s]
            g_part[r - lo] = acc

    def rank_to_user(self, g_rank, out):
        g_rank, out = g_rank.numpy(), out.numpy()
        out[self.rank_user] = g_rank


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, case, q):
    import torch.distributed as dist
    from oracle.chain import ChainOracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, src, dst = case
        P = HostSplitPhases(n, src, dst)
        f = W.int_values(n, 3, -1000, 1000, seed=11)            # replicated input
        g = pdist.row_sharded_zeta(P, torch.from_numpy(f))
        ok = bool((g.numpy() == ChainOracle(n, src, dst).zeta(f)).all())
        lo, hi = pdist.column_shard(8, world, rank)
        q.put((rank, ok, (lo, hi)))
    finally:
        dist.destroy_process_group()


@pytest.mark.skipif(pz is None, reason="libposet.so not built")
@pytest.mark.parametrize("name", ["paper12", "window300", "layered"])
def test_row_sharded_zeta_world2_gloo(name):
    cases = {
        "paper12": (12, *W.paper_example_edges()),
        "window300": (300, *W.window_dag(300, 2, 64, 0, forced=True)),
        "layered": (8 * 16, *W.layered_dag(8, 16, 3, 1)),
    }
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, cases[name], q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    res.sort()
    assert all(ok for _, ok, _ in res)
    # column shards of a batch of 8 partition it
    assert [c for _, _, c in res] == [(0, 4), (4, 8)]


def test_shard_ranges_partition():
    if pz is None:
        pytest.skip("libposet.so not built")
    for n in (0, 1, 7, 100, 101):
        for world in (1, 2, 3, 8):
            got = [pdist.shard_range(n, world, r)[:2] for r in range(world)]
            assert got[0][0] == 0 and got[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(got, got[1:]))
            cols = [pdist.column_shard(n, world, r) for r in range(world)]
            assert cols[0][0] == 0 and cols[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(cols, cols[1:]))
