"""Multi-GPU plumbing (one process per GPU, torch.distributed over NCCL).

Two ways the hot path shards:

* **Batched functions -> column sharding** (``column_shard``): every rank
  holds the whole poset (replicated index table) and transforms its own
  B_local columns.  No collective on the data path; weak scaling.

* **Single-function zeta -> row sharding** (``row_sharded_zeta``): rank p
  owns the slot range S_p and the rank-row range R_p (equal contiguous
  splits).  It scans S_p (kernel iii, carry-in 0), all-gathers the per-range
  scan tails (G x 2 x B words), combines them into its carry
  (``poset_combine_tails``) and adds it to the rows before its first chain
  start, all-gathers F over NCCL (in place), gathers g for R_p (kernel iv)
  and all-gathers the rank-ordered g, which ``poset_rank_to_user`` scatters
  into user order.

Single-function Möbius is not sharded: its U-solve dependency chain
(depth D_U) does not split across GPUs (north star).

Every arithmetic step runs in libposet.so; this module only sizes ranges and
calls collectives.  ``emulate_row_sharded_zeta`` runs the same sequence of
library calls for G emulated ranks on one GPU (the collectives become
buffer copies), so the split-phase path is testable with one device.
"""
from __future__ import annotations

import math


def shard_range(n: int, world: int, rank: int):
    """Equal contiguous split of [0, n): (lo, hi, chunk)."""
    chunk = max(1, math.ceil(n / world)) if n else 1
    lo = min(n, rank * chunk)
    hi = min(n, lo + chunk)
    return lo, hi, chunk


def column_shard(batch: int, world: int, rank: int):
    """Columns [lo, hi) of a batch of functions owned by ``rank``."""
    per = math.ceil(batch / world)
    lo = min(batch, rank * per)
    return lo, min(batch, lo + per)


def _all_gather(out, inp, group=None):
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_gather_into_tensor(out, inp, group=group)
    else:   # gloo: list form into contiguous row-chunk views of `out`
        dist.all_gather(list(out.chunk(dist.get_world_size(group))), inp.contiguous(), group=group)


def row_sharded_zeta(P, f, group=None, out=None):
    """Single-function (or small-batch) zeta sharded by rows over the
    process group.  ``P``: the rank's Poset (same poset on every rank);
    ``f``: [n][B] on this rank's device (replicated input).  Returns g
    [n][B] (user order) on every rank."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = P.n
    f2 = f.reshape(n, -1)
    B = f2.shape[1]
    lo, hi, chunk = shard_range(n, world, rank)
    dev = f.device
    # F for all slots, padded to world*chunk rows + the zero row n
    F = torch.zeros((world * chunk + 1, B), dtype=f.dtype, device=dev)
    tail = torch.zeros((2, B), dtype=f.dtype, device=dev)
    P.scan_slots(f2, F, tail, lo, hi)
    tails = torch.empty((world, 2, B), dtype=f.dtype, device=dev)
    _all_gather(tails.view(world * 2, B), tail, group)
    carry = torch.zeros((B,), dtype=f.dtype, device=dev)
    P.combine_tails(tails, world, rank, carry)
    P.scan_carry(F, carry, lo, hi)
    _all_gather(F[: world * chunk], F[rank * chunk:(rank + 1) * chunk].clone(), group)
    F[n].zero_()
    g_part = torch.zeros((chunk, B), dtype=f.dtype, device=dev)
    if hi > lo:
        P.gather_rows(F, g_part, lo, hi)
    g_rank = torch.empty((world * chunk, B), dtype=f.dtype, device=dev)
    _all_gather(g_rank, g_part, group)
    if out is None:
        out = torch.empty_like(f2)
    P.rank_to_user(g_rank[:n].contiguous(), out)
    return out.reshape(f.shape)


def shard_index(P, group=None, rank=None, world=None):
    """Keep only this rank's index rows (``poset_shard_rows``): 4·k·n/G bytes
    per rank instead of 4·n·k.  Rank 0 keeps the Möbius
    tables (single-function Möbius runs there); the others drop them."""
    if rank is None or world is None:
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
    lo, hi, _ = shard_range(P.n, world, rank)
    P.shard_rows(lo, hi, drop_moebius=rank != 0)
    return lo, hi


def emulate_row_sharded_zeta(P, f, world: int):
    """The call sequence of ``row_sharded_zeta`` for ``world`` emulated ranks
    on one GPU; each collective becomes a copy.  For tests only -- no kernel
    waits on another.  ``P`` is one handle for every rank, or a list of
    ``world`` handles of the same poset (e.g. each with its rows sharded by
    ``shard_index``): rank p's calls then go to ``P[p]``."""
    import torch
    Ps = list(P) if isinstance(P, (list, tuple)) else [P] * world
    P = Ps[0]
    n = P.n
    f2 = f.reshape(n, -1)
    B = f2.shape[1]
    chunk = shard_range(n, world, 0)[2]
    F = torch.zeros((world * chunk + 1, B), dtype=f.dtype, device=f.device)
    tails = torch.zeros((world, 2, B), dtype=f.dtype, device=f.device)
    for p in range(world):
        lo, hi, _ = shard_range(n, world, p)
        Ps[p].scan_slots(f2, F, tails[p], lo, hi)
    for p in range(world):
        lo, hi, _ = shard_range(n, world, p)
        carry = torch.zeros((B,), dtype=f.dtype, device=f.device)
        Ps[p].combine_tails(tails, world, p, carry)
        Ps[p].scan_carry(F, carry, lo, hi)
    F[n].zero_()
    g_rank = torch.zeros((world * chunk, B), dtype=f.dtype, device=f.device)
    for p in range(world):
        lo, hi, _ = shard_range(n, world, p)
        if hi > lo:
            part = torch.zeros((chunk, B), dtype=f.dtype, device=f.device)
            Ps[p].gather_rows(F, part, lo, hi)
            g_rank[p * chunk:(p + 1) * chunk] = part
    out = torch.empty_like(f2)
    P.rank_to_user(g_rank[:n].contiguous(), out)
    return out.reshape(f.shape)


def nvls_buffer_bytes(n: int, world: int, batch: int) -> int:
    """Bytes of the F buffer ``nvls_row_sharded_zeta`` views: world·chunk + 1
    rows (the zero row n) of ``batch`` 8-byte values."""
    chunk = shard_range(n, world, 0)[2]
    return (world * chunk + 1) * batch * 8


def nvls_row_sharded_zeta(Ps, fs, buf, out=None):
    """Row-sharded zeta with the all-gather of F fused into the scan (SURVEY
    §8(f) N3): "rank" p -- handle ``Ps[p]``, replicated input ``fs[p]`` on
    its device -- scans its slot range with ``poset_scan_slots_mc``, whose
    every F row goes through the NVLS multicast address ``buf.mc`` and so
    lands on every device bound to ``buf`` (no F all-gather follows).  Each
    device then applies every range's carry (``poset_combine_tails`` over the
    per-range scan tails, then ``poset_scan_carry``; only the rows before a
    range's first chain start change) to its own copy, zeroes row n, and rank
    p gathers its rank rows [lo_p, hi_p) (kernel iv).  g is assembled in user
    order on ``fs[0]``'s device.

    One process drives all ranks: ``buf.devices`` lists one device per rank
    (multi-GPU), or one device for all ranks (emulated ranks sharing one F,
    the 1-GPU test).  Cross-process sharing of the multicast object (one
    process per GPU) is not built (include/poset.h)."""
    import torch
    world = len(Ps)
    P0 = Ps[0]
    n = P0.n
    B = fs[0].reshape(n, -1).shape[1]
    dt = fs[0].dtype
    chunk = shard_range(n, world, 0)[2]
    shared = len(buf.devices) == 1
    if not shared and len(buf.devices) != world:
        raise ValueError("buf.devices: one device per rank, or one device for all ranks")
    bidx = [0 if shared else p for p in range(world)]
    Fs = {d: buf.tensor(d, (world * chunk + 1, B), dt) for d in sorted(set(bidx))}
    tails = []
    for p in range(world):
        lo, hi, _ = shard_range(n, world, p)
        f2 = fs[p].reshape(n, -1)
        tail = torch.zeros((2, B), dtype=dt, device=f2.device)
        Ps[p].scan_slots_mc(f2, buf.mc, tail, lo, hi)
        tails.append(tail)
    for d in buf.devices:   # every rank's multicast stores have landed everywhere
        torch.cuda.synchronize(d)
    for d, F in Fs.items():
        Pd = Ps[bidx.index(d)]
        tails_all = torch.stack([t.to(F.device) for t in tails]).contiguous()
        for p in range(world):
            lo, hi, _ = shard_range(n, world, p)
            carry = torch.zeros((B,), dtype=dt, device=F.device)
            Pd.combine_tails(tails_all, world, p, carry)
            Pd.scan_carry(F, carry, lo, hi)
        F[n].zero_()
    dev0 = fs[0].device
    g_rank = torch.zeros((world * chunk, B), dtype=dt, device=dev0)
    for p in range(world):
        lo, hi, _ = shard_range(n, world, p)
        if hi > lo:
            F = Fs[bidx[p]]
            part = torch.zeros((chunk, B), dtype=dt, device=F.device)
            Ps[p].gather_rows(F, part, lo, hi)
            g_rank[p * chunk:(p + 1) * chunk] = part.to(dev0)
    if out is None:
        out = torch.empty((n, B), dtype=dt, device=dev0)
    P0.rank_to_user(g_rank[:n].contiguous(), out)
    return out.reshape(fs[0].shape)
