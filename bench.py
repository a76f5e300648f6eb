#!/usr/bin/env python
"""Benchmark: zeta + Möbius round trip (one "step" = kernels iii, iv, v and
the chain difference over one batch) on the BASELINE.json metric
"zeta/Möbius n·k gathers/s and HBM GB/s vs peak, at 1/2/4/8 B200".

    python bench.py [--gpus N --steps K --warmup W] [--config C5w] [--impl ours|reference]

* Workload (default): C5w = BASELINE.json configs[4] (n=16M random window DAG,
  W=64, B=32 fp64) in its width-bounded reading (reading W1); the literal
  C5 needs a 161 TB dense table.  Setup (one-time) is timed
  separately and reported under "setup".
* Multi-GPU: torchrun, one process per GPU; batched functions shard by column
  (each rank transforms its own B columns: weak scaling, no data-path
  collective).  Time = max over ranks of CUDA-event time.
* value: n·k·B gathers per transform x 2 transforms x steps x ranks / time.
* e2e: same metric through the C-ABI with pinned HOST buffers (H2D + D2H in
  the timed region).
* roofline: the dominant kernel's algorithmic bytes / its CUDA-event time
  recorded by the library on the launching stream inside the timed region.
* cpu_baseline / --impl reference: the CPU oracle O2 (the paper's sequential
  Algs. 3-4 in plain C, oracle/chain_oracle.c) on a bounded prefix sample.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PHASES = ("scan", "gather", "perm", "moebius_solve", "chain_diff")
KERNEL_NAMES = {"scan": "k_scan_tiles+k_scan_carry_tiles (iii)", "gather": "k_gather (iv)",
                "perm": "k_to_rank_major", "moebius_solve": "k_moeb_* (v)",
                "chain_diff": "k_chain_diff"}
MOEB_NAMES = ["auto", "level", "grid", "warp", "ring", "csr", "ringws", "ringdf", "ringcl", "ringcw"]


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="C5w")
    ap.add_argument("--dtype", default=None, choices=[None, "i64", "f64"])
    ap.add_argument("--batch", type=int, default=None, help="functions per rank")
    ap.add_argument("--scale", type=float, default=1.0)
    ap.add_argument("--moebius-kernel", default="auto", choices=MOEB_NAMES)
    ap.add_argument("--gather-variant", type=int, default=0, help="dense gather kernel for B%%32==0 (tuning)")
    ap.add_argument("--gather-pi-cfg", type=int, default=0, help="gather-order kernel configuration (tuning)")
    ap.add_argument("--ringcl-helpers", type=int, default=0, help="RINGCL helper CTAs (tuning; 0 = auto)")
    ap.add_argument("--ringcw-sleep", type=int, default=-1, help="RINGCW level-warp poll interval ns (tuning)")
    ap.add_argument("--ringcl-chunk", type=int, default=0, help="RINGCL owner stage chunk (tuning; 0 = plan)")
    ap.add_argument("--scan-mode", type=int, default=0, help="zeta scan: 0 auto, 1 single pass, 2 three kernels")
    ap.add_argument("--ring-debug", type=int, default=0, help="timing experiments only (invalid results)")
    ap.add_argument("--pipeline", default="auto", choices=["auto", "on", "off"],
                    help="batched pipeline: batch i+1's zeta on the SMs batch i's ring-family Möbius "
                         "leaves free (two streams; auto = when the Möbius leaves SMs free)")
    ap.add_argument("--inflight", type=int, default=1, choices=[1, 2, 3, 4],
                    help="Möbius solves in flight in the pipeline (2: RINGCL with one helper SM per column, "
                         "two batches' solves overlap; 3 / 4: RINGDF, one SM per column; a throughput "
                         "option, not the default)")
    ap.add_argument("--e2e-steps", type=int, default=20)
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="strong: BASELINE's global batch split over ranks (default); weak: per-rank batch")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-inflight2", action="store_true", help="skip the two-solves-in-flight throughput leg")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-provenance", action="store_true")
    ap.add_argument("--cpu-sample", type=int, default=None, help="oracle prefix size")
    return ap.parse_args()


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi samples during the timed region (B200_PROFILING.md)."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-i", str(self.device), "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def dist_init():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    return world, rank, local


def survey_bytes(n, k, B, info=None):
    """SURVEY §8(d) algorithmic bytes per transform CALL: 4·n·k index
    (4·nnz for the sparse table) + 32·n·B (f read, F written, F read once,
    g written).  The roofline's `achieved` uses these for the transform whose
    kernel dominates; the per-kernel models below split them by kernel."""
    idx = 4 * n * k
    if info is not None and info.get("zeta_sparse"):
        idx = 4 * info["nnz"]
    return idx + 32 * n * B


def alg_bytes(n, k, B, info=None):
    """Each kernel's own algorithmic bytes per launch."""
    d = {
        "scan": 16 * n * B + 4 * n,                 # f read, F write, slot->user
        "gather": 4 * n * k + 16 * n * B + 4 * n,   # index stream, F read once, g write
        "perm": 16 * n * B + 4 * n,                 # g read, gP write, rank->user
        "moebius_solve": 4 * n * k + 24 * n * B + 8 * n,   # index, g read, F write + read once
        "chain_diff": 16 * n * B + 4 * n,
    }
    if info is not None and info.get("zeta_sparse"):
        # sparse U-rows: 4 bytes per stored entry + row pointers instead of 4nk
        sparse = info["csr_bytes"] + 8 * n
        d["gather"] = sparse + 16 * n * B + 4 * n
    if info is not None and info.get("moebius_kernel") == 5:
        d["moebius_solve"] = info["csr_bytes"] + 32 * n * B + 8 * n   # rows, g, F w+r, f
    if info is not None and info.get("moebius_kernel") in (4, 6, 7, 8):
        # ring schedules: the schedule's own tables once (shared by the B CTAs
        # through L2), gP read, f written, rank->user rows; F never leaves
        # shared memory (RINGCL: nor the far sums -- DSMEM)
        tab = {4: "ring_bytes", 6: "rws_bytes", 7: "rdf_bytes", 8: "rdf_bytes"}[info["moebius_kernel"]]
        d["moebius_solve"] = info.get(tab, info["dist_bytes"]) + 16 * n * B + 4 * n
    return d


def ncu_traffic(config, phase):
    """DRAM bytes (read + write) per launch of the phase's kernel from the
    committed ncu --set full capture summary (profiles/ncu_traffic.json,
    written by scripts/profile_summaries.py from a .ncu-rep of this bench);
    (None, reason) when there is no capture for this config and phase."""
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        d = json.load(open(tpath))
        ent = d.get(config, {}).get(phase)
        if isinstance(ent, dict):
            return ent.get("bytes"), f"profiles/ncu_traffic.json ({ent.get('capture', '?')})"
        if ent is not None:
            return ent, "profiles/ncu_traffic.json"
    except Exception:
        pass
    return None, "no ncu capture for this config/phase"


def oracle_prefix(wl, B, n_sample, dtype):
    """The CPU oracle O2 on the down-closed prefix of the workload's first
    n_sample vertices (generator ids are bottom-up, so the prefix is itself a
    poset of the same family) and its input f."""
    import workloads as W
    from oracle.chain import ChainOracle
    m = wl.src < n_sample
    O = ChainOracle(n_sample, wl.src[m], wl.dst[m])
    f = (W.int_values(n_sample, B, -1000, 1000, seed=1) if dtype == "i64"
         else W.normal_values(n_sample, B, seed=1))
    return O, f


def oracle_time(O, f, parallel):
    """Seconds of one zeta + one Möbius (Algs. 3-4; `parallel`: the OpenMP
    build -- chains / rows in parallel, Möbius by Alg. 5 antichain by
    antichain)."""
    t0 = time.perf_counter()
    if parallel:
        O.moebius_omp(O.zeta_omp(f))
    else:
        O.moebius(O.zeta(f))
    return time.perf_counter() - t0


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, world, rank):
    """The reference arm: the CPU oracle (OpenMP build, all host cores) on a
    bounded prefix sample of the same workload, per step one zeta + one
    Möbius; rank 0 only."""
    if rank != 0:
        return 0
    import workloads as W
    from oracle.chain import threads
    wl = W.make_workload(args.config, args.scale, args.dtype, args.batch)
    n_s = args.cpu_sample or min(wl.n, 1_000_000)
    O, f = oracle_prefix(wl, wl.batch, n_s, wl.dtype)
    for _ in range(args.warmup):
        oracle_time(O, f, True)
    tot_t = sum(oracle_time(O, f, True) for _ in range(args.steps))
    units = 2 * n_s * O.k * wl.batch
    value = units * args.steps / tot_t
    sample = (f"prefix n={n_s} of {args.config} (k={O.k}, nnz={O.nnz}), B={wl.batch} {wl.dtype}, "
              f"zeta+Möbius Algs. 3-5 OpenMP on {threads()} threads, setup excluded")
    line = {"impl": "reference", "metric": "zeta/Möbius n·k gathers/s", "value": value,
            "unit": "n·k·B gathers/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * tot_t / args.steps,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
            "dtype": wl.dtype, "data": "synthetic",
            "config": {"workload": args.config, "n": wl.n, "global_batch": wl.batch},
            "cpu_baseline": {"value": value, "unit": "n·k·B gathers/s", "cores": threads(),
                             "host_cores": host_cores(), "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "n·k·B gathers/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def main():
    args = parse()
    world, rank, local = dist_init()
    if args.impl == "reference":
        return run_reference(args, world, rank)
    import numpy as np
    import torch
    import paper_2211_13706_b200 as pz
    import workloads as W
    torch.cuda.set_device(local)
    wl = W.make_workload(args.config, args.scale, args.dtype, args.batch)
    B = wl.batch
    t0 = time.perf_counter()
    P = pz.Poset(wl.n, wl.src, wl.dst, device=local)
    setup_s = time.perf_counter() - t0
    info = P.info()
    kern = MOEB_NAMES.index(args.moebius_kernel)
    P.set_option("moebius_kernel", kern)
    P.set_option("gather_variant", args.gather_variant)
    P.set_option("gather_pi_cfg", args.gather_pi_cfg)
    if args.ring_debug:
        P.set_option("ring_debug", args.ring_debug)
    if args.ringcl_helpers:
        P.set_option("ringcl_helpers", args.ringcl_helpers)
    if args.scan_mode:
        P.set_option("scan_mode", args.scan_mode)
    if args.ringcl_chunk:
        P.set_option("ringcl_chunk", args.ringcl_chunk)
    if args.ringcw_sleep >= 0:
        P.set_option("ringcw_sleep", args.ringcw_sleep)
    # strong scaling (default): BASELINE's global batch split over the ranks
    # by columns (no data-path collective); a single function (batch < world)
    # is row-sharded for zeta (NCCL all-gathers, dist.row_sharded_zeta) with
    # Möbius on rank 0 (its dependency chain does not shard, north star).
    # --scaling weak: every rank its own full batch.
    from paper_2211_13706_b200 import dist as pdist
    GB = wl.batch if args.scaling == "strong" else wl.batch * world
    row_mode = args.scaling == "strong" and world > 1 and wl.batch < world
    if args.scaling == "weak":
        f_host = np.ascontiguousarray(wl.values(seed=1 + rank))
        cols = (0, wl.batch)
    else:
        f_all = wl.values(seed=1)
        cols = (0, wl.batch) if row_mode else pdist.column_shard(wl.batch, world, rank)
        f_host = np.ascontiguousarray(f_all[:, cols[0]:cols[1]])
        del f_all
    shard = None
    if row_mode:
        # row-sharded index: each rank keeps its 4·k·n/G
        # bytes of table rows (D_U first: it needs the whole table)
        P.set_option("compute_depth_u", 1)
        slo, shi = pdist.shard_index(P)
        shard = {"rows": [slo, shi], "index_bytes_per_rank": P.info()["table_bytes"],
                 "index_bytes_unsharded": 4 * info["n"] * info["k"]}
    B = f_host.shape[1]
    x = torch.from_numpy(f_host).cuda()
    g = torch.empty_like(x)
    y = torch.empty_like(x)
    n, k = info["n"], info["k"]

    def step():
        if row_mode:
            pdist.row_sharded_zeta(P, x, out=g)
            if rank == 0:
                P.moebius(g, out=y)
        elif B > 0:
            P.zeta(x, out=g)
            P.moebius(g, out=y)

    # Batched pipeline: a ring-family Möbius occupies one
    # cluster of SMs per column (C5w: 32 x 3 = 96 of 148) for ~100 ms, so
    # batch i+1's zeta runs on the SMs it leaves free, on a second stream
    # (the library orders only calls that share scratch: zeta and ring-family
    # Möbius use disjoint lanes, include/poset.h).  The Möbius stream has the
    # higher priority so its clusters are placed before the zeta's CTAs; the
    # zeta's persistent gather grid is sized to the free SMs (option zeta_sms).
    def set_inflight(nfl):
        """Schedule for nfl solves side by side: 2 = RINGCL with one helper SM
        per column (64 SMs per solve at B = 32), 3 / 4 = RINGDF (one SM per
        column); 1 restores the command line's choice."""
        P.set_option("moebius_kernel", MOEB_NAMES.index("ringdf") if nfl >= 3 else kern)
        P.set_option("ringcl_helpers", 1 if nfl == 2 else args.ringcl_helpers)
        P.set_option("solves_inflight", nfl)

    if args.inflight >= 2:
        set_inflight(args.inflight)
    step()   # first call: builds the lazy tables and resolves the Möbius footprint
    torch.cuda.synchronize()
    inf0 = P.info()
    ring_fam = MOEB_NAMES[inf0["moebius_kernel"]] in ("ring", "ringws", "ringdf", "ringcl", "ringcw")
    free_sms = inf0["num_sms"] - args.inflight * inf0["moebius_sms"]
    use_pipe = (not row_mode and B > 0 and ring_fam and free_sms >= 8 and args.pipeline != "off") or \
        (args.pipeline == "on" and not row_mode and B > 0)
    zeta_budget = max(free_sms, 1) if use_pipe else 0
    if use_pipe:
        s_z = torch.cuda.Stream(priority=0)
        # two Möbius streams, alternating: batch i+1's permutation kernel
        # (its own rank-major buffer) runs while batch i's solve is still on
        # the SMs; the library keeps the solves themselves one at a time
        s_m = [torch.cuda.Stream(priority=-1) for _ in range(4)]

    def make_pipe(inflight, budget):
        NB = 2 + (inflight - 1)                # g buffers: one per batch between zeta and Möbius
        NS = max(2, inflight)                  # Möbius streams (round-robin), one output each
        return {"NB": NB, "NS": NS, "budget": budget,
                "gb": [g] + [torch.empty_like(x) for _ in range(NB - 1)],
                "ys": [y] + [torch.empty_like(x) for _ in range(NS - 1)] if inflight >= 2 else [y, y],
                "ev_z": [torch.cuda.Event() for _ in range(NB)],
                "ev_m": [torch.cuda.Event() for _ in range(NB)]}

    pipe0 = make_pipe(args.inflight, zeta_budget) if use_pipe else None

    def run_steps(nsteps, pipe=None):
        pipe = pipe or pipe0
        if not use_pipe:
            for _ in range(nsteps):
                step()
            return
        cur = torch.cuda.current_stream()
        s_z.wait_stream(cur)
        for sm in s_m:
            sm.wait_stream(cur)
        NB, gb, ys, ev_z, ev_m = pipe["NB"], pipe["gb"], pipe["ys"], pipe["ev_z"], pipe["ev_m"]
        NS = pipe["NS"]
        P.set_option("zeta_sms", 0)            # the prologue zeta has the whole GPU
        P.zeta(x, out=gb[0], stream=s_z)
        ev_z[0].record(s_z)
        P.set_option("zeta_sms", pipe["budget"])
        for i in range(nsteps):
            b, sm = i % NB, s_m[i % NS]
            sm.wait_event(ev_z[b])
            P.moebius(gb[b], out=ys[i % NS], stream=sm)
            ev_m[b].record(sm)
            if i + 1 < nsteps:
                nb = (i + 1) % NB
                if i + 1 >= NB:                 # gb[nb] was Möbius(i+1-NB)'s input
                    s_z.wait_event(ev_m[nb])
                P.zeta(x, out=gb[nb], stream=s_z)
                ev_z[nb].record(s_z)
        for sm in s_m:
            cur.wait_stream(sm)
        cur.wait_stream(s_z)
        P.set_option("zeta_sms", 0)

    run_steps(args.warmup)
    torch.cuda.synchronize()
    # correctness spot check of the timed computation (round trip)
    if wl.dtype == "i64":
        y_last = pipe0["ys"][(args.warmup - 1) % pipe0["NS"]] if use_pipe and args.warmup > 0 else y
        ok = bool(torch.equal(y_last, x)) if (rank == 0 or not row_mode) else None
    else:
        ok = None   # fp64 Möbius on deep posets is ill-conditioned (reading G8)
    P.set_option("profile", 1)
    P.profile_read()
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    clocks = ClockSampler(local)
    clocks.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run_steps(args.steps)
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    prof, launches = P.profile_read()
    P.set_option("profile", 0)
    if args.ring_debug:
        print("ring_debug counters:", P.debug_read().tolist(), file=sys.stderr, flush=True)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    if world > 1:
        torch.distributed.all_reduce(ms_t, op=torch.distributed.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    units_step = 2 * n * k * GB            # whole job, all ranks
    value = units_step * args.steps / (ms_max / 1e3)

    # per-kernel roofline (this rank; rank 0 reports)
    peak, peak_kind = peaks()
    info = P.info()
    ab = alg_bytes(n, k, B, info)
    kernels = {}
    for ph in PHASES:
        tms, calls = prof[ph]
        if calls == 0:
            continue
        per = tms / calls
        gbs = ab[ph] / (per / 1e3) / 1e9
        kernels[ph] = {"kernel": KERNEL_NAMES[ph], "ms_per_call": per, "share": tms / ms,
                       "alg_bytes": ab[ph], "achieved_gbs": gbs, "frac": gbs / peak}
    if not kernels:   # row-sharded zeta only on this rank (split phases are not phase-timed)
        kernels = {"moebius_solve": {"kernel": KERNEL_NAMES["moebius_solve"], "ms_per_call": ms / args.steps,
                                     "share": 1.0, "alg_bytes": ab["moebius_solve"], "achieved_gbs": 0.0,
                                     "frac": 0.0}}
    dom = max(kernels, key=lambda p: kernels[p]["share"])
    traffic, tsrc = ncu_traffic(args.config, dom)
    sb = survey_bytes(n, k, B, info)
    # the dominant kernel is one transform's kernel: §8(d) bytes of that call
    dom_ms = kernels[dom]["ms_per_call"]
    roof = {"bound": "hbm", "kernel": kernels[dom]["kernel"], "alg_bytes": sb,
            "alg_bytes_basis": "SURVEY §8(d): 4nk + 32nB per transform call",
            "achieved": sb / (dom_ms / 1e3) / 1e9, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": sb / (dom_ms / 1e3) / 1e9 / peak,
            "kernel_bytes": kernels[dom]["alg_bytes"], "kernel_frac": kernels[dom]["frac"],
            "traffic": traffic, "traffic_source": tsrc}
    # the zeta gather is the kernel the north star's roofline target names;
    # in the pipeline it runs on the SMs the Möbius leaves free, so its
    # full-GPU rate comes from a serial pass after the timed region
    serial_k = None
    if use_pipe:
        P.set_option("profile", 1)
        P.profile_read()
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        sprof, _ = P.profile_read()
        P.set_option("profile", 0)
        serial_k = {}
        for ph in ("scan", "gather", "perm", "moebius_solve"):
            tms, calls = sprof[ph]
            if calls:
                per = tms / calls
                serial_k[ph] = {"ms_per_call": per, "achieved_gbs": ab[ph] / (per / 1e3) / 1e9,
                                "frac": ab[ph] / (per / 1e3) / 1e9 / peak}
        for ph in kernels:
            if ph in serial_k:
                kernels[ph]["serial_ms_per_call"] = serial_k[ph]["ms_per_call"]
    zroof = None
    if serial_k and "gather" in serial_k:
        zt, zsrc = ncu_traffic(args.config, "gather")
        zroof = {"bound": "hbm", "kernel": kernels["gather"]["kernel"],
                 "alg_bytes": kernels["gather"]["alg_bytes"],
                 "alg_bytes_basis": "SURVEY §8(d) zeta bytes minus the scan's 16nB: 4nk + 16nB",
                 "achieved": serial_k["gather"]["achieved_gbs"], "peak": peak, "peak_kind": peak_kind,
                 "unit": "GB/s", "frac": serial_k["gather"]["frac"], "traffic": zt, "traffic_source": zsrc,
                 "measured": "serial pass on all SMs after the timed region (in the pipeline the gather "
                             f"runs on the {zeta_budget} SMs the Möbius leaves free: "
                             f"{kernels['gather']['ms_per_call']:.2f} ms per call, overlapped)"}
    elif "gather" in kernels:
        zt, zsrc = ncu_traffic(args.config, "gather")
        zroof = {"bound": "hbm", "kernel": kernels["gather"]["kernel"],
                 "alg_bytes": kernels["gather"]["alg_bytes"],
                 "alg_bytes_basis": "SURVEY §8(d) zeta bytes minus the scan's 16nB: 4nk + 16nB",
                 "achieved": kernels["gather"]["achieved_gbs"], "peak": peak, "peak_kind": peak_kind,
                 "unit": "GB/s", "frac": kernels["gather"]["frac"], "traffic": zt, "traffic_source": zsrc}
    if dom == "moebius_solve":
        try:
            if P.info()["depth_u"] < 0:
                P.set_option("compute_depth_u", 1)
            du = P.info()["depth_u"]
        except pz.PosetError:   # sparse-rows poset: D_U needs the dense table
            du = None
        roof["note"] = (f"latency-bound triangular solve: {info['ell']} dependent levels, D_U = {du}, "
                        f"{1e3 * dom_ms / max(info['ell'], 1):.3f} µs per level")
        # the bound that matters for a dependent level sweep: per-level time
        # against the measured floor of one level hand-off between two warps
        # (mbarrier arrive -> try_wait wake, scripts/micro/handoff.cu: 91 cycles)
        mhz = (clk or {}).get("sm_mhz") or (clk or {}).get("sm_max_mhz") or 1965.0
        cyc = dom_ms * 1e-3 * mhz * 1e6 / max(info["ell"], 1)
        roof["latency"] = {"cycles_per_level": cyc, "floor_cycles_per_level": 91.0,
                           "floor": "two-warp mbarrier hand-off, measured (scripts/micro/handoff.cu)",
                           "frac": 91.0 / cyc, "depth_u": du,
                           "us_per_DU_step": 1e3 * dom_ms / max(du, 1) if du else None,
                           "cycles_per_DU_step": dom_ms * 1e-3 * mhz * 1e6 / max(du, 1) if du else None}

    # e2e: C-ABI with pinned host buffers, copies inside the timed region
    e2e = None
    if not args.no_e2e and not row_mode:
        fp = torch.from_numpy(f_host).pin_memory()
        # (a) the production pattern: every step copies its input f from pinned
        # host memory and reads its result (the round trip's output) back,
        # with the copies of step i+-1 overlapping step i's transforms
        # (copy streams + events, two buffer slots; the transforms are the
        # library's public calls on one compute stream, the intermediate g
        # stays on the device)
        def e2e_run(NSL, budget, K):
            """K e2e steps over NSL buffer slots (one Möbius stream per slot)."""
            rt_ok = None
            s_in, s_cmp, s_out = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
            # pipelined: the Möbius on its own high-priority stream (see run_steps)
            s_mb = [torch.cuda.Stream(priority=-1) for _ in range(NSL)] if use_pipe else [s_cmp] * NSL
            xin = [torch.empty_like(x) for _ in range(NSL)]
            yout = [torch.empty_like(x) for _ in range(NSL)]
            gd2 = [torch.empty_like(x) for _ in range(NSL)] if use_pipe else [torch.empty_like(x)] * NSL
            res = [torch.empty_like(fp).pin_memory() for _ in range(NSL)]
            ev = lambda: torch.cuda.Event()
            in_done, in_free, out_done, out_free = [ev() for _ in range(NSL)], [ev() for _ in range(NSL)], \
                [ev() for _ in range(NSL)], [ev() for _ in range(NSL)]
            z_done, g_free = [ev() for _ in range(NSL)], [ev() for _ in range(NSL)]

            def pipelined(steps):
                P.set_option("zeta_sms", budget)
                for i in range(steps):
                    sl = i % NSL
                    with torch.cuda.stream(s_in):
                        if i >= NSL:
                            s_in.wait_event(in_free[sl])
                        xin[sl].copy_(fp, non_blocking=True)
                        in_done[sl].record(s_in)
                    s_cmp.wait_event(in_done[sl])
                    if i >= NSL and use_pipe:
                        s_cmp.wait_event(g_free[sl])
                    P.zeta(xin[sl], out=gd2[sl], stream=s_cmp)
                    in_free[sl].record(s_cmp)
                    z_done[sl].record(s_cmp)
                    s_mb[sl].wait_event(z_done[sl])
                    if i >= NSL:
                        s_mb[sl].wait_event(out_free[sl])
                    P.moebius(gd2[sl], out=yout[sl], stream=s_mb[sl])
                    g_free[sl].record(s_mb[sl])
                    out_done[sl].record(s_mb[sl])
                    with torch.cuda.stream(s_out):
                        s_out.wait_event(out_done[sl])
                        res[sl].copy_(yout[sl], non_blocking=True)
                        out_free[sl].record(s_out)
                P.set_option("zeta_sms", 0)

            pipelined(NSL)
            torch.cuda.synchronize()
            if wl.dtype == "i64":
                rt_ok = bool((res[NSL - 1].numpy() == f_host).all())
            if world > 1:
                torch.distributed.barrier()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s_in.wait_stream(torch.cuda.current_stream())
            a0.record(s_in)
            pipelined(K)
            s_in.wait_stream(s_out)
            for sm in s_mb:
                s_in.wait_stream(sm)
            a1.record(s_in)
            torch.cuda.synchronize()
            ems = torch.tensor([a0.elapsed_time(a1)], dtype=torch.float64, device="cuda")
            if world > 1:
                torch.distributed.all_reduce(ems, op=torch.distributed.ReduceOp.MAX)
            return float(ems.item()), rt_ok

        K = args.e2e_steps
        ems, rt_ok = e2e_run(2, zeta_budget, K)
        e2e = {"value": units_step * K / (ems / 1e3), "unit": "n·k·B gathers/s",
               "h2d_bytes_per_step": n * GB * 8, "d2h_bytes_per_step": n * GB * 8,
               "ms_per_step": ems / K, "steps": K,
               "round_trip_exact": rt_ok if wl.dtype == "i64" else None,
               "path": ("per step: f (pinned host) -> device copy, poset_zeta then poset_moebius (g stays "
                        "on the device" + ("; the Möbius on its own high-priority stream, so batch i+1's "
                                           "zeta overlaps batch i's Möbius" if use_pipe else
                                           ", one compute stream") +
                        "), result -> pinned host copy; copies on their own streams, overlapping the "
                        "neighbouring steps' transforms")}
        # the same with three batches' RINGDF solves in flight (three slots)
        if use_pipe and args.inflight == 1 and world == 1 and not args.no_inflight2 and \
                MOEB_NAMES[inf0["moebius_kernel"]] == "ringcl":
            try:
                set_inflight(3)
                step()
                torch.cuda.synchronize()
                inf3 = P.info()
                free3 = inf3["num_sms"] - 3 * inf3["moebius_sms"]
                if free3 >= 8:
                    K3 = 3 * max(K // 3, 1)
                    ems3, ok3 = e2e_run(3, free3, K3)
                    e2e["three_solves_inflight"] = {
                        "value": units_step * K3 / (ems3 / 1e3), "ms_per_step": ems3 / K3, "steps": K3,
                        "round_trip_exact": ok3, "moebius_kernel": MOEB_NAMES[inf3["moebius_kernel"]],
                        "zeta_sms": free3}
            finally:
                set_inflight(1)
        # (b) context: both transforms staged through host memory by the library
        # itself (zeta host -> host, Möbius host -> host, serial)
        gp = torch.empty_like(fp).pin_memory()
        P.zeta(fp, out=gp)
        P.moebius(gp, out=gp)
        torch.cuda.synchronize()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record()
        for _ in range(2):
            P.zeta(fp, out=gp)
            P.moebius(gp, out=gp)
        a1.record()
        torch.cuda.synchronize()
        e2e["staged_host_both"] = {"ms_per_step": a0.elapsed_time(a1) / 2,
                                   "h2d_bytes_per_step": 2 * n * GB * 8, "d2h_bytes_per_step": 2 * n * GB * 8,
                                   "path": "poset_zeta and poset_moebius each host -> host (library-staged copies)"}
        del fp, gp

    # throughput with two batches' solves in flight (option solves_inflight,
    # DESIGN.md §5.5): one helper SM per column instead of two, so two RINGCL
    # solves sit side by side and the zeta takes the remaining SMs.  Reported
    # beside the headline (which keeps one solve at a time: lower per-batch
    # latency, and the dominant kernel's launch duration is the roofline's).
    two = None
    if use_pipe and args.inflight == 1 and world == 1 and not args.no_inflight2 and \
            MOEB_NAMES[inf0["moebius_kernel"]] == "ringcl":
        two = {}
        try:
            for nfl in (2, 3):
                set_inflight(nfl)
                step()
                torch.cuda.synchronize()
                inf2 = P.info()
                free2 = inf2["num_sms"] - nfl * inf2["moebius_sms"]
                if free2 < 8:
                    continue
                pipe2 = make_pipe(nfl, free2)
                run_steps(nfl + 1, pipe2)
                torch.cuda.synchronize()
                ok2 = bool(torch.equal(pipe2["ys"][0], x)) if wl.dtype == "i64" else None
                b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                b0.record()
                run_steps(args.steps, pipe2)
                b1.record()
                torch.cuda.synchronize()
                ms2 = b0.elapsed_time(b1)
                two[str(nfl)] = {
                    "ms_per_step": ms2 / args.steps, "value": units_step * args.steps / (ms2 / 1e3),
                    "unit": "n·k·B gathers/s", "steps": args.steps, "solves_inflight": nfl,
                    "moebius_kernel": MOEB_NAMES[inf2["moebius_kernel"]],
                    "moebius_sms_per_solve": inf2["moebius_sms"], "zeta_sms": free2, "round_trip_exact": ok2}
                del pipe2
            two["note"] = ("batches' solves side by side (2: RINGCL with one helper SM per column; 3: RINGDF, "
                           "one SM per column), the zeta on the remaining SMs; per-batch latency is higher "
                           "than the headline's")
        finally:
            set_inflight(1)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle.chain import threads
        n_s = args.cpu_sample or min(wl.n, 1_000_000)
        O, fs = oracle_prefix(wl, B, n_s, wl.dtype)
        t_par = oracle_time(O, fs, True)
        t_seq = oracle_time(O, fs, False)
        units = 2 * n_s * O.k * B
        cpu = {"value": units / t_par, "unit": "n·k·B gathers/s", "cores": threads(),
               "host_cores": host_cores(), "kind": "oracle",
               "sample": (f"prefix n={n_s} of {args.config} (k={O.k}, nnz={O.nnz}), B={B} {wl.dtype}, "
                          f"one zeta + one Möbius (Algs. 3-4; OpenMP, Möbius by Alg. 5), setup excluded, "
                          f"{t_par:.2f} s"),
               "single_core": {"value": units / t_seq, "cores": 1, "seconds": t_seq}}
        del O, fs

    prov = None
    if rank == 0 and not args.no_provenance:
        prov = {"sha256_edges": W.sha256_arrays(wl.src, wl.dst), "sha256_f_rank0": W.sha256_arrays(f_host),
                "generator": "workloads.make_workload (numpy PCG64, DAG seed 0, values seed 1)"}
    if rank == 0:
        line = {
            "metric": "zeta/Möbius n·k gathers/s", "value": value, "unit": "n·k·B gathers/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_max / args.steps, "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": wl.dtype, "data": "synthetic",
            "config": {"workload": args.config, "desc": wl.desc, "n": n, "k": k,
                       "batch_per_rank": B, "global_batch": GB, "ell": info["ell"],
                       "q": info["q"], "nnz": info["nnz"], "edges": info["m"],
                       "moebius_kernel": MOEB_NAMES[info["moebius_kernel"]],
                       "reach": info["reach"],
                       "parallelism": (f"zeta row-shard x{world} + NCCL all-gather, Möbius on rank 0"
                                       if row_mode else f"column-shard x{world}"),
                       "depth_u": P.info()["depth_u"], "provenance": prov, "index_shard": shard,
                       "pipeline": ({"zeta_sms": zeta_budget, "moebius_sms": inf0["moebius_sms"],
                                     "solves_inflight": args.inflight,
                                     "how": "batch i+1's zeta (low-priority stream, gather grid on the free "
                                            "SMs) overlaps batch i's Möbius (high-priority stream); every "
                                            "step still runs scan, gather, permutation and U-solve on its "
                                            "own batch"}
                                    if use_pipe else None),
                       "l2": "inputs > L2 (index table 4nk B, F 8nB B): no flush needed"},
            "gbs_per_step": sum(ab[p] for p in kernels) / (ms_max / args.steps / 1e3) / 1e9,
            # nnz(N)·B per second: the work the method needs;
            # n·k·B above counts the dense table's entries, ∞ included
            "value_nnz": 2 * info["nnz"] * GB * args.steps / (ms_max / 1e3),
            "roofline": roof, "zeta_roofline": zroof, "kernels": kernels, "cpu_baseline": cpu, "e2e": e2e,
            "throughput_solves_inflight": two,
            "gpu_launches": launches, "clocks": clk, "round_trip_exact": ok,
            "setup": {"seconds": setup_s, "ingest": info["t_ingest"], "levels": info["t_levels"],
                      "match": info["t_match"], "chains": info["t_chains"],
                      "upload": info["t_upload"], "mtable": info["t_mtable"],
                      "dist_table": info["t_dist"], "gather_order_table_bytes": P.info()["gather_bytes"],
                      "depth_u_seconds": P.info()["t_depth"]},
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
