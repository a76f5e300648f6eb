"""GPU parity: the CUDA path (through the C-ABI) against the CPU oracle.

Bar (BASELINE.json north star): int64 bit-exact (Z/2^64); fp64 within
|Δ| <= 1e-9 * Σ_{y⪯x}|f(y)| (scale computed by the oracle).  Möbius fp64 is
only compared where μ is bounded (Boolean lattice, shallow posets; reading G8
of DESIGN.md); deep posets use int64 round trips.
"""
import numpy as np
import pytest

from conftest import assert_fp64_close, load_facts, load_matrix
import workloads as W

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2211_13706_b200 as pz  # noqa: E402
from oracle import brute  # noqa: E402
from oracle.chain import ChainOracle, zeta_sampled_edges  # noqa: E402

KERNELS = [pz.MOEB_LEVEL, pz.MOEB_GRID, pz.MOEB_WARP, pz.MOEB_RING, pz.MOEB_CSR, pz.MOEB_RINGWS,
           pz.MOEB_RINGDF, pz.MOEB_RINGCL, pz.MOEB_RINGCW]


def kernels_for(P):
    """Every Möbius schedule that applies to P (RING needs a bounded reach,
    CSR needs the sparse rows, built when RING does not apply)."""
    info = P.info()
    return [k for k in KERNELS
            if (k != pz.MOEB_RING or info["dist_bytes"] > 0) and (k != pz.MOEB_CSR or info["csr_bytes"] > 0)
            and (k != pz.MOEB_RINGWS or info["ringws"]) and (k != pz.MOEB_RINGDF or info["ringdf"] & 1)
            and (k != pz.MOEB_RINGCL or info["ringdf"] & 2) and (k != pz.MOEB_RINGCW or info["ringdf"] & 4)]
facts = load_facts()
PAPER_CHAINS = [[int(v) - 1 for v in c.split(",")] for c in facts["chains"].split(";")]


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def gpu_zeta(P, f):
    return host(P.zeta(dev(f)))


def gpu_moebius(P, g, kernel=None):
    if kernel is not None:
        P.set_option("moebius_kernel", kernel)
    out = host(P.moebius(dev(g)))
    if kernel is not None:
        P.set_option("moebius_kernel", pz.MOEB_AUTO)
    return out


# ------------------------------------------------------------ paper example

def test_example_paper_N_and_transforms(paper_example):
    n, src, dst = paper_example
    P = pz.Poset(n, src, dst, chains=PAPER_CHAINS)
    info = P.info()
    assert info["k"] == 4 and info["nnz"] == int(facts["nnz_N"]) and info["ell"] == 5
    # N (paper labels, -1 = ∞) -> bottom-up positions
    N = load_matrix("N.txt")
    pos = {}
    for c in PAPER_CHAINS:
        for p, v in enumerate(reversed(c)):
            pos[v] = p
    want = np.where(N > 0, np.vectorize(lambda v: pos.get(v - 1, -1))(N), -1)
    assert (P.export_mtable() == want).all()
    Z, M = load_matrix("Z.txt"), load_matrix("M.txt")
    f = W.int_values(12, 5, -100, 100, seed=3)
    assert (gpu_zeta(P, f) == Z @ f).all()
    for kern in kernels_for(P):
        assert (gpu_moebius(P, f, kern) == M @ f).all()
    ff = W.normal_values(12, 4, seed=4)
    assert_fp64_close(gpu_zeta(P, ff), Z @ ff, Z @ np.abs(ff))


def test_example_own_matching(paper_example):
    n, src, dst = paper_example
    P = pz.Poset(n, src, dst)
    assert P.info()["k"] == 4
    Z, M = load_matrix("Z.txt"), load_matrix("M.txt")
    f = W.int_values(12, 3, -100, 100, seed=5)
    assert (gpu_zeta(P, f) == Z @ f).all()
    assert (gpu_moebius(P, f) == M @ f).all()


# ------------------------------------------------------ m-table via Thm. 3

@pytest.mark.parametrize("name,n,make", [
    ("C1", 1000, lambda: W.window_dag(1000, 3, 50, 0)),
    ("C5w", 1500, lambda: W.window_dag(1500, 2, 64, 1, forced=True)),
    ("C4", 8 * 64, lambda: W.layered_dag(8, 64, 3, 2)),
    ("bool9", 512, lambda: W.boolean_lattice(9)),
])
def test_mtable_is_downset_count(name, n, make):
    """Thm. 3: m(x,j) + 1 = |↓x ∩ Z_j| for the library's own
    chains; brute-force down-sets from the oracle."""
    src, dst = make()
    P = pz.Poset(n, src, dst)
    chain, pos, level, rank = P.export_chains()
    mt = P.export_mtable()
    down = brute.downsets(n, src, dst)
    k = P.k
    for x in range(n):
        members = brute._bits(down[x], n)
        cnt = np.bincount(chain[members], minlength=k)
        assert (mt[x] + 1 == cnt).all(), x
    assert P.info()["nnz"] == int((mt >= 0).sum())


# ---------------------------------------------- O2 parity, many instances

def instances():
    yield "C1", 1000, *W.window_dag(1000, 3, 50, 0)
    yield "C3lit_20k", 20000, *W.window_dag(20000, 2, 1000, 0)
    yield "C3w_30k", 30000, *W.window_dag(30000, 2, 1000, 0, forced=True)
    yield "C4lit_64L", 64 * 256, *W.layered_dag(64, 256, 3, 0)
    yield "C4w_128L", 128 * 256, *W.layered_dag(128, 256, 3, 0, forced=True)
    yield "C5lit_20k", 20000, *W.window_dag(20000, 2, 64, 0)
    yield "C5w_50k", 50000, *W.window_dag(50000, 2, 64, 0, forced=True)
    yield "bool12", 4096, *W.boolean_lattice(12)
    yield "ER4_5k", 5000, *W.erdos_renyi(5000, 4, 1)
    yield "ER6_3k", 3000, *W.erdos_renyi(3000, 6, 2)


@pytest.fixture(scope="module")
def built():
    cache = {}

    def get(name, n, src, dst):
        if name not in cache:
            cache[name] = (pz.Poset(n, src, dst), ChainOracle(n, src, dst))
        return cache[name]
    return get


@pytest.mark.parametrize("inst", list(instances()), ids=lambda t: t[0])
@pytest.mark.parametrize("B", [1, 3, 32])
def test_int64_zeta_moebius_vs_O2(inst, B, built):
    name, n, src, dst = inst
    P, O = built(name, n, src, dst)
    f = W.int_values(n, B, -1000, 1000, seed=B)
    g = gpu_zeta(P, f)
    assert (g == O.zeta(f)).all()
    for kern in kernels_for(P):
        if kern == pz.MOEB_LEVEL and P.ell > 3000:
            continue
        assert (gpu_moebius(P, g, kern) == f).all(), kern
    h = W.int_values(n, B, -10**17, 10**17, seed=B + 100)     # arbitrary g, wraps
    assert (gpu_moebius(P, h) == O.moebius(h)).all()


@pytest.mark.parametrize("inst", list(instances()), ids=lambda t: t[0])
@pytest.mark.parametrize("B", [1, 4])
def test_fp64_zeta_vs_O2(inst, B, built):
    name, n, src, dst = inst
    P, O = built(name, n, src, dst)
    f = W.normal_values(n, B, seed=7 + B)
    assert_fp64_close(gpu_zeta(P, f), O.zeta(f), O.zeta(np.abs(f)))


@pytest.mark.parametrize("name,n,make", [
    ("C1", 1000, lambda: W.window_dag(1000, 3, 50, 0)),
    ("C5w_2k", 2000, lambda: W.window_dag(2000, 2, 64, 0, forced=True)),
    ("C3w_20k", 20000, lambda: W.window_dag(20000, 2, 1000, 0, forced=True)),
    ("C4w_24L", 24 * 256, lambda: W.layered_dag(24, 256, 3, 0, forced=True)),
])
def test_fp64_moebius_shallow_vs_O2(name, n, make):
    """fp64 Möbius only where |μ| stays small (reading G8)."""
    src, dst = make()
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    f = W.normal_values(n, 2, seed=3)
    g = O.zeta(f)
    want = O.moebius(g)
    for kern in kernels_for(P):
        assert_fp64_close(gpu_moebius(P, g, kern), want, O.zeta(np.abs(want)))


# --------------------------------------------------- C2: Boolean lattice 2^16

def test_C2_boolean_lattice_vs_yates():
    bits = 16
    n = 1 << bits
    src, dst = W.boolean_lattice(bits)
    P = pz.Poset(n, src, dst)
    info = P.info()
    assert info["k"] == 12870 and info["ell"] == 17
    f = W.normal_values(n, 1, seed=1)
    g = gpu_zeta(P, f)
    assert_fp64_close(g, brute.yates_zeta(bits, f), brute.yates_zeta(bits, np.abs(f)))
    gy = brute.yates_zeta(bits, f)
    for kern in kernels_for(P):
        assert_fp64_close(gpu_moebius(P, gy, kern), brute.yates_moebius(bits, gy),
                          brute.yates_zeta(bits, np.abs(f)))
    fi = W.int_values(n, 2, -1000, 1000, seed=2)
    gi = gpu_zeta(P, fi)
    assert (gi == brute.yates_zeta(bits, fi)).all()
    assert (gpu_moebius(P, gi) == fi).all()


# ------------------------------------------------------- RING schedule

def test_ring_schedule_selection_and_limits():
    """RING is chosen for bounded-reach posets, refused where it cannot run."""
    n = 20000
    src, dst = W.window_dag(n, 2, 64, 3, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    info = P.info()
    assert info["dist_bytes"] > 0 and 0 < info["reach"] < 65535
    assert info["moebius_kernel"] in (pz.MOEB_RINGCL, pz.MOEB_RINGCW) and info["ringws"] == 1
    assert info["ringdf"] & 3 == 3
    for B in (1, 2, 7, 33):
        f = W.int_values(n, B, -1000, 1000, seed=B)
        g = gpu_zeta(P, f)
        assert (gpu_moebius(P, g) == f).all(), B
        h = W.int_values(n, B, -10**17, 10**17, seed=B + 9)
        want = O.moebius(h)
        assert (gpu_moebius(P, h, pz.MOEB_RING) == want).all(), B
        assert (gpu_moebius(P, h, pz.MOEB_RINGWS) == want).all(), B
        assert (gpu_moebius(P, h, pz.MOEB_RINGDF) == want).all(), B
        assert info["ringdf"] & 2
        assert (gpu_moebius(P, h, pz.MOEB_RINGCL) == want).all(), B
        for nh in (1, 2, 3):   # helper CTAs per column (cluster of nh + 1)
            P.set_option("ringcl_helpers", nh)
            assert (gpu_moebius(P, h, pz.MOEB_RINGCL) == want).all(), (B, nh)
            if info["ringdf"] & 4:
                assert (gpu_moebius(P, h, pz.MOEB_RINGCW) == want).all(), (B, nh)
        P.set_option("ringcl_helpers", 0)
        for lpe in (1, 2, 4, 8):
            P.set_option("ring_lpe", lpe)
            assert (gpu_moebius(P, h, pz.MOEB_RING) == want).all(), (B, lpe)
        P.set_option("ring_lpe", 8)
    # wide levels (Boolean lattice 2^12: 924-element middle level) do not fit;
    # there AUTO takes the sparse-row schedule
    Pb = pz.Poset(4096, *W.boolean_lattice(12))
    assert Pb.info()["dist_bytes"] == 0
    assert Pb.info()["csr_bytes"] > 0 and Pb.info()["moebius_kernel"] == pz.MOEB_CSR
    assert Pb.info()["zeta_sparse"] == 1            # fill < 1/2: zeta over the sparse rows
    Pb.set_option("moebius_kernel", pz.MOEB_RING)
    with pytest.raises(pz.PosetError) as e:
        Pb.moebius(dev(np.zeros((4096, 1), np.int64)))
    assert e.value.code == "EINVAL"


# ---------------------------------------------------------------- edge cases

@pytest.mark.parametrize("wide", [70, 150])
def test_ring_schedules_wide_levels_and_large_batch(wide):
    """A level of three (five) 32-element passes: the multi-pass level body
    of RINGDF / RINGCL and their serial passes beyond the register
    passes, and a batch too large for CTA pairs (AUTO falls back to RINGDF),
    bit-exact against O2."""
    # a width-8 window DAG, then one level of `wide` elements, each above two
    # elements of the base's top level
    n0 = 3000
    s0, d0 = W.window_dag(n0, 2, 8, 3, forced=True)
    _, _, _, lvl = pz.analyze(n0, s0, d0, want_chains=True)
    top = np.flatnonzero(lvl == lvl.max())
    rng = np.random.default_rng(4)
    new = np.repeat(np.arange(n0, n0 + wide, dtype=np.int64), 2)
    tgt = top[rng.integers(0, top.shape[0], size=new.shape[0])]
    n = n0 + wide
    src, dst = np.concatenate([s0, new]), np.concatenate([d0, tgt])
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    info = P.info()
    assert info["max_level_width"] >= wide   # several passes of 32 in one level
    if not info["ringdf"] & 1:
        pytest.skip("RINGDF does not fit this poset")
    for B in (1, 33):
        h = W.int_values(n, B, -10**17, 10**17, seed=B + 3)
        want = O.moebius(h)
        assert (gpu_moebius(P, h, pz.MOEB_RINGDF) == want).all(), B
        if info["ringdf"] & 2:
            assert (gpu_moebius(P, h, pz.MOEB_RINGCL) == want).all(), B
        if info["ringdf"] & 4:
            assert (gpu_moebius(P, h, pz.MOEB_RINGCW) == want).all(), B

    h = W.int_values(n, 80, -10**17, 10**17, seed=11)   # 2 x 80 CTAs > 148 SMs
    assert (gpu_moebius(P, h) == O.moebius(h)).all()


def test_edge_cases_tiny():
    for n, (src, dst) in [(1, W.antichain_dag(1)), (7, W.antichain_dag(7)), (40, W.chain_dag(40)),
                          (2, (np.array([1, 1]), np.array([0, 0])))]:
        P = pz.Poset(n, src, dst)
        f = W.int_values(n, 3, -9, 9, seed=n)
        O = ChainOracle(n, src, dst)
        assert (gpu_zeta(P, f) == O.zeta(f)).all()
        assert (gpu_moebius(P, f) == O.moebius(f)).all()


def test_ragged_batches_and_1d():
    n = 3000
    src, dst = W.window_dag(n, 2, 64, 4, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    for B in (2, 5, 6, 12, 40, 64, 96):
        f = W.int_values(n, B, -1000, 1000, seed=B)
        assert (gpu_zeta(P, f) == O.zeta(f)).all(), B
        assert (gpu_moebius(P, O.zeta(f)) == f).all(), B
    f1 = W.int_values(n, 1, -5, 5, seed=1)[:, 0]
    assert (host(P.zeta(dev(f1))) == O.zeta(f1)).all()


@pytest.mark.parametrize("variant", [0, 1, 2, 3, 4])
def test_dense_gather_variants(variant):
    """The three dense zeta-gather kernels for batch % 32 == 0 agree with O2
    (bit-exact int64, tolerance fp64), including a ragged rank tail."""
    n = 5003
    src, dst = W.window_dag(n, 2, 64, 7, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    P.set_option("gather_variant", variant)
    try:
        for B in (32, 64):
            f = W.int_values(n, B, -10**15, 10**15, seed=B)
            assert (gpu_zeta(P, f) == O.zeta(f)).all(), B
            ff = W.normal_values(n, B, seed=B + 1)
            assert_fp64_close(gpu_zeta(P, ff), O.zeta(ff), O.zeta(np.abs(ff)))
    finally:
        P.set_option("gather_variant", 0)


@pytest.mark.parametrize("cfg", [0, 1, 2, 3, 4, 5, 6, 7])
def test_gather_order_configs(cfg):
    """The gather-order kernel's configurations (option gather_pi_cfg; 4 is
    the delta-list gather) against O2, bit-exact int64 and fp64 within the
    tolerance, with ∞ entries (the bottom of the poset), a ragged tile and
    1, 2 and 4 columns per lane (B = 32, 64, 96, 128)."""
    n = 7003
    src, dst = W.window_dag(n, 2, 64, 9, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    P.set_option("gather_pi_cfg", cfg)
    try:
        for B in (32, 64, 96, 128):
            f = W.int_values(n, B, -10**15, 10**15, seed=B + cfg)
            assert (gpu_zeta(P, f) == O.zeta(f)).all(), B
            ff = W.normal_values(n, B, seed=B + 2)
            assert_fp64_close(gpu_zeta(P, ff), O.zeta(ff), O.zeta(np.abs(ff)))
            # 16 decades of magnitude: the delta list's carried sums fail its
            # error certificate at many positions (the direct re-sum path)
            fw = ff * 10.0 ** np.random.default_rng(B).uniform(-8, 8, size=ff.shape)
            assert_fp64_close(gpu_zeta(P, fw), O.zeta(fw), O.zeta(np.abs(fw)))
    finally:
        P.set_option("gather_pi_cfg", 0)


def test_host_buffers_and_inplace():
    n = 5000
    src, dst = W.window_dag(n, 2, 64, 5, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    f = W.int_values(n, 4, -1000, 1000, seed=1)
    g = P.zeta(f)                      # numpy in/out: staged by the library
    torch.cuda.synchronize()
    assert (g == O.zeta(f)).all()
    pinned = torch.from_numpy(f).pin_memory()
    out = torch.empty_like(pinned).pin_memory()
    P.zeta(pinned, out=out)
    torch.cuda.synchronize()
    assert (out.numpy() == O.zeta(f)).all()
    x = dev(f)
    P.zeta(x, out=x)                   # in place
    P.moebius(x, out=x)
    assert (host(x) == f).all()


def test_errors_through_abi():
    with pytest.raises(pz.PosetError) as e:
        pz.Poset(2, np.array([0, 1]), np.array([1, 0]))
    assert e.value.code == "ECYCLE"
    with pytest.raises(pz.PosetError) as e:
        pz.Poset(2, np.array([1]), np.array([1]))
    assert e.value.code == "ESELFLOOP"
    src, dst = W.paper_example_edges()
    with pytest.raises(pz.PosetError) as e:
        pz.Poset(12, src, dst, chains=[[2, 3]] + [[v] for v in range(12) if v not in (2, 3)])
    assert e.value.code == "ENOTCHAIN"
    with pytest.raises(pz.PosetError) as e:
        pz.Poset(12, src, dst, chains=[[v] for v in range(11)])
    assert e.value.code == "ENOTPARTITION"
    P = pz.Poset(12, src, dst)
    with pytest.raises(ValueError):
        P.zeta(dev(np.zeros((11, 1), np.int64)))
    with pytest.raises(TypeError):
        P.zeta(dev(np.zeros((12, 1), np.float32)))


def test_literal_C3_is_etoobig():
    n = 1_000_000
    src, dst = W.window_dag(n, 2, 1000, 0)
    with pytest.raises(pz.PosetError) as e:
        pz.Poset(n, src, dst)
    assert e.value.code == "ETOOBIG"


# ------------------------------------------------------ split-phase (dist)

@pytest.mark.parametrize("G", [1, 3, 4])
def test_split_phase_row_sharded_zeta(G):
    """Row-sharded single-function zeta (north star): G emulated ranks, each
    scans its slot range, the tails are combined into carries, the F ranges
    are concatenated (the all-gather) and each rank gathers its rows."""
    from paper_2211_13706_b200 import dist
    n = 40000
    src, dst = W.window_dag(n, 2, 1000, 0, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    for dtype in ("i64", "f64"):
        f = W.int_values(n, 2, -1000, 1000, 1) if dtype == "i64" else W.normal_values(n, 2, 1)
        g = dist.emulate_row_sharded_zeta(P, dev(f), G)
        got = host(g)
        if dtype == "i64":
            assert (got == O.zeta(f)).all()
        else:
            assert_fp64_close(got, O.zeta(f), O.zeta(np.abs(f)))


@pytest.mark.parametrize("G", [2, 3])
def test_sharded_index_rows(G):
    """The row-sharded index (poset_shard_rows): each of G
    handles keeps only its 4·k·n/G bytes of rows; the split-phase zeta over
    the G handles matches O2, rows outside a shard and the whole-table calls
    are refused, rank 0 keeps its Möbius tables, the others drop them."""
    from paper_2211_13706_b200 import dist
    n = 30011
    src, dst = W.window_dag(n, 2, 200, 5, forced=True)
    O = ChainOracle(n, src, dst)
    Ps = [pz.Poset(n, src, dst) for _ in range(G)]
    k = Ps[0].k
    for p, P in enumerate(Ps):
        lo, hi = dist.shard_index(P, rank=p, world=G)
        assert P.info()["table_bytes"] == 4 * k * (hi - lo)
    for dtype, B in (("i64", 1), ("i64", 32), ("f64", 3)):
        f = W.int_values(n, B, -10**12, 10**12, 2) if dtype == "i64" else W.normal_values(n, B, 2)
        got = host(dist.emulate_row_sharded_zeta(Ps, dev(f), G))
        if dtype == "i64":
            assert (got == O.zeta(f)).all(), B
        else:
            assert_fp64_close(got, O.zeta(f), O.zeta(np.abs(f)))
    F = torch.zeros((n + 1, 1), dtype=torch.int64, device="cuda")
    g = torch.zeros((n, 1), dtype=torch.int64, device="cuda")
    with pytest.raises(pz.PosetError):
        Ps[0].gather_rows(F, g, 0, n)            # beyond rank 0's rows
    with pytest.raises(pz.PosetError):
        Ps[0].zeta(dev(W.int_values(n, 1, -5, 5, 1)))
    h = W.int_values(n, 2, -10**15, 10**15, 4)
    assert (gpu_moebius(Ps[0], h) == O.moebius(h)).all()   # rank 0 keeps the ring tables
    with pytest.raises(pz.PosetError):
        Ps[1].moebius(dev(h))


# ------------------------------------------------------------ full sizes
#
# The configs bench.py times, at full size, compared ELEMENT BY ELEMENT with
# O2 (every x, every column): zeta of the bench's f, Möbius of an arbitrary
# int64 g (wrapping in Z/2^64, so not the image of a small f) under every
# schedule that applies, and a DFS-sampled check straight from the edge list
# (oracle_zeta_sampled_edges, pinned in test_oracle_pins.py) that shares
# nothing with O2's chains or niv table.

_FULL = {}


def _full(name, dtype, B):
    wl = W.make_workload(name, dtype=dtype, batch=B)
    if name not in _FULL:
        _FULL.clear()                       # one full-size poset resident at a time
        _FULL[name] = (pz.Poset(wl.n, wl.src, wl.dst), ChainOracle(wl.n, wl.src, wl.dst))
    return (wl, *_FULL[name])


def _sampled(wl, f, got):
    rng = np.random.default_rng(0)
    xs = np.unique(np.concatenate([np.array([0, wl.n - 1]), rng.integers(0, wl.n, 24)]))
    want, scale = zeta_sampled_edges(wl.n, wl.src, wl.dst, f, xs)
    if f.dtype == np.int64:
        assert (got[xs] == want).all()
    else:
        assert_fp64_close(got[xs], want, scale)


FULL_CASES = [("C3w", "f64", 1), ("C3w", "i64", 1), ("C4w", "i64", 64), ("C5w", "i64", 32),
              ("C5w", "f64", 32)]


@pytest.mark.parametrize("name,dtype,B", FULL_CASES)
def test_full_size_every_element_vs_O2(name, dtype, B):
    wl, P, O = _full(name, dtype, B)
    f = wl.values(seed=1)
    assert P.k == O.k and P.info()["ell"] == O.ell          # unique quantities (G15)
    x = dev(f)
    g = host(P.zeta(x))
    if dtype == "i64":
        want = O.zeta(f)
        bad = int((g != want).any(axis=1).sum())
        assert bad == 0, f"{bad} of {wl.n} rows differ"
        del want
        back = host(P.moebius(dev(g)))
        assert (back == f).all()
        # an arbitrary g (wraps): every schedule against O2 element by element
        h = W.int_values(wl.n, B, -10**17, 10**17, seed=11)
        want_h = O.moebius(h)
        hd = dev(h)
        for kern in [None] + kernels_for(P):
            if kern in (pz.MOEB_LEVEL, pz.MOEB_GRID, pz.MOEB_WARP) and P.info()["ell"] > 3000:
                continue                     # seconds per call at full size; covered above
            got = gpu_moebius_dev(P, hd, kern)
            bad = int((got != want_h).any(axis=1).sum())
            assert bad == 0, f"schedule {kern}: {bad} of {wl.n} rows differ"
    else:
        want = O.zeta(f)
        assert_fp64_close(g, want, O.zeta(np.abs(f)))
    _sampled(wl, f, g)


def gpu_moebius_dev(P, gd, kernel):
    if kernel is not None:
        P.set_option("moebius_kernel", kernel)
    try:
        return host(P.moebius(gd))
    finally:
        P.set_option("moebius_kernel", pz.MOEB_AUTO)


# ------------------------------------------------ sparse rows, no dense M (N1)

@pytest.mark.parametrize("inst", list(instances()), ids=lambda t: t[0])
def test_sparse_direct_rows_vs_dense_and_O2(inst, built):
    """POSET_SETUP_SPARSE: the U-rows built straight from the DAG (Thm. 4
    max-merge of the children's rows; the paper's sparse N,
    P:L292) equal the dense table's rows (same chains: the matching is
    deterministic), and zeta / Möbius over them match O2 bit-exactly."""
    name, n, src, dst = inst
    Pd, O = built(name, n, src, dst)
    Ps = pz.Poset(n, src, dst, sparse=True)
    info = Ps.info()
    assert info["zeta_sparse"] == 1 and info["moebius_kernel"] == pz.MOEB_CSR
    assert info["nnz"] == Pd.info()["nnz"] and info["k"] == Pd.k
    assert (Ps.export_mtable() == Pd.export_mtable()).all()
    for B in (1, 32, 5):
        f = W.int_values(n, B, -10**17, 10**17, seed=B + 40)
        assert (gpu_zeta(Ps, f) == O.zeta(f)).all(), B
        assert (gpu_moebius(Ps, f) == O.moebius(f)).all(), B
    ff = W.normal_values(n, 2, seed=8)
    assert_fp64_close(gpu_zeta(Ps, ff), O.zeta(ff), O.zeta(np.abs(ff)))
    with pytest.raises(pz.PosetError):
        gpu_moebius(Ps, f, pz.MOEB_RINGDF)        # schedules that need the dense table refuse


# ------------------------------------------- randomized schedule stress --
# No race checker runs on this pool, so the hand-rolled
# memory-ordering protocols of the ring schedules (mbarrier level phases,
# DSMEM st.async with transaction counts, RINGCW's tagged records, the CSR
# grid barrier) are exercised on many seeded random shapes: window DAGs of
# random window / degree / size (levels of 1 to > 96 elements, reach from a
# few ranks to the ring limit), layered DAGs of random width, each against O2
# bit-exact in Z/2^64 under every schedule that applies.

def _random_shapes():
    rng = np.random.default_rng(2026)
    for i in range(40):
        kind = rng.integers(0, 3)
        if kind < 2:
            n = int(rng.integers(300, 12000))
            Wd = int(rng.integers(3, 400))
            d = int(rng.integers(1, 5))
            yield f"win{i}_n{n}_W{Wd}_d{d}", n, *W.window_dag(n, d, Wd, int(rng.integers(0, 1000)),
                                                              forced=bool(kind))
        else:
            L, w = int(rng.integers(8, 80)), int(rng.integers(4, 120))
            yield f"lay{i}_{L}x{w}", L * w, *W.layered_dag(L, w, int(rng.integers(1, 4)), int(rng.integers(0, 1000)),
                                                            forced=True)


_SEEN = set()


@pytest.mark.parametrize("shape", list(_random_shapes()), ids=lambda t: t[0])
def test_schedules_on_random_shapes(shape):
    name, n, src, dst = shape
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    _SEEN.update(kernels_for(P))
    rng = np.random.default_rng(n)
    for B in (1, int(rng.integers(2, 40))):
        h = W.int_values(n, B, -10**17, 10**17, seed=B + 7)
        want = O.moebius(h)
        hd = dev(h)
        for kern in [None] + kernels_for(P):
            if kern in (pz.MOEB_LEVEL, pz.MOEB_GRID, pz.MOEB_WARP) and P.info()["ell"] > 2000:
                continue
            helpers = (1, 2, 3) if kern in (pz.MOEB_RINGCL, pz.MOEB_RINGCW) else (0,)
            for nh in helpers:
                P.set_option("ringcl_helpers", nh)
                got = gpu_moebius_dev(P, hd, kern)
                assert (got == want).all(), (name, B, kern, nh)
        P.set_option("ringcl_helpers", 0)
        f = W.int_values(n, B, -10**17, 10**17, seed=B + 8)
        assert (gpu_zeta(P, f) == O.zeta(f)).all(), (name, B)


def test_random_shapes_reached_the_ring_schedules():
    """The stress set above is not vacuous: it ran RINGDF, RINGCL and RINGCW
    and the sparse-row schedule on some shapes."""
    if not _SEEN:
        pytest.skip("run together with test_schedules_on_random_shapes")
    assert {pz.MOEB_RINGDF, pz.MOEB_RINGCL, pz.MOEB_RINGCW, pz.MOEB_CSR} <= _SEEN, _SEEN


@pytest.mark.parametrize("mode", [1, 2])
def test_scan_modes(mode):
    """Both zeta scans (single pass with a decoupled look-back, and
    the three-kernel scan) against O2 over batch sizes that cover 1..32
    columns per tile, several column groups and many tiles (long chains cross
    hundreds of tiles), int64 bit-exact and fp64 within the tolerance."""
    n = 60013
    src, dst = W.window_dag(n, 2, 64, 11, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    P.set_option("scan_mode", mode)
    try:
        for B in (1, 3, 32, 33, 64, 96):
            f = W.int_values(n, B, -10**15, 10**15, seed=B + 30)
            assert (gpu_zeta(P, f) == O.zeta(f)).all(), B
        ff = W.normal_values(n, 32, seed=5)
        assert_fp64_close(gpu_zeta(P, ff), O.zeta(ff), O.zeta(np.abs(ff)))
    finally:
        P.set_option("scan_mode", 0)


def test_pipelined_zeta_and_moebius_on_two_streams():
    """The batched pipeline (bench --pipeline): zetas on one
    stream, with the persistent gather grid sized to the SMs the Möbius leaves
    free (option zeta_sms), overlapping ring-family Möbius calls on a second,
    high-priority stream -- the two use disjoint scratch lanes
    (include/poset.h), so the library does not serialise them.  Every batch:
    zeta vs O2 bit-exact (int64) and the Möbius round trip exact; then two
    zetas on two streams (same lane: ordered by the library) and a 3-SM zeta
    budget, both vs O2."""
    n = 120_000
    src, dst = W.window_dag(n, 2, 64, 3, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    B = 32
    fs = [W.int_values(n, B, -10**15, 10**15, seed=50 + i) for i in range(4)]
    xs = [dev(f) for f in fs]
    P.moebius(P.zeta(xs[0]))
    torch.cuda.synchronize()
    info = P.info()
    assert info["moebius_kernel"] in (pz.MOEB_RINGCL, pz.MOEB_RINGDF)
    assert 0 < info["moebius_sms"] < info["num_sms"]
    P.set_option("zeta_sms", info["num_sms"] - info["moebius_sms"])
    try:
        cur = torch.cuda.current_stream()
        s_z = torch.cuda.Stream(priority=0)
        s_m = [torch.cuda.Stream(priority=-1), torch.cuda.Stream(priority=-1)]
        for st in (s_z, *s_m):
            st.wait_stream(cur)
        gs = [torch.empty_like(x) for x in xs]
        ys = [torch.empty_like(x) for x in xs]
        ev = [torch.cuda.Event() for _ in xs]
        for i, x in enumerate(xs):        # zeta i+1.. queue behind zeta i, Möbius i overlaps them;
            P.zeta(x, out=gs[i], stream=s_z)   # Möbius on alternating streams (double-buffered
            ev[i].record(s_z)                  # rank-major g, solves ordered by the library)
            s_m[i % 2].wait_event(ev[i])
            P.moebius(gs[i], out=ys[i], stream=s_m[i % 2])
        torch.cuda.synchronize()
        for i, f in enumerate(fs):
            assert (host(gs[i]) == O.zeta(f)).all(), i
            assert (host(ys[i]) == f).all(), i
        a, b = torch.cuda.Stream(), torch.cuda.Stream()
        a.wait_stream(cur)
        b.wait_stream(cur)
        g1, g2 = torch.empty_like(xs[1]), torch.empty_like(xs[2])
        P.zeta(xs[1], out=g1, stream=a)
        P.zeta(xs[2], out=g2, stream=b)
        torch.cuda.synchronize()
        assert (host(g1) == O.zeta(fs[1])).all()
        assert (host(g2) == O.zeta(fs[2])).all()
        P.set_option("zeta_sms", 3)
        assert (gpu_zeta(P, fs[3]) == O.zeta(fs[3])).all()
    finally:
        P.set_option("zeta_sms", 0)


@pytest.mark.parametrize("nfl", [2, 3, 4])
def test_solves_in_flight_vs_O2(nfl):
    """Option solves_inflight = 2..4 (bench --inflight): that
    many batches' solves (2: RINGCL with one helper SM per column; 3 / 4:
    RINGDF, one SM per column) run side by side on as many streams, each with
    its own rank-major input lane, while the next zetas run on the remaining
    SMs.  Möbius of arbitrary (wrapping) int64 g vs O2
    bit-exact for every batch, and the zeta -> Möbius round trip exact."""
    n = 120_000
    src, dst = W.window_dag(n, 2, 64, 3, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    B = 32
    gs_h = [W.int_values(n, B, -2**62, 2**62, seed=70 + i) for i in range(6)]
    fs = [W.int_values(n, B, -10**15, 10**15, seed=80 + i) for i in range(4)]
    if nfl == 2:
        P.set_option("ringcl_helpers", 1)
    else:
        P.set_option("moebius_kernel", pz.MOEB_RINGDF)
    P.set_option("solves_inflight", nfl)
    try:
        P.moebius(P.zeta(dev(fs[0])))
        torch.cuda.synchronize()
        info = P.info()
        assert info["moebius_kernel"] == (pz.MOEB_RINGCL if nfl == 2 else pz.MOEB_RINGDF)
        assert nfl * info["moebius_sms"] < info["num_sms"]
        cur = torch.cuda.current_stream()
        s_m = [torch.cuda.Stream(priority=-1) for _ in range(nfl)]
        s_z = torch.cuda.Stream(priority=0)
        for st in (s_z, *s_m):
            st.wait_stream(cur)
        # (a) arbitrary g, alternating streams: solves i and i+1 overlap
        gd = [dev(g) for g in gs_h]
        out = [torch.empty_like(g) for g in gd]
        for st in s_m:
            st.wait_stream(cur)
        for i, g in enumerate(gd):
            P.moebius(g, out=out[i], stream=s_m[i % nfl])
        torch.cuda.synchronize()
        for i, g in enumerate(gs_h):
            assert (host(out[i]) == O.moebius(g)).all(), i
        # (b) the pipeline: zetas on the free SMs beside two solves
        P.set_option("zeta_sms", info["num_sms"] - nfl * info["moebius_sms"])
        xs = [dev(f) for f in fs]
        zs = [torch.empty_like(x) for x in xs]
        ys = [torch.empty_like(x) for x in xs]
        ev = [torch.cuda.Event() for _ in xs]
        for i, x in enumerate(xs):
            P.zeta(x, out=zs[i], stream=s_z)
            ev[i].record(s_z)
            s_m[i % nfl].wait_event(ev[i])
            P.moebius(zs[i], out=ys[i], stream=s_m[i % nfl])
        torch.cuda.synchronize()
        for i, f in enumerate(fs):
            assert (host(zs[i]) == O.zeta(f)).all(), i
            assert (host(ys[i]) == f).all(), i
    finally:
        P.set_option("zeta_sms", 0)
        P.set_option("ringcl_helpers", 0)
        P.set_option("moebius_kernel", pz.MOEB_AUTO)
        P.set_option("solves_inflight", 1)


@pytest.mark.parametrize("G", [1, 3])
def test_nvls_fused_scan_row_sharded_zeta(G):
    """the row-sharded zeta with the F all-gather fused into
    the scan epilogue -- every F row stored with multimem.st through an NVLS
    multicast address (poset_scan_slots_mc) -- for G emulated ranks on one
    GPU (all bound to the one device's buffer), vs O2: int64 bit-exact, fp64
    within the tolerance.  Skips when the driver / device has no multicast."""
    from paper_2211_13706_b200 import dist as pdist
    n = 30011
    src, dst = W.window_dag(n, 2, 64, 7, forced=True)
    P, O = pz.Poset(n, src, dst), ChainOracle(n, src, dst)
    try:
        buf = pz.NvlsBuffer([0], pdist.nvls_buffer_bytes(n, G, 8))
    except pz.PosetError as e:   # pragma: no cover - depends on the box
        pytest.skip(f"no NVLS multicast here: {e}")
    try:
        for B in (1, 3, 8):
            f = W.int_values(n, B, -10**15, 10**15, seed=B + 60)
            g = pdist.nvls_row_sharded_zeta([P] * G, [dev(f)] * G, buf)
            assert (host(g) == O.zeta(f)).all(), B
        ff = W.normal_values(n, 2, seed=9)
        g = pdist.nvls_row_sharded_zeta([P] * G, [dev(ff)] * G, buf)
        assert_fp64_close(host(g), O.zeta(ff), O.zeta(np.abs(ff)))
    finally:
        buf.close()
