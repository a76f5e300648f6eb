"""Pins of the CPU oracle against what the paper and mathematics fix
(``-m "not gpu"``).  Nothing here touches the CUDA path.

Sources of truth: the paper's printed 12-node example (tests/golden/*.txt,
each citing its PAPER.md lines), closed forms (Yates subset sums on the
Boolean lattice, cumsum / diff on a chain, identity on an antichain,
μ(S,T) = (-1)^|T\\S| on the Boolean lattice), brute force on tiny inputs
(width, maximum matching, longest chain), and invariants (Thm. 3, μ∘ζ = id,
linearity, decomposition invariance).
"""
import numpy as np
import pytest

from conftest import assert_fp64_close, load_facts, load_matrix
from oracle import brute
from oracle.chain import ChainOracle, zeta_sampled_edges
import workloads as W

facts = load_facts()
PAPER_CHAINS = [[int(v) - 1 for v in c.split(",")] for c in facts["chains"].split(";")]


def ids(s):
    return [int(v) - 1 for v in s.split(",")]


# ---------------------------------------------------------------- example --

def test_example_adjacency_matches_edges(paper_example):
    n, src, dst = paper_example
    A = load_matrix("A.txt")
    A2 = np.zeros((12, 12), dtype=np.int64)
    A2[src, dst] = 1
    assert (A == A2).all()


def test_O1_closure_is_printed_Z(paper_example):
    n, src, dst = paper_example
    Z = load_matrix("Z.txt")
    assert (brute.zeta_matrix(n, src, dst) == Z).all()


def test_O1_mobius_recursion_is_printed_M(paper_example):
    n, src, dst = paper_example
    M = load_matrix("M.txt")
    assert (np.array(brute.mobius_function(n, src, dst)) == M).all()
    Z = load_matrix("Z.txt")
    assert (Z @ M == np.eye(12, dtype=np.int64)).all()          # Cor. 1: Z^-1 = M


def test_O1_transforms_on_example_match_printed_matrices(paper_example):
    n, src, dst = paper_example
    Z, M = load_matrix("Z.txt"), load_matrix("M.txt")
    f = W.int_values(12, 5, -100, 100, seed=3)
    assert (brute.zeta(n, src, dst, f) == Z @ f).all()
    g = W.int_values(12, 5, -100, 100, seed=4)
    assert (brute.moebius(n, src, dst, g) == M @ g).all()
    ff = W.normal_values(12, 3, seed=5)
    assert_fp64_close(brute.zeta(n, src, dst, ff), Z @ ff, Z @ np.abs(ff))


def test_example_downset_and_g_x1(paper_example):
    n, src, dst = paper_example
    down = brute.downsets(n, src, dst)
    assert sorted(v for v in range(12) if (down[3] >> v) & 1) == ids(facts["down_4"])
    e = np.eye(12, dtype=np.int64)
    g = brute.zeta(n, src, dst, e)             # column y = zeta of indicator of y
    assert sorted(np.nonzero(g[0])[0].tolist()) == ids(facts["g_x1"])


def test_O2_injected_chains_reproduce_printed_N(paper_example):
    n, src, dst = paper_example
    O = ChainOracle(n, src, dst, chains=PAPER_CHAINS)
    N = load_matrix("N.txt")                   # paper labels, -1 = ∞
    want = np.where(N > 0, N - 1, -1)
    assert (O.niv_dense() == want).all()
    assert O.nnz == int(facts["nnz_N"]) == int((N > 0).sum())
    assert O.niv_dense()[3].tolist() == ids(facts["niv_4"])


def test_O2_factorisation_U_V_Vinv_B(paper_example):
    n, src, dst = paper_example
    O = ChainOracle(n, src, dst, chains=PAPER_CHAINS)
    niv = O.niv_dense()
    chain, nxt, _, _ = O.chains()
    U = np.zeros((12, 12), dtype=np.int64)
    for x in range(12):
        for v in niv[x]:
            if v >= 0:
                U[x, v] = 1
    V = np.zeros((12, 12), dtype=np.int64)
    for x in range(12):
        y = x
        while True:
            V[x, y] = 1
            if nxt[y] == y:
                break
            y = nxt[y]
    Vinv = np.eye(12, dtype=np.int64)
    for x in range(12):
        if nxt[x] != x:
            Vinv[x, nxt[x]] = -1
    assert (U == load_matrix("U.txt")).all()
    assert (V == load_matrix("V.txt")).all()
    assert (Vinv == load_matrix("Vinv.txt")).all()
    assert (U @ V == load_matrix("Z.txt")).all()                # Eq. zfac
    # P = (1,2,4,12,11,8,5)(3,9,10,6) as a position -> vertex map
    sigma = list(range(12))
    for cyc in facts["perm_cycles"].split(";"):
        c = ids(cyc)
        for a, b in zip(c, c[1:] + c[:1]):
            sigma[a] = b
    B = V[np.ix_(sigma, sigma)]
    assert (B == load_matrix("B.txt")).all()
    Binv = load_matrix("Binv.txt")
    assert (B @ Binv == np.eye(12, dtype=np.int64)).all()


def test_example_operation_counts(paper_example):
    n, src, dst = paper_example
    O = ChainOracle(n, src, dst, chains=PAPER_CHAINS)
    k = O.k
    assert n - k == int(facts["ops_V"])              # P^-1 B P: n - k
    assert O.nnz - n == int(facts["ops_U"])          # U: nnz - n
    assert O.nnz - k == int(facts["ops_total"])      # total nnz - k
    Z = load_matrix("Z.txt")
    # erratum G6: the printed Z has nnz 52, so Z costs nnz(Z) - n = 40, not 39
    assert int(Z.sum()) - n == 40 != int(facts["ops_Z_printed"])


def test_example_width_levels_and_own_matching(paper_example):
    n, src, dst = paper_example
    O = ChainOracle(n, src, dst)
    assert O.k == int(facts["width"]) == brute.width_bruteforce(n, src, dst)
    assert O.ell == int(facts["ell"]) == brute.longest_chain(n, src, dst)
    Z = brute.zeta_matrix(n, src, dst)
    ac = ids(facts["antichain"])
    assert all(Z[a, b] == 0 for a in ac for b in ac if a != b)
    lc = ids(facts["longest_chain"])
    assert all(Z[a, b] == 1 for a, b in zip(lc, lc[1:]))
    Zp = load_matrix("Z.txt")
    Mp = load_matrix("M.txt")
    f = W.int_values(12, 4, -50, 50, seed=9)
    assert (O.zeta(f) == Zp @ f).all()
    assert (O.moebius(f) == Mp @ f).all()


# ---------------------------------------------------------- closed forms --

@pytest.mark.parametrize("bits", [1, 3, 6, 9])
def test_yates_pins_O1_and_O2_on_boolean_lattice(bits):
    n = 1 << bits
    src, dst = W.boolean_lattice(bits)
    f = W.int_values(n, 3, -1000, 1000, seed=bits)
    want = brute.yates_zeta(bits, f)
    O = ChainOracle(n, src, dst)
    assert (O.zeta(f) == want).all()
    assert (O.moebius(want) == f).all()
    assert (brute.yates_moebius(bits, want) == f).all()
    if n <= 128:
        assert (brute.zeta(n, src, dst, f) == want).all()
        assert (brute.moebius(n, src, dst, want) == f).all()
    ff = W.normal_values(n, 2, seed=bits)
    wf = brute.yates_zeta(bits, ff)
    scale = brute.yates_zeta(bits, np.abs(ff))
    assert_fp64_close(O.zeta(ff), wf, scale)
    assert_fp64_close(O.moebius(wf), brute.yates_moebius(bits, wf), brute.yates_zeta(bits, np.abs(ff)))
    # width of 2^bits is C(bits, bits//2) (Sperner); path cover attains it
    from math import comb
    assert O.k == comb(bits, bits // 2)
    assert O.ell == bits + 1


def test_yates_itself_on_tiny_lattice():
    # Yates vs explicit subset enumeration (definition of the powerset zeta)
    bits = 4
    f = W.int_values(16, 1, -9, 9, seed=0)[:, 0]
    g = brute.yates_zeta(bits, f.reshape(-1, 1))[:, 0]
    for S in range(16):
        assert g[S] == sum(f[T] for T in range(16) if T & S == T)


def test_boolean_mobius_function_closed_form():
    bits = 3
    src, dst = W.boolean_lattice(bits)
    M = brute.mobius_function(8, src, dst)
    for S in range(8):
        for T in range(8):
            want = (-1) ** bin(T & ~S).count("1") if (S & T) == S else 0
            assert M[T][S] == want


@pytest.mark.parametrize("n", [1, 2, 7, 40])
def test_chain_closed_form(n):
    src, dst = W.chain_dag(n)
    f = W.int_values(n, 3, -100, 100, seed=n)
    O = ChainOracle(n, src, dst)
    assert O.k == 1 and O.q == n and O.ell == n
    assert (O.zeta(f) == np.cumsum(f, axis=0)).all()
    d = np.diff(f, axis=0, prepend=np.zeros((1, 3), np.int64))
    assert (O.moebius(f) == d).all()
    assert (brute.zeta(n, src, dst, f) == np.cumsum(f, axis=0)).all()
    assert (brute.moebius(n, src, dst, f) == d).all()


@pytest.mark.parametrize("n", [1, 5, 33])
def test_antichain_identity(n):
    src, dst = W.antichain_dag(n)
    f = W.normal_values(n, 2, seed=n)
    O = ChainOracle(n, src, dst)
    assert O.k == n and O.ell == 1 and O.nnz == n
    assert (O.zeta(f) == f).all() and (O.moebius(f) == f).all()
    assert (brute.zeta(n, src, dst, f) == f).all()


# ------------------------------------------------------ O2 vs O1, invariants

def small_instances():
    yield "C1", 1000, *W.window_dag(1000, 3, 50, 0)
    yield "C1_300", 300, *W.window_dag(300, 3, 50, 7)
    yield "C3lit", 600, *W.window_dag(600, 2, 100, 1)
    yield "C3w", 700, *W.window_dag(700, 2, 100, 2, forced=True)
    yield "C4lit", 6 * 32, *W.layered_dag(6, 32, 3, 3)
    yield "C4w", 8 * 32, *W.layered_dag(8, 32, 3, 4, forced=True)
    yield "C5w", 900, *W.window_dag(900, 2, 64, 5, forced=True)
    yield "C5lit", 500, *W.window_dag(500, 2, 64, 6)
    yield "ER4", 400, *W.erdos_renyi(400, 4, 8)
    yield "ER6", 300, *W.erdos_renyi(300, 6, 9)


@pytest.mark.parametrize("inst", list(small_instances()), ids=lambda t: t[0])
def test_O2_equals_O1_and_round_trip(inst):
    name, n, src, dst = inst
    O = ChainOracle(n, src, dst)
    f = W.int_values(n, 3, -1000, 1000, seed=11)
    g1 = brute.zeta(n, src, dst, f)
    g2 = O.zeta(f)
    assert (g1 == g2).all()
    assert (O.moebius(g2) == f).all()                       # μ∘ζ = id (exact ring)
    assert (brute.moebius(n, src, dst, g1) == f).all()
    h = W.int_values(n, 2, -10**17, 10**17, seed=12)         # arbitrary g, wraparound
    assert (O.moebius(h) == brute.moebius(n, src, dst, h)).all()
    ff = W.normal_values(n, 2, seed=13)
    assert_fp64_close(O.zeta(ff), brute.zeta(n, src, dst, ff), brute.zeta_abs(n, src, dst, ff))
    assert O.ell == brute.longest_chain(n, src, dst)


@pytest.mark.parametrize("inst", list(small_instances())[:6], ids=lambda t: t[0])
def test_thm3_reachability_identity(inst):
    """Thm. 3: ↓x ∩ Z_j is the prefix of chain j up to niv_j(x),
    so |↓x ∩ Z_j| = (bottom-up position of niv_j(x)) + 1, and the prefixes
    partition ↓x."""
    name, n, src, dst = inst
    O = ChainOracle(n, src, dst)
    niv = O.niv_dense()
    chain, nxt, _, _ = O.chains()
    # bottom-up positions
    pos = np.zeros(n, dtype=np.int64)
    has_pred = np.zeros(n, bool)
    has_pred[nxt[nxt != np.arange(n)]] = True
    for top in np.nonzero(~has_pred)[0]:
        seq = [top]
        while nxt[seq[-1]] != seq[-1]:
            seq.append(nxt[seq[-1]])
        for p, v in enumerate(reversed(seq)):
            pos[v] = p
    down = brute.downsets(n, src, dst)
    for x in range(0, n, max(1, n // 97)):
        members = [y for y in range(n) if (down[x] >> y) & 1]
        cnt = np.bincount(chain[members], minlength=O.k)
        m = np.where(niv[x] >= 0, pos[np.maximum(niv[x], 0)], -1)
        assert (cnt == m + 1).all()


def test_decomposition_invariance():
    n = 400
    src, dst = W.window_dag(n, 3, 40, 21)
    f = W.int_values(n, 2, -1000, 1000, seed=1)
    a = ChainOracle(n, src, dst)
    singles = ChainOracle(n, src, dst, chains=[[v] for v in range(n)])
    assert singles.k == n
    assert (a.zeta(f) == singles.zeta(f)).all()
    assert (a.moebius(f) == singles.moebius(f)).all()


def test_linearity():
    n = 500
    src, dst = W.window_dag(n, 2, 64, 3, forced=True)
    O = ChainOracle(n, src, dst)
    a = W.int_values(n, 2, -10**6, 10**6, seed=1)
    b = W.int_values(n, 2, -10**6, 10**6, seed=2)
    assert (O.zeta(3 * a - b) == 3 * O.zeta(a) - O.zeta(b)).all()
    assert (O.moebius(3 * a - b) == 3 * O.moebius(a) - O.moebius(b)).all()


@pytest.mark.parametrize("seed", range(6))
def test_matching_is_maximum_and_path_cover(seed):
    """Alg. 1: k = n - |maximum matching of G'| (König), brute-forced; the
    chains are vertex-disjoint paths of E (next edges are DAG edges)."""
    n = 9
    src, dst = W.erdos_renyi(n, 3.0, seed)
    if src.shape[0] > 20:
        src, dst = src[:20], dst[:20]
    O = ChainOracle(n, src, dst)
    assert O.k == n - brute.max_matching_bruteforce(n, src, dst)
    chain, nxt, _, _ = O.chains()
    E = set(zip(src.tolist(), dst.tolist()))
    for v in range(n):
        if nxt[v] != v:
            assert (v, int(nxt[v])) in E and chain[v] == chain[nxt[v]]
    assert O.k >= brute.width_bruteforce(n, src, dst)       # Dilworth lower bound


def test_sampled_brute_zeta_matches(paper_example):
    n = 2000
    src, dst = W.window_dag(n, 2, 64, 0, forced=True)
    O = ChainOracle(n, src, dst)
    f = W.normal_values(n, 4, seed=2)
    xs = np.array([0, 1, 63, 64, 999, 1999])
    g, ab = O.zeta_sampled(f, xs)
    full = brute.zeta(n, src, dst, f)
    assert_fp64_close(g, full[xs], ab)
    fi = W.int_values(n, 4, -100, 100, seed=3)
    gi, _ = O.zeta_sampled(fi, xs)
    assert (gi == brute.zeta(n, src, dst, fi)[xs]).all()


def test_errors():
    with pytest.raises(ValueError):
        ChainOracle(2, np.array([0, 1]), np.array([1, 0]))        # 2-cycle
    with pytest.raises(ValueError):
        ChainOracle(2, np.array([1]), np.array([1]))              # self loop
    with pytest.raises(ValueError):   # 3,4 incomparable (P:L247 antichain)
        ChainOracle(12, *W.paper_example_edges(), chains=[[2, 3]] + [[v] for v in range(12) if v not in (2, 3)])
    with pytest.raises(brute.CycleError):
        brute.downsets(2, np.array([0, 1]), np.array([1, 0]))


def _edge_sample_cases():
    s, d = W.window_dag(1200, 2, 64, 3, forced=True)
    yield "window_w", 1200, s, d
    s, d = W.window_dag(900, 3, 50, 1)
    yield "window_lit", 900, s, d
    s, d = W.layered_dag(6, 64, 3, 2, forced=True)
    yield "layered", 6 * 64, s, d
    s, d = W.boolean_lattice(8)
    yield "bool8", 256, s, d
    # duplicate edges (each edge twice, shuffled) and an isolated vertex
    s, d = W.window_dag(700, 2, 30, 5)
    rng = np.random.default_rng(9)
    perm = rng.permutation(2 * s.shape[0])
    yield "dups", 701, np.concatenate([s, s])[perm], np.concatenate([d, d])[perm]


@pytest.mark.parametrize("case", list(_edge_sample_cases()), ids=lambda c: c[0])
def test_zeta_sampled_edges_is_pinned_to_O1(case):
    """The DFS checker used at full size (oracle_zeta_sampled_edges) against
    the O1 closure sums, Eq. inv-formula: int64 bit-exact in Z/2^64,
    fp64 within the tolerance, and its Σ|f| scale equal to O1's zeta(|f|)."""
    name, n, src, dst = case
    rng = np.random.default_rng(1)
    xs = np.unique(np.concatenate([[0, n - 1], rng.integers(0, n, 40)]))
    fi = W.int_values(n, 3, -10**18, 10**18, seed=4)          # wraps in Z/2^64
    gi, none = zeta_sampled_edges(n, src, dst, fi, xs)
    assert none is None
    assert (gi == brute.zeta(n, src, dst, fi)[xs]).all()
    ff = W.normal_values(n, 2, seed=5)
    gf, ab = zeta_sampled_edges(n, src, dst, ff, xs)
    assert_fp64_close(gf, brute.zeta(n, src, dst, ff)[xs], brute.zeta_abs(n, src, dst, ff)[xs])
    np.testing.assert_allclose(ab, brute.zeta_abs(n, src, dst, ff)[xs], rtol=1e-12)


@pytest.mark.parametrize("case", list(_edge_sample_cases()), ids=lambda c: c[0])
def test_parallel_oracle_equals_sequential(case):
    """The OpenMP CPU baseline (chains / rows in parallel; Möbius by Alg. 5,
    antichain by antichain) sums the same terms in the same
    order as the sequential Algs. 3-4: identical bits for int64 and fp64."""
    name, n, src, dst = case
    O = ChainOracle(n, src, dst)
    for f in (W.int_values(n, 5, -10**18, 10**18, seed=2), W.normal_values(n, 3, seed=3)):
        g = O.zeta(f)
        assert np.array_equal(O.zeta_omp(f), g)
        assert np.array_equal(O.moebius_omp(g), O.moebius(g))
