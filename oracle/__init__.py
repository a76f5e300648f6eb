"""CPU ORACLE for the chain-decomposition zeta / Moebius transforms.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import, call,
link or execute anything under ``oracle/``.  The product package
``paper_2211_13706_b200`` never imports it, and the two share no code: the
only module both use is ``workloads`` (seeded random draws, no arithmetic of
the method).

Two independent oracles:

* **O1** ``oracle.brute`` -- the plain definitions (PAPER.md Eq. inv-formula
  P:L11-16, Cor. 1 P:L143-151): transitive closure by DP over children,
  g = Z f by direct sums, f = Z^-1 g by triangular back-substitution
  (P:L155-156), the Moebius-function recursion (Thm. 1), and the
  Boolean-lattice Yates subset-sum transform as a closed form.
* **O2** ``oracle.chain`` -- the paper's sequential chain algorithm, step by
  step in plain C (``chain_oracle.c``): Alg. 1 matching, Alg. 6 levels,
  Alg. 2 niv, Alg. 3 zeta, Alg. 4 Moebius.  Used as the oracle for large n.

Pins (``tests/test_oracle_pins.py``, ``-m "not gpu"``): the paper's printed
12-node Z, M, N, U, V, B^-1, V^-1, niv(4), down-set of 4, op counts; Yates on
Boolean lattices; closed forms for chains and antichains; mu∘zeta = id;
Thm. 3 reachability identity; brute-force width / matching on tiny inputs.
Every function here is pinned; none is "parity unpinned".
"""
