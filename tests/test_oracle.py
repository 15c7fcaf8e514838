"""Pin the CPU oracle (oracle/sap_oracle.c) before trusting it.

1. Golden vectors produced by the UNMODIFIED reference (tests/golden/*.npz,
   made by tests/golden/make_golden.py through oracle/_ref) must be
   reproduced bit for bit.
2. The reference's own known-answer tests are restated against the oracle
   (proj/tests/test_banded_core.cpp, test_spike.cpp, test_krylov.cpp).
3. Where oracle/_ref is loadable, random cases are cross-checked bit for bit.
"""
import glob
import os

import numpy as np
import pytest

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "*.npz")) if not p.endswith("criterion2.npz"))


def _load(path):
    z = np.load(path)
    return {k: z[k] for k in z.files}


@pytest.mark.parametrize("path", CASES, ids=[os.path.basename(p)[:-4] for p in CASES])
def test_oracle_reproduces_reference_goldens(oracle, path):
    g = _load(path)
    n, k, d, seed, p = int(g["n"]), int(g["k"]), float(g["d"]), int(g["seed"]), int(g["p"])
    band, rhs = oracle.random_banded(n, k, d, seed)
    assert np.array_equal(band, g["band"]) and np.array_equal(rhs, g["rhs"])
    f = oracle.factor_blocks(n, k, band, p, True)
    for key in ("lu", "ul", "boosts", "boosts_ul", "norms"):
        assert np.array_equal(f[key], g[key]), key
    if p > 1:
        s = oracle.spikes(n, k, band, p)
        for key in ("B", "C", "vb", "wt", "rbar", "rbar_boosts"):
            assert np.array_equal(s[key], g[key]), key
    for kind, tag in ((0, "c"), (1, "d")):
        assert np.array_equal(oracle.apply(n, k, band, p, kind, rhs), g["m_" + tag])
        x, st = oracle.solve_banded(n, k, band, rhs, p, kind, max_iterations=100)
        assert st["iterations"] == float(g["it_" + tag])
        assert st["failure"] == int(g["fail_" + tag])
        assert np.array_equal(st["residual_history"], g["hist_" + tag])
        assert np.array_equal(x, g["x_" + tag])


def test_oracle_reproduces_acceptance_criterion2(oracle):
    """proj/tests/acceptance.cpp:103-154 per-seed iterations and residuals (and
    proj/test_output.txt:26 for the failing d = 0.1 seeds)."""
    g = np.load(os.path.join(GOLDEN, "criterion2.npz"))
    for d, seed, it, res, fail in g["rows"]:
        band, rhs = oracle.random_banded(10000, 50, float(d), int(seed))
        _, st = oracle.solve_banded(10000, 50, band, rhs, 8, 0, max_iterations=50)
        assert st["iterations"] == it and st["final_relative_residual"] == res and st["failure"] == int(fail)
    # the published failing-seed residuals (proj/test_output.txt:26)
    d01 = [r for r in g["rows"] if r[0] == 0.1]
    assert ["%.3g" % r[3] for r in d01] == ["2.65e-10", "5.66e-09", "5.75e-10", "7.48e-08", "4.79e-06"]
    band, rhs = oracle.random_banded(10000, 10, 1.0, 1)
    _, st = oracle.solve_banded(10000, 10, band, rhs, 4, 1)
    assert st["iterations"] == g["config1"][0] == 3.25


def test_known_answer_zero_pivot_boost(oracle):
    """proj/tests/test_banded_core.cpp:257-277."""
    band = np.zeros(2 * 3)
    band[0 * 3 + (0 - 1 + 1) + 1 - 1] = 0.0
    # a(0,1) = 1 at slot 1*3 + (0-1+1) = 3; a(1,0) = 1 at slot 0*3 + (1-0+1) = 2
    band[3] = 1.0
    band[2] = 1.0
    f = oracle.factor_blocks(2, 1, band, 1, False, boost_eps=1e-6)
    lu = f["lu"]
    assert f["boosts"][0] == 1 and f["norms"][0] == 1.0
    assert lu[1] == 1e-6 and lu[3] == 1.0
    l10 = lu[2]
    assert l10 == 1.0 / 1e-6 and lu[4] == -l10


def test_identity_factors(oracle):
    """proj/tests/test_banded_core.cpp:241-255."""
    n, k = 5, 2
    band = np.zeros(n * (2 * k + 1))
    band[np.arange(n) * (2 * k + 1) + k] = 1.0
    f = oracle.factor_blocks(n, k, band, 1, True)
    assert f["boosts"][0] == 0 and f["boosts_ul"][0] == 0
    assert np.array_equal(f["lu"], band) and np.array_equal(f["ul"], band)


def test_partition_layout(oracle):
    """proj/tests/test_banded_core.cpp:185-212."""
    s, o = oracle.partition_layout(10, 3, 1)
    assert list(s) == [4, 3, 3] and list(o) == [0, 4, 7, 10]
    with pytest.raises(oracle.OracleError):
        oracle.partition_layout(10, 3, 2)
    lib = oracle.lib()
    assert [lib.sapo_max_feasible_partitions(*a) for a in [(10, 2), (10, 0), (7, 3), (12, 3), (5, 3)]] == [2, 10, 1, 2, 0]


def test_ul_is_reversed_lu_bitwise(oracle):
    """SURVEY §8c identity used by the GPU UL kernel: UL(A) == rev(LU(rev(A)))."""
    for seed in range(6):
        n, k = 60 + seed, 1 + seed
        band = oracle.random_banded(n, k, 0.3 + 0.4 * seed, 100 + seed, with_rhs=False)
        ul = oracle.factor_blocks(n, k, band, 1, True)["ul"]
        lu_rev = oracle.factor_blocks(n, k, band[::-1].copy(), 1, False)["lu"]
        assert np.array_equal(ul, lu_rev[::-1])


def test_identity_blocks_tips_are_couplings(oracle):
    """proj/tests/test_spike.cpp:94-134 (identity diagonal blocks)."""
    n, k = 8, 2
    w = 2 * k + 1
    band = np.zeros(n * w)

    def put(i, j, v):
        band[j * w + (i - j + k)] = v

    for i in range(n):
        put(i, i, 1.0)
    put(2, 4, 0.5); put(3, 4, 0.25); put(3, 5, 0.5); put(4, 2, 0.3); put(4, 3, 0.1); put(5, 3, 0.3)
    s = oracle.spikes(n, k, band, 2)
    assert np.array_equal(s["vb"], s["B"]) and np.array_equal(s["wt"], s["C"])


def test_krylov_identity_quarter_iteration(oracle):
    """proj/tests/test_krylov.cpp:62-76 through the identity (k = 0) band and no preconditioner."""
    n = 10
    b = oracle.uniform_stream(101, n)
    band = np.ones(n)
    x, st = oracle.solve_banded(n, 0, band, b, 1, 3)
    assert st["converged"] and st["iterations"] == 0.25
    assert list(st["residual_history"]) == [1.0, 0.0]
    assert np.array_equal(x, b)


@pytest.mark.skipif(not os.path.exists(os.path.join(os.path.dirname(GOLDEN), "..", "oracle", "_ref", "libsapref.so")),
                    reason="compiled reference not present")
def test_oracle_matches_compiled_reference_random(oracle):
    rng = np.random.default_rng(7)
    for _ in range(6):
        k = int(rng.integers(0, 12))
        p = int(rng.integers(1, 6))
        n = max(p * max(2 * k, 1), 1) + int(rng.integers(0, 200))
        d = float(rng.choice([0.08, 0.3, 1.0, 1.5]))
        seed = int(rng.integers(0, 2**31))
        band, rhs = oracle.random_banded(n, k, d, seed)
        rb, rr = oracle.ref_random_banded(n, k, d, seed)
        assert np.array_equal(band, rb) and np.array_equal(rhs, rr)
        f, g = oracle.factor_blocks(n, k, band, p, True), oracle.ref_factor_blocks(n, k, band, p, True)
        assert all(np.array_equal(f[q], g[q]) for q in ("lu", "ul", "boosts", "boosts_ul", "norms"))
        for kind in (0, 1):
            try:
                mine = oracle.apply(n, k, band, p, kind, rhs)
            except oracle.OracleError as e:
                with pytest.raises(oracle.OracleError):
                    oracle.ref_apply(n, k, band, p, kind, rhs)
                assert e.code == 2
                continue
            assert np.array_equal(mine, oracle.ref_apply(n, k, band, p, kind, rhs))
            x, st = oracle.solve_banded(n, k, band, rhs, p, kind, max_iterations=40)
            y, su = oracle.ref_solve_banded(n, k, band, rhs, p, kind, max_iterations=40)
            assert st["iterations"] == su["iterations"] and np.array_equal(x, y)
