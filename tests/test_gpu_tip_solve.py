"""SaP-C apply, first block solve from tip sweeps (sap_options::tip_solve).

apply_preconditioner (spike.hpp:323-347) reads g = D^{-1} r only at each block's first and last w rows. With
tip_solve = 0 those rows come from the LU sweeps with the backward sweep stopped after the last w rows and from
UL sweeps (bottom-up unit-upper, then top-down lower, stopped after the first w rows), side by side; tip_solve = 1
runs the reference's full LU block solve. Both are compared with each other and with the oracle's apply; the
automatic choice must fall back to the full LU solve whenever a pivot was boosted (a boosted LU and UL are
different perturbations of A_b) or the chunk triangles call for substitution.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel2(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


def _solver(sap, n, k, band, p, tip_solve, **kw):
    s = sap.Solver(p=p, precond=sap.PrecondKind.coupled, tip_solve=tip_solve, krylov=sap.KrylovOptions(**kw))
    s.setup(band, n, k)
    return s


CASES = [
    # n, k, d, seed, p -- unequal blocks, K not a multiple of 32, partial last chunks, blocks barely above 2K,
    # one interface, config-2's K
    (3000, 200, 1.0, 15, 3),
    (2000, 50, 1.0, 12, 8),
    (997, 33, 0.8, 18, 7),
    (1500, 64, 1.2, 14, 4),
    (6001, 200, 1.0, 21, 12),
    (480, 100, 1.0, 22, 2),
    (2400, 300, 0.7, 19, 2),
    (5000, 45, 0.5, 23, 9),
]


@pytest.mark.parametrize("n,k,d,seed,p", CASES)
def test_tip_sweeps_match_full_block_solve_and_oracle(sap, oracle, n, k, d, seed, p):
    band, rhs = oracle.random_banded(n, k, d, seed)
    with _solver(sap, n, k, band, p, 0) as a, _solver(sap, n, k, band, p, 1) as b:
        ra, rb = a.report(), b.report()
        assert ra["total_boosts"] == 0 and ra["total_boosts_ul"] == 0
        assert ra["ul_tip_sweeps"] == 1 and rb["ul_tip_sweeps"] == 0
        ga, gb = a.apply_preconditioner(rhs), b.apply_preconditioner(rhs)
        assert rel2(ga, gb) <= 1e-13
        assert rel2(ga, oracle.apply(n, k, band, p, 0, rhs)) <= 1e-12
        # in place through device pointers (in == out): the tip sweeps work on their own copies
        import torch
        x = torch.from_numpy(rhs.copy()).cuda()
        a.apply_preconditioner(x, out=x)
        assert np.array_equal(x.cpu().numpy(), ga)


def test_tip_sweeps_solve_iterations_equal(sap, oracle):
    n, k, p = 20000, 120, 10
    band, b = oracle.random_banded(n, k, 1.0, 31)
    with _solver(sap, n, k, band, p, 0) as a, _solver(sap, n, k, band, p, 1) as c:
        xa, sa = a.solve(b)
        xc, sc = c.solve(b)
        assert sa.converged and sc.converged
        assert sa.iterations == sc.iterations
        assert rel2(xa, xc) <= 1e-10
        xr, so = oracle.ref_solve_banded(n, k, band, b, p, 0)  # the compiled reference (oracle/_ref)
        assert abs(sa.iterations - so["iterations"]) <= 1.0
        assert rel2(xa, xr) <= 1e-8


def test_boosted_factorization_keeps_full_lu_solve(sap, oracle):
    """A zero pivot (boosted, test_block_factors.cpp style): the automatic choice is the reference's solve."""
    n, k, p = 400, 4, 4
    band, rhs = oracle.random_banded(n, k, 1.0, 41)
    w = 2 * k + 1
    band = band.copy()
    band[100 * w + k] = 0.0  # A(100, 100) = 0: the first LU pivot of block 1 (rows 100..199) is boosted
    with _solver(sap, n, k, band, p, 0) as a, _solver(sap, n, k, band, p, 1) as b:
        ra = a.report()
        assert ra["total_boosts"] + ra["total_boosts_ul"] > 0
        assert ra["ul_tip_sweeps"] == 0
        assert np.array_equal(a.apply_preconditioner(rhs), b.apply_preconditioner(rhs))


def test_low_dominance_keeps_full_lu_solve(sap, oracle):
    """Config-3-like d = 0.06: substitution sweeps (ill-conditioned chunk triangles) or boosts keep the LU path."""
    n, k, p = 3000, 200, 2
    band, rhs = oracle.random_banded(n, k, 0.06, 16)
    with _solver(sap, n, k, band, p, 0) as a:
        r = a.report()
        if r["sweep_substitution"] or r["total_boosts"] or r["total_boosts_ul"]:
            assert r["ul_tip_sweeps"] == 0
        got = a.apply_preconditioner(rhs)
        assert rel2(got, oracle.apply(n, k, band, p, 0, rhs)) <= 1e-6
