"""drop_off on the device (proj/include/sap/pipeline.hpp:59-99) against the compiled reference:
the kept half-bandwidth k_after is an integer decision over floating-point sums formed in the
reference's order, so it must equal the reference's exactly; the solve through the dropped-band
preconditioner follows solve_sparse (pipeline.hpp:265-344) with iterations within +-1."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ref(oracle):
    if not oracle.has_ref():
        pytest.skip("compiled reference absent")
    return oracle


def _random_csr(n, spread, per_row, seed, unsorted=False):
    rng = np.random.default_rng(seed)
    rp, ci, v = [0], [], []
    for i in range(n):
        js = {i} | {int(x) for x in np.clip(i + rng.integers(-spread, spread + 1, per_row), 0, n - 1)}
        js = sorted(js)
        if unsorted:
            rng.shuffle(js)
        for j in js:
            ci.append(j)
            v.append(float(per_row + 2) if j == i else rng.uniform(-1, 1))
        rp.append(len(ci))
    return np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)


@pytest.mark.parametrize("seed,unsorted", [(1, False), (2, True), (3, False)])
def test_drop_off_k_matches_reference(sap, ref, seed, unsorted):
    n = 4000
    rp, ci, v = _random_csr(n, 300, 6, seed, unsorted)
    s = sap.Solver(p=4, precond=sap.PrecondKind.decoupled)
    for tol in (0.0, 1e-4, 0.01, 0.03, 0.05, 0.08, 0.1, 0.15, 0.2, 0.3, 1.0):
        want, _ = ref.ref_drop_off(n, rp, ci, v, tol)
        got = s.setup_from_csr_drop(rp, ci, v, tol)
        assert got == want, (tol, got, want)
    with pytest.raises(ValueError, match="tolerance must lie in"):
        s.setup_from_csr_drop(rp, ci, v, 1.5)
    s.close()


def test_drop_off_threshold_ties(sap, ref):
    """Masses that make suf[c + 1] land exactly on the threshold: equal-magnitude entries, tol chosen
    from the reference's own sums."""
    n = 600
    rp, ci, v = [0], [], []
    for i in range(n):
        for j in (i - 7, i - 3, i, i + 3, i + 7):
            if 0 <= j < n:
                ci.append(j)
                v.append(4.0 if j == i else 0.5)
        rp.append(len(ci))
    rp, ci, v = np.array(rp, np.int32), np.array(ci, np.int32), np.array(v)
    s = sap.Solver(p=2, precond=sap.PrecondKind.decoupled)
    for tol in np.linspace(0.0, 0.5, 26):
        want, _ = ref.ref_drop_off(n, rp, ci, v, float(tol))
        assert s.setup_from_csr_drop(rp, ci, v, float(tol)) == want, tol
    s.close()


@pytest.mark.parametrize("kind,tol", [(0, 0.05), (1, 0.05), (0, 0.2)])
def test_drop_off_solve_matches_solve_sparse(sap, ref, kind, tol):
    """solve_sparse with drop_tol (no DB / CM): band assembled from the dropped matrix, Krylov on the
    full CSR operator."""
    n = 6000
    rp, ci, v = _random_csr(n, 60, 5, 11)
    xs = np.linspace(-1.0, 2.0, n)
    rhs = ref.csr_matvec(n, rp, ci, v, xs)
    xr, so = ref.ref_solve_sparse(n, rp, ci, v, rhs, 4, kind, drop_tol=tol)
    assert so["converged"]
    s = sap.Solver(p=4, precond=kind)
    assert s.setup_from_csr_drop(rp, ci, v, tol) == so["k_after"]
    s.set_operator_csr(rp, ci, v)
    x, st = s.solve(rhs)
    assert st.converged and st.final_relative_residual <= 1e-10
    assert abs(st.iterations - so["iterations"]) <= 1.0, (st.iterations, so["iterations"])
    assert np.linalg.norm(x - xr) <= 1e-8 * np.linalg.norm(xr)
    s.close()
