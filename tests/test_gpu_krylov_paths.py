"""GPU parity for the Krylov paths and preconditioner kinds not covered by test_gpu_parity.py:

* BiCGStab(l) at ell = 1, 3, 8 against the oracle (krylov.hpp:110-350; the polynomial update packs
  3 (ell - 1) + 3 coefficients, so ell = 8 exercises every slot);
* the breakdown / single-restart path (krylov.hpp:155-167, :335-345) with the zero operator of
  proj/tests/test_krylov.cpp:201-217;
* the diagonal preconditioner (pipeline.hpp:151-161) in FP64 and at T = float (mixed_precision),
  M r bit-exact against a numpy restatement and the solve against the compiled reference.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def rel2(a, b):
    den = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (den if den > 0 else 1.0)


@pytest.mark.parametrize("ell", [1, 3, 8])
@pytest.mark.parametrize("d,kind", [(0.3, 1), (0.2, 1), (0.2, 0)])
def test_bicgstab_ell_matches_oracle(sap, oracle, ell, d, kind):
    """Oracle iterations (ell = 1 / 3 / 8): d=0.3 SaP-D 10 / 3.5 / 1.5; d=0.2 SaP-D 24.5 / 7.75 / 3;
    d=0.2 SaP-C 1 / 0.75 / 0.75 -- several sweeps through the MGS and polynomial updates."""
    n, k, p = 6000, 24, 12
    band, rhs = oracle.random_banded(n, k, d, 101)
    _, so = oracle.solve_banded(n, k, band, rhs, p, kind, ell=ell, max_iterations=200)
    s = sap.Solver(p=p, precond=kind, krylov=sap.KrylovOptions(ell=ell, max_iterations=200))
    s.setup(band, n, k)
    x, st = s.solve(rhs)
    assert so["converged"] and st.converged
    assert st.final_relative_residual <= 1e-10
    assert abs(st.iterations - so["iterations"]) <= 1.0, (ell, st.iterations, so["iterations"])
    # one true residual per BiCGStab step, iterations in quarters of the 2 ell steps of a sweep
    # (krylov.hpp:134-141): quarters = ceil(4 steps / (2 ell))
    steps = len(st.residual_history) - 1
    assert st.iterations == -(-4 * steps // (2 * ell)) / 4.0
    r = rhs - oracle.band_matvec(n, k, band, x)
    assert np.linalg.norm(r) <= 1e-10 * np.linalg.norm(rhs) * (1 + 1e-6)
    s.close()


def test_ell_above_maximum_is_invalid_argument(sap):
    s = sap.Solver(p=1, precond=sap.PrecondKind.none, krylov=sap.KrylovOptions(ell=9))
    s.setup(np.ones(4), 4, 0)
    with pytest.raises(ValueError, match="ell"):
        s.solve(np.ones(4))
    s.close()


@pytest.mark.parametrize("csr", [False, True])
def test_zero_operator_exhausts_the_single_restart(sap, oracle, csr):
    """test_krylov.cpp:201-217: the zero operator breaks down, the restart breaks down again, the solve
    reports breakdown; a second solve gives the same residual history."""
    b = np.array([1.0, -2.0])
    s = sap.Solver(p=1, precond=sap.PrecondKind.none)
    s.setup(np.zeros(2), 2, 0)
    if csr:
        s.set_operator_csr(np.zeros(3, np.int32), np.zeros(0, np.int32), np.zeros(0))
    _, st = s.solve(b)
    assert not st.converged and st.failure == sap.KrylovFailure.breakdown
    _, again = s.solve(b)
    assert again.failure == sap.KrylovFailure.breakdown
    assert again.residual_history == st.residual_history
    _, so = oracle.solve_banded(2, 0, np.zeros(2), b, 1, 3)
    assert so["failure"] == int(sap.KrylovFailure.breakdown)
    assert np.array_equal(np.asarray(st.residual_history), so["residual_history"])
    s.close()


def _diag_ref(n, k, band, x, mixed, eps=1e-10):
    """build_precond_op<T>'s diagonal branch (pipeline.hpp:151-161) + apply (spike.hpp:304-351) in numpy."""
    a = band.reshape(n, 2 * k + 1)
    if mixed:
        af = a.astype(np.float32).astype(np.float64)
    else:
        af = a
    # inf_norm: row sums of |entries| (in double), ascending column order (banded_matrix.hpp:84-96)
    rows = np.zeros(n)
    for i in range(n):
        acc = 0.0
        for j in range(max(0, i - k), min(n - 1, i + k) + 1):
            acc += abs(af[j, i - j + k])
        rows[i] = acc
    scale = rows.max() if n else 0.0
    T = np.float32 if mixed else np.float64
    bv = T(eps * (scale if scale > 0 else 1.0))
    d = a[:, k].astype(T)
    d = np.where(np.abs(d) < bv, np.where(d < 0, -bv, bv), d).astype(T)
    return (x.astype(T) / d).astype(np.float64)


@pytest.mark.parametrize("mixed", [False, True])
def test_diagonal_preconditioner(sap, oracle, mixed):
    n, k = 3000, 6
    band, rhs = oracle.random_banded(n, k, 1.2, 77)
    band.reshape(n, 2 * k + 1)[123, k] = 0.0  # a zero diagonal entry: boosted to +bv
    kr = sap.KrylovOptions(mixed_precision=mixed, max_iterations=300)
    s = sap.Solver(p=1, precond=sap.PrecondKind.diagonal, krylov=kr)
    s.setup(band, n, k)
    mr = s.apply_preconditioner(rhs)
    want = _diag_ref(n, k, band, rhs, mixed)
    assert np.array_equal(mr, want)
    x, st = s.solve(rhs)
    xr, so = oracle.ref_solve_banded(n, k, band, rhs, 1, 2, max_iterations=300, mixed_precision=mixed)
    assert st.converged == so["converged"]
    if so["converged"]:
        assert st.final_relative_residual <= 1e-10
        assert abs(st.iterations - so["iterations"]) <= 1.0, (st.iterations, so["iterations"])
        assert rel2(x, xr) <= 1e-8
    s.close()


def test_bicgstab2_host_synchronisations_per_sweep(sap, oracle):
    """Device-side Krylov bookkeeping: a BiCGStab(2) sweep synchronises with the host about 7 times (the two
    rho / g scalars of each BiCG step, its true residual with the next step's dot products batched into it,
    the MGS trial's residual, one read-back of the device-side MGS, the final residual with the next sweep's
    rho) instead of once per dot product (15); iterations unchanged against the oracle."""
    n, k, p = 6000, 24, 12
    band, rhs = oracle.random_banded(n, k, 0.2, 101)
    _, so = oracle.solve_banded(n, k, band, rhs, p, 1, ell=2, max_iterations=200)
    s = sap.Solver(p=p, precond=1, krylov=sap.KrylovOptions(ell=2, max_iterations=200))
    s.setup(band, n, k)
    x, st = s.solve(rhs)
    assert st.converged and abs(st.iterations - so["iterations"]) <= 1.0
    sweeps = int(np.ceil(st.iterations))
    assert sweeps >= 3
    syncs = s.report()["krylov_host_syncs"]
    assert syncs <= 7 * sweeps + 3, (syncs, sweeps)
    s.close()
