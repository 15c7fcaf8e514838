"""solve_sparse on the device (pipeline.hpp:213-369) after the reference's host stage.

The reference's sparse pipeline is: DB reordering (+ row/column scaling) and CM reordering on the host
(graph algorithms; north_star keeps them the reference's host stage), then drop-off, band assembly,
partitioning, the SaP preconditioner, and BiCGStab(l) over the reordered, untruncated CSR operator, and
finally the inverse permutation / column scaling of the solution.

``solve_reordered`` is everything after the host stage, on the device through the C ABI:

* ``sap_setup_from_csr_drop`` -- drop_off (pipeline.hpp:59-99), assemble_banded (:103-115) and the setup
  (build_precond_op, :140-202) with the device-side timers T_Drop / T_Asmbl / T_LU / ...;
* ``sap_set_operator_csr`` -- the Krylov operator is the reordered CSR matrix itself (:336-338);
* ``sap_solve`` -- BiCGStab(l) (:340-344); then x[i] = z[cm_perm[i]] * col_scale[i] (:360-368).

The host stage's output (reordered CSR, right-hand side, permutation, scaling) comes from the caller; the
tests and tools/config4.py take it from the compiled reference (oracle.ref_host_stage).
"""
from __future__ import annotations

import time

import numpy as np

from .solver import KrylovOptions, PrecondKind, Solver


def solve_reordered(rp, ci, v, rhs, cm_perm, col_scale, p: int, drop_tol: float,
                    precond: PrecondKind = PrecondKind.coupled, krylov: KrylovOptions | None = None,
                    device: int = 0, repeat: int = 1):
    """Returns (x in the caller's ordering, SolveStats, report dict with k_after and the stage times).
    `repeat` > 1 re-runs setup + solve and reports the last run (warm timings)."""
    n = len(rp) - 1
    s = Solver(p=p, precond=precond, krylov=krylov, device=device)
    try:
        for _ in range(max(1, repeat)):
            t0 = time.perf_counter()
            k_after = s.setup_from_csr_drop(rp, ci, v, drop_tol)
            s.set_operator_csr(rp, ci, v)
            z, st = s.solve(rhs)
            wall = time.perf_counter() - t0
        rep = s.report()
        rep["k_after"] = k_after
        rep["wall_setup_solve"] = wall
        x = np.asarray(z)[np.asarray(cm_perm)] * np.asarray(col_scale)
        return x, st, rep
    finally:
        s.close()
