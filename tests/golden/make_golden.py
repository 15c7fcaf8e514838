"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/*.npz. Every array is the reference's own output
(factor_blocks, extract_coupling, compute_spike_tips, apply_preconditioner,
build_precond_op + run_krylov) on testsup::random_banded inputs.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

# (name, n, k, d, seed, p)
CASES = [
    ("small_d1", 200, 5, 1.0, 1, 4),
    ("small_d01", 300, 7, 0.1, 2, 3),
    ("k1", 64, 1, 0.5, 3, 4),
    ("k0", 50, 0, 1.3, 4, 5),
    ("ragged", 403, 9, 0.7, 5, 5),
]


def case(name, n, k, d, seed, p):
    band, rhs = O.ref_random_banded(n, k, d, seed)
    out = dict(n=n, k=k, d=d, seed=seed, p=p, band=band, rhs=rhs)
    f = O.ref_factor_blocks(n, k, band, p, True)
    out.update(lu=f["lu"], ul=f["ul"], boosts=f["boosts"], boosts_ul=f["boosts_ul"], norms=f["norms"])
    if p > 1:
        s = O.ref_spikes(n, k, band, p)
        out.update(B=s["B"], C=s["C"], vb=s["vb"], wt=s["wt"], rbar=s["rbar"], rbar_boosts=s["rbar_boosts"])
    for kind, tag in ((0, "c"), (1, "d")):
        out["m_" + tag] = O.ref_apply(n, k, band, p, kind, rhs)
        x, st = O.ref_solve_banded(n, k, band, rhs, p, kind, max_iterations=100)
        out["x_" + tag] = x
        out["it_" + tag] = st["iterations"]
        out["hist_" + tag] = st["residual_history"]
        out["fail_" + tag] = st["failure"]
    np.savez_compressed(os.path.join(OUT, name + ".npz"), **out)


def criterion2():
    # proj/tests/acceptance.cpp:103-154: N=10000, K=50, P=8, SaP-C + BiCGStab(2),
    # seeds 1000*(di+1)+s, rel_tol 1e-10, max 50 iterations.
    rows = []
    for di, d in enumerate([0.1, 0.5, 1.0, 1.2]):
        for s in range(5):
            seed = 1000 * (di + 1) + s
            band, rhs = O.ref_random_banded(10000, 50, d, seed)
            _, st = O.ref_solve_banded(10000, 50, band, rhs, 8, 0, max_iterations=50)
            rows.append((d, seed, st["iterations"], st["final_relative_residual"], st["failure"]))
    # config 1 (BASELINE.json configs[0]): N=10000 K=10 d=1 P=4 SaP-D, seed 1
    band, rhs = O.ref_random_banded(10000, 10, 1.0, 1)
    _, st = O.ref_solve_banded(10000, 10, band, rhs, 4, 1)
    cfg1 = np.array([st["iterations"], st["final_relative_residual"]])
    np.savez_compressed(os.path.join(OUT, "criterion2.npz"), rows=np.array(rows), config1=cfg1)


if __name__ == "__main__":
    for c in CASES:
        case(*c)
        print("wrote", c[0])
    criterion2()
    print("wrote criterion2")
