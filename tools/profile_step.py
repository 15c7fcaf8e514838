"""One config-2 time-to-solution (setup + solve) for ncu captures.

    ncu --set full -k regex:k_band_lu -s 0 -c 1 -o gpurun_out/lu python tools/profile_step.py --precond C
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_07919_b200 as S  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--precond", choices=["C", "D"], default="C")
ap.add_argument("--n", type=int, default=200000)
ap.add_argument("--k", type=int, default=200)
ap.add_argument("--p", type=int, default=50)
ap.add_argument("--reps", type=int, default=1)
a = ap.parse_args()
band, rhs = S.random_banded(a.n, a.k, 1.0, 1)
s = S.Solver(p=a.p, precond=S.PrecondKind.coupled if a.precond == "C" else S.PrecondKind.decoupled)
for _ in range(a.reps):
    s.setup(band, a.n, a.k)
    x, st = s.solve(rhs)
print(st.iterations, st.final_relative_residual, s.report())
