"""Iterations of the GPU solve on a committed golden fixture vs the reference's (tests/golden/NAME.npz)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1509_07919_b200 as S  # noqa: E402

g = np.load(os.path.join(ROOT, "tests", "golden", sys.argv[1] + ".npz"))
n, k, p = int(g["n"]), int(g["k"]), int(g["p"])
for kind, tag in ((0, "c"), (1, "d")):
    s = S.Solver(p=p, precond=kind, krylov=S.KrylovOptions(max_iterations=100))
    s.setup(g["band"], n, k)
    x, st = s.solve(g["rhs"])
    print(tag, "gpu", st.iterations, "ref", float(g["it_" + tag]), "res", st.final_relative_residual,
          "x diff", np.linalg.norm(x - g["x_" + tag]) / np.linalg.norm(g["x_" + tag]))
    s.close()
