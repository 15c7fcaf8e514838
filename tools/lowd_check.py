"""Low diagonal dominance check: GPU vs the compiled reference (oracle/_ref) on the same input --
iterations, boosts, factor / tip / M*r differences. Usage: python tools/lowd_check.py N K D P [C|D]"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle as O  # noqa: E402
import paper_1509_07919_b200 as S  # noqa: E402

n, k, d, p = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), int(sys.argv[4])
pre = sys.argv[5] if len(sys.argv) > 5 else "C"
kind = 0 if pre == "C" else 1
band, rhs = O.ref_random_banded(n, k, d, 1)
t0 = time.time()
xr, sr = O.ref_solve_banded(n, k, band, rhs, p, kind)
print(f"reference: iterations {sr['iterations']} residual {sr['final_relative_residual']:.3e} ({time.time() - t0:.1f}s)")
s = S.Solver(p=p, precond=S.PrecondKind.coupled if pre == "C" else S.PrecondKind.decoupled)
s.setup(band, n, k)
x, st = s.solve(rhs)
print(f"gpu      : iterations {st.iterations} residual {st.final_relative_residual:.3e} converged {st.converged}")
print("gpu residual history", [f"{v:.2e}" for v in st.residual_history[:12]])
print("ref residual history", [f"{v:.2e}" for v in sr["residual_history"][:12]])
fr = O.ref_factor_blocks(n, k, band, p, pre == "C")
for which, key in ((0, "lu"), (1, "ul")):
    if fr[key] is None:
        continue
    got, bo, _ = s.factors(which)
    ref = fr[key]
    e = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
    rb = fr["boosts"] if which == 0 else fr["boosts_ul"]
    print(f"{key}: normwise rel diff {e:.3e}; max|F| {np.max(np.abs(ref)):.3e}; boosts gpu {int(bo.sum())} ref {int(rb.sum())}")
sp = O.ref_spikes(n, k, band, p)
for t in (0, p // 2, p - 2):
    g = s.spike(t)
    w2 = k * k
    for q in ("vb", "wt", "rbar"):
        rr = sp[q][t * w2:(t + 1) * w2]
        print(f"  iface {t} {q}: normwise rel diff {np.max(np.abs(g[q] - rr)) / np.max(np.abs(rr)):.3e}")
r = np.random.default_rng(0).uniform(-1, 1, n)
mg = s.apply_preconditioner(r)
mr = O.ref_apply(n, k, band, p, kind, r)
print(f"M*r rel diff {np.linalg.norm(mg - mr) / np.linalg.norm(mr):.3e}")
# accuracy of the GPU solution itself, residual recomputed on the host (compensated)
ax = O.band_matvec(n, k, band, x)
print(f"host-recomputed residual of gpu x: {np.linalg.norm(rhs - ax) / np.linalg.norm(rhs):.3e};"
      f" of ref x: {np.linalg.norm(rhs - O.band_matvec(n, k, band, xr)) / np.linalg.norm(rhs):.3e};"
      f" |x_gpu - x_ref|/|x_ref| = {np.linalg.norm(x - xr) / np.linalg.norm(xr):.3e}, |x| = {np.linalg.norm(xr):.3e}")
