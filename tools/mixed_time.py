"""Mixed precision (FP32 factorization, build_precond_op<float>) vs FP64 at configs 2 and 3: setup / solve
device times, iterations, and the reference's FP32 path for comparison (iterations).
    python tools/mixed_time.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_07919_b200 as S

CASES = [(200000, 200, 1.0, 50, "C"), (200000, 200, 1.0, 50, "D"), (200000, 50, 1.0, 50, "C"),
         (200000, 100, 0.5, 50, "C"), (200000, 10, 1.0, 50, "D")]
for n, k, d, p, kind in CASES:
    band, rhs = S.random_banded(n, k, d, 1)
    db = torch.from_numpy(band).cuda()
    pk = S.PrecondKind.coupled if kind == "C" else S.PrecondKind.decoupled
    row = []
    for mixed in (False, True):
        with S.Solver(p=p, precond=pk, krylov=S.KrylovOptions(mixed_precision=mixed)) as s:
            for _ in range(2):
                s.setup(db, n, k)
                x, st = s.solve(rhs)
            r = s.report()
            t_setup = r["t_lu"] + r["t_bc"] + r["t_spk"] + r["t_lurdcd"]
            row.append(f"{'FP32' if mixed else 'FP64'}: setup {t_setup*1e3:.2f} ms (LU kernel "
                       f"{r['t_factor_kernel']*1e3:.2f}), solve {r['t_kry']*1e3:.2f} ms, {st.iterations} it, "
                       f"res {st.final_relative_residual:.1e}")
    print(f"n={n} k={k} d={d} p={p} {kind}: " + " | ".join(row), flush=True)
