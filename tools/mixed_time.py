"""Config 2 time-to-solution with the FP32 preconditioner (KrylovOptions.mixed_precision) vs FP64."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1509_07919_b200 as S  # noqa: E402

n, k, p = 200000, 200, 50
band_h, rhs_h = S.random_banded(n, k, 1.0, 1)
band = torch.from_numpy(band_h).cuda()
rhs = torch.from_numpy(rhs_h).cuda()
for kind in (S.PrecondKind.coupled, S.PrecondKind.decoupled):
    for mixed in (False, True):
        s = S.Solver(p=p, precond=kind, krylov=S.KrylovOptions(mixed_precision=mixed))
        stream = torch.cuda.Stream()
        s.set_stream(stream)
        best = None
        with torch.cuda.stream(stream):
            for i in range(4):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                s.setup(band, n, k)
                x, st = s.solve(rhs)
                e1.record(stream)
                torch.cuda.synchronize()
                t = e0.elapsed_time(e1)
                if i and (best is None or t < best[0]):
                    best = (t, s.report(), st)
        t, r, st = best
        print(f"{'SaP-C' if kind == 0 else 'SaP-D'} mixed={mixed}: {t:.3f} ms (setup t_lu {r['t_lu'] * 1e3:.3f}, "
              f"t_kry {r['t_kry'] * 1e3:.3f}), iterations {st.iterations}, residual {st.final_relative_residual:.2e}")
        s.close()
