"""Repeat setups in the lu_df_check pattern (3 setups per handle, then a solve) to catch intermittent
k_band_lu_df dependency timeouts; the setup raises CudaError with the timed-out wait's details."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, paper_1509_07919_b200 as S

cases = [(20000, 100, 0.5, 5, False), (3000, 64, 1.0, 3, True), (20011, 77, 1.0, 7, True), (3000, 64, 1.0, 3, False)]
fails = 0
for rep in range(int(os.environ.get("REPS", "8"))):
    for (n, k, d, p, dev) in cases:
        band, rhs = S.random_banded(n, k, d, 1)
        src = torch.from_numpy(band).cuda() if dev else band
        with S.Solver(p=p, device=0) as s:
            try:
                for _ in range(3):
                    s.setup(src, n, k)
                x, st = s.solve(rhs)
                if not st.converged or st.iterations > 2:
                    fails += 1
                    print(rep, n, k, p, dev, "BAD SOLVE", st.iterations, st.final_relative_residual, flush=True)
            except Exception as e:
                fails += 1
                print(rep, n, k, p, dev, "ERR", e, flush=True)
print("fails", fails)
