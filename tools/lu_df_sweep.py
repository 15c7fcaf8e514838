"""Factor-kernel time of the single-CTA LU (lu_kernel=1) vs the dataflow LU (lu_kernel=2) over shapes (device band)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, paper_1509_07919_b200 as S

CASES = [(200000, 300, 50, "C"), (200000, 300, 50, "D"), (200000, 500, 50, "C"), (200000, 500, 50, "D"),(2000000, 128, 512, "C"), (2000000, 128, 512, "D"), (2000000, 128, 64, "C"), (200000, 64, 50, "C"),
         (200000, 100, 50, "C"), (200000, 160, 50, "C"), (200000, 200, 50, "C"), (200000, 200, 50, "D"),
         (200000, 224, 50, "C"), (200000, 200, 25, "C")]
for n, k, p, kind in CASES:
    band, rhs = S.random_banded(n, k, 1.0, 1)
    db = torch.from_numpy(band).cuda()
    del band
    res = []
    for lk in (1, 2):
        with S.Solver(p=p, precond=S.PrecondKind.coupled if kind == "C" else S.PrecondKind.decoupled, device=0,
                      lu_kernel=lk) as s:
            ts = []
            for _ in range(4):
                s.setup(db, n, k)
                ts.append(s.report()["t_factor_kernel"])
            res.append(min(ts[1:]) * 1e3)
    print(f"n={n} k={k} p={p} {kind}: single-CTA {res[0]:.3f} ms, dataflow {res[1]:.3f} ms", flush=True)
    del db
    torch.cuda.empty_cache()
