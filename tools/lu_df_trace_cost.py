import sys, os; sys.path.insert(0, "/root/repo")
import torch, paper_1509_07919_b200 as S
from paper_1509_07919_b200 import _lib
n, k, p = 200000, 200, 50
band, rhs = S.random_banded(n, k, 1.0, 1)
db = torch.from_numpy(band).cuda()
for mode in (0, 1, 0, 1):
    _lib.load().sap_dev_lu_df_trace_mode(mode)
    with S.Solver(p=p, precond=S.PrecondKind.decoupled, lu_kernel=2) as s:
        ts = []
        for _ in range(4):
            s.setup(db, n, k)
            ts.append(s.report()["t_factor_kernel"] * 1e3)
    print("trace mode", mode, "t_factor ms", [round(t, 3) for t in ts], flush=True)
