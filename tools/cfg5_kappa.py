import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_1509_07919_b200 as S
n, k, p = 2000000, 128, 512
band_h, rhs_h = S.random_banded(n, k, 1.0, 1)
band = torch.from_numpy(band_h).cuda(); rhs = torch.from_numpy(rhs_h).cuda()
for tri in ["", "inverse"]:
    s = S.Solver(p=p, precond=S.PrecondKind.coupled, triangle_solve=1 if tri else 0)
    s.setup(band, n, k); x, st = s.solve(rhs); s.setup(band, n, k); x, st = s.solve(rhs)
    print(tri or "auto", "t_kry", s.report()["t_kry"], st.iterations)
    s.close()
