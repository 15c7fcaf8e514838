import sys; sys.path.insert(0, "/root/repo")
import torch, paper_1509_07919_b200 as S
n, k, p = 200000, 200, 50
band, rhs = S.random_banded(n, k, 1.0, 1)
db = torch.from_numpy(band).cuda(); x = torch.from_numpy(rhs).cuda(); y = torch.empty_like(x)
for kind, ts, name in ((1, 0, "SaP-D"), (0, 1, "SaP-C full LU first solve"), (0, 0, "SaP-C tip sweeps")):
    with S.Solver(p=p, precond=kind, tip_solve=ts) as s:
        s.setup(db, n, k)
        for _ in range(3): s.apply_preconditioner(x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(20): s.apply_preconditioner(x, y)
        e1.record(); torch.cuda.synchronize()
        print(f"  {name}: {e0.elapsed_time(e1) * 1e3 / 20:.1f} us per apply (ul_tip_sweeps={s.report()['ul_tip_sweeps']})", flush=True)
