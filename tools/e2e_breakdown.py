"""Where the end-to-end time goes (config 2, host band in pinned memory through sap_setup_banded +
sap_solve): the report's stage timers and the host wall time of each call.
    python tools/e2e_breakdown.py [C|D]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1509_07919_b200 as S

kind = sys.argv[1] if len(sys.argv) > 1 else "C"
n, k, p = 200000, 200, 50
band, rhs = S.random_banded(n, k, 1.0, 1)
bp = torch.from_numpy(band).pin_memory()
rp = torch.from_numpy(rhs).pin_memory()
xp = torch.empty(n, dtype=torch.float64).pin_memory()
pk = S.PrecondKind.coupled if kind == "C" else S.PrecondKind.decoupled
with S.Solver(p=p, precond=pk) as s:
    for it in range(4):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        s.setup(bp, n, k) if False else S._lib.load().sap_setup_banded(s._h, n, k, __import__("ctypes").c_void_p(bp.data_ptr()), 0)
        t1 = time.perf_counter()
        x, st = s.solve(rp.numpy())
        t2 = time.perf_counter()
        r = s.report()
        if it:
            keys = ("t_dtransf", "t_lu", "t_factor_kernel", "t_bc", "t_spk", "t_lurdcd", "t_kry")
            print(f"setup wall {1e3*(t1-t0):.2f} ms, solve wall {1e3*(t2-t1):.2f} ms | " +
                  " ".join(f"{q} {1e3*r[q]:.2f}" for q in keys) + f" | it {st.iterations}", flush=True)
