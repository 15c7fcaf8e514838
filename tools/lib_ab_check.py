"""Bitwise A/B of two builds of libsap_gpu.so: factors, tips and M r on a few shapes.

    python tools/lib_ab_check.py LIB_A LIB_B
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHAPES = [(4000, 20, 4, 1.0), (20000, 200, 5, 1.0), (12345, 64, 7, 0.3), (3001, 33, 3, 0.8), (9000, 150, 6, 0.1),
          (200000, 200, 50, 1.0)]

if __name__ == "__main__":
    if sys.argv[1] == "--dump":
        sys.path.insert(0, ROOT)
        import paper_1509_07919_b200 as S
        res = {}
        for i, (n, k, p, d) in enumerate(SHAPES):
            band, rhs = S.random_banded(n, k, d, 3 + i)
            s = S.Solver(p=p, precond=S.PrecondKind.coupled)
            s.setup(band, n, k)
            res[f"lu{i}"], res[f"b{i}"], _ = s.factors(0)
            res[f"ul{i}"], res[f"bu{i}"], _ = s.factors(1)
            res[f"m{i}"] = s.apply_preconditioner(rhs)
            res[f"t{i}"] = s.report()["t_factor_kernel"]
            s.close()
        np.savez(sys.argv[2], **res)
        sys.exit(0)
    outs = []
    for j, lib in enumerate(sys.argv[1:3]):
        env = dict(os.environ, SAP_GPU_LIB=os.path.abspath(lib))
        subprocess.run([sys.executable, __file__, "--dump", f"/tmp/ab{j}.npz"], check=True, env=env)
        outs.append(np.load(f"/tmp/ab{j}.npz"))
    a, b = outs
    ok = True
    for key in a.files:
        if key.startswith("t"):
            print(f"{key}: factor kernel {float(a[key]) * 1e3:.3f} ms vs {float(b[key]) * 1e3:.3f} ms")
            continue
        same = np.array_equal(a[key], b[key])
        ok &= same
        if not same:
            print(f"{key}: DIFF rel {np.max(np.abs(a[key] - b[key])) / max(np.max(np.abs(b[key])), 1e-300):.3e}")
    print("ALL BITWISE" if ok else "DIFFERENCES")
