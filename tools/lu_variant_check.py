"""Compare the default LU kernel's factors with SAP_LU_SEQ=1 (k_band_lu_seq) bit for bit.

Run twice by the driver below: each process dumps factors for a few shapes; then compared.
    python tools/lu_variant_check.py            # runs both variants in subprocesses and compares
"""
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
SHAPES = [(4000, 20, 4, 1.0), (20000, 200, 5, 1.0), (12345, 64, 7, 0.3), (3001, 33, 3, 0.8), (9000, 150, 6, 0.1),
          (641, 10, 2, 1.0), (2000, 1, 3, 1.0)]


def dump(out):
    import paper_1509_07919_b200 as S
    res = {}
    for i, (n, k, p, d) in enumerate(SHAPES):
        band, rhs = S.random_banded(n, k, d, 3 + i)
        s = S.Solver(p=p, precond=S.PrecondKind.coupled)
        s.setup(band, n, k)
        lu, b, _ = s.factors(0)
        ul, bu, _ = s.factors(1)
        res[f"lu{i}"], res[f"ul{i}"], res[f"b{i}"], res[f"bu{i}"] = lu, ul, b, bu
        res[f"m{i}"] = s.apply_preconditioner(rhs)
        s.close()
    np.savez(out, **res)


if __name__ == "__main__":
    if len(sys.argv) > 1:
        dump(sys.argv[1])
        sys.exit(0)
    env = dict(os.environ)
    subprocess.run([sys.executable, __file__, "/tmp/lu_new.npz"], check=True, env=env)
    env["SAP_LU_SEQ"] = "1"
    subprocess.run([sys.executable, __file__, "/tmp/lu_seq.npz"], check=True, env=env)
    a, b = np.load("/tmp/lu_new.npz"), np.load("/tmp/lu_seq.npz")
    ok = True
    for key in a.files:
        same = np.array_equal(a[key], b[key])
        diff = 0.0 if same else float(np.max(np.abs(a[key] - b[key])) / max(np.max(np.abs(b[key])), 1e-300))
        print(f"{key}: {'bitwise' if same else f'DIFF rel {diff:.3e}'}")
        ok &= same
    print("ALL BITWISE" if ok else "DIFFERENCES")
