"""Dump the band factors (LU, UL, boosts, reduced blocks) of both LU kernels over a fixed case list, so two
builds can be compared bitwise (a kernel rewrite that must not change a single bit).

    python tools/factor_ab.py dump TAG          # on a GPU box: gpurun_out/fab_TAG.npz
    python tools/factor_ab.py cmp TAG_A TAG_B   # anywhere
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")

# n, k, d, p, coupled; d < 1 exercises pivot boosting, n % p and n / p % 32 != 0 the short last panel
CASES = [
    (3000, 64, 1.0, 3, True),
    (20011, 77, 1.0, 7, True),
    (9000, 130, 0.2, 4, True),
    (40000, 200, 0.06, 10, True),
    (40000, 200, 1.0, 10, False),
    (40000, 224, 1.0, 8, False),
    (40000, 300, 0.5, 8, True),
    (50000, 401, 0.5, 9, False),
    (30000, 500, 1.0, 5, True),
]


def dump(tag):
    import torch
    sys.path.insert(0, ROOT)
    import paper_1509_07919_b200 as S
    out = {}
    for ci, (n, k, d, p, coupled) in enumerate(CASES):
        band, _ = S.random_banded(n, k, d, 1)
        kind = S.PrecondKind.coupled if coupled else S.PrecondKind.decoupled
        for lk in (1, 2):
            with S.Solver(p=p, precond=kind, device=0, lu_kernel=lk) as s:
                s.setup(torch.from_numpy(band).cuda(), n, k)
                s.synchronize()
                lu, b, _ = s.factors(0)
                out[f"{ci}_{lk}_lu"], out[f"{ci}_{lk}_lub"] = lu, b
                if coupled:
                    ul, b2, _ = s.factors(1)
                    out[f"{ci}_{lk}_ul"], out[f"{ci}_{lk}_ulb"] = ul, b2
                    for t in range(p - 1):
                        out[f"{ci}_{lk}_rbar{t}"] = s.spike(t)["rbar"]
            print(f"case {ci} lu_kernel {lk} boosts {int(np.sum(out[f'{ci}_{lk}_lub']))}", flush=True)
    os.makedirs(OUT, exist_ok=True)
    np.savez_compressed(os.path.join(OUT, f"fab_{tag}.npz"), **out)


def cmp(a, b):
    A = np.load(os.path.join(OUT, f"fab_{a}.npz"))
    B = np.load(os.path.join(OUT, f"fab_{b}.npz"))
    bad = [key for key in A.files if not np.array_equal(A[key], B[key])]
    missing = set(A.files) ^ set(B.files)
    print(f"{len(A.files)} arrays, {len(bad)} differ, {len(missing)} missing: {bad[:10]} {sorted(missing)[:5]}")
    return 1 if bad or missing else 0


if __name__ == "__main__":
    if sys.argv[1] == "dump":
        dump(sys.argv[2])
    else:
        sys.exit(cmp(sys.argv[2], sys.argv[3]))
