"""Dataflow LU: factor-kernel time vs strips per worker item (lu.cu A.grp), config 2 (N 200k, K 200, P 50),
SaP-C and SaP-D; the factors must be bitwise the same for every group size.

    python tools/lu_df_group.py            # on a GPU box
"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1509_07919_b200 as S  # noqa: E402
from paper_1509_07919_b200 import _lib  # noqa: E402


def main():
    n, k, p = 200000, 200, 50
    band, _ = S.random_banded(n, k, 1.0, 1)
    src = torch.from_numpy(band).cuda()
    lib = _lib.load()
    for kind in (S.PrecondKind.decoupled, S.PrecondKind.coupled):
        ref = None
        for g in (1, 2, 3, 0):
            lib.sap_dev_lu_df_group(g)
            ts = []
            with S.Solver(p=p, precond=kind, device=0) as s:
                for _ in range(7):
                    s.setup(src, n, k)
                    s.synchronize()
                    ts.append(s.report()["t_factor_kernel"] * 1e3)
                lu = s.factors(0)[0]
            same = True if ref is None else np.array_equal(ref, lu)
            ref = lu if ref is None else ref
            print(f"{'C' if kind == S.PrecondKind.coupled else 'D'} group {g or 'auto'}: factor kernel ms "
                  f"median {np.median(ts[2:]):.3f} min {min(ts[2:]):.3f}  bitwise {same}", flush=True)
    lib.sap_dev_lu_df_group(0)


if __name__ == "__main__":
    main()
