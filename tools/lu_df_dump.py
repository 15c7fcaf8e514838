"""Dump LU/UL factor stores of the single-CTA and the dataflow kernel for one case (debugging aid).
    python tools/lu_df_dump.py n k d p [C|D] [dev]"""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1509_07919_b200 as S  # noqa: E402

n, k, p = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[4])
d = float(sys.argv[3])
kind = S.PrecondKind.coupled if (len(sys.argv) < 6 or sys.argv[5] == "C") else S.PrecondKind.decoupled
dev = len(sys.argv) > 6 and sys.argv[6] == "dev"
band, rhs = S.random_banded(n, k, d, 1)
out = {}
for df in (0, 1):
    with S.Solver(p=p, precond=kind, device=0, lu_kernel=2 if df else 1) as s:
        s.setup(torch.from_numpy(band).cuda() if dev else band, n, k)
        s.synchronize()
        out[f"lu{df}"] = s.factors(0)[0]
        if kind == S.PrecondKind.coupled:
            out[f"ul{df}"] = s.factors(1)[0]
w = 2 * k + 1
sizes = S.make_partition_layout(n, p, k).sizes
for nm in ("lu", "ul"):
    if nm + "0" not in out:
        continue
    off = 0
    for blk, m in enumerate(sizes):
        x = out[nm + "0"][off: off + m * w].reshape(m, w)
        y = out[nm + "1"][off: off + m * w].reshape(m, w)
        off += m * w
        bad = np.argwhere(x != y)
        if len(bad) == 0:
            continue
        cols = np.unique(bad[:, 0])
        print(f"{nm} block {blk} m={m}: {len(bad)} bad entries in {len(cols)} columns; steps {sorted(set((cols // 32).tolist()))[:20]}")
        for c in cols[:6]:
            rows = bad[bad[:, 0] == c][:, 1] - k + c
            print(f"   col {c} (step {c // 32}, col-in-step {c % 32}): rows {rows[:12].tolist()} ... n={len(rows)}; "
                  f"in-matrix {[(0 <= r < m) for r in rows[:6]]}")
        break
