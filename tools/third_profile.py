"""One third-stage SaP-C setup at config-2 size for ncu (argv[1]: 'scrambled' (K_b = 10) or 'full' (K_b = K))."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_1509_07919_b200 as S  # noqa: E402

n, k, p = 200000, 200, 50
case = sys.argv[1] if len(sys.argv) > 1 else "scrambled"
if case == "full":
    bandh, _ = S.random_banded(n, k, 1.0, 1)
    kb, perms = np.full(p, k, np.int32), None
else:
    kn, win = 10, 40
    rng = np.random.default_rng(3)
    pos = np.arange(n)
    w0 = (pos // win) * win
    perm = w0 + win - 1 - (pos - w0)
    bandh = np.zeros(n * (2 * k + 1))
    rowsum = np.zeros(n)
    for d in range(-kn, kn + 1):
        if d == 0:
            continue
        i = np.arange(max(0, -d), min(n, n - d))
        v = rng.uniform(-1, 1, i.size)
        v[v == 0] = 0.5
        rowsum[i] += np.abs(v)
        bandh[perm[i + d] * (2 * k + 1) + (perm[i] - perm[i + d] + k)] = v
    bandh[perm * (2 * k + 1) + k] = rowsum
    kb, hp, pm = O.ref_third_stage(n, k, bandh, p, 0)
    lay = S.make_partition_layout(n, p, k)
    perms = [pm[o:o + m] if h else None for o, m, h in zip(lay.offsets, lay.sizes, hp)]
band = torch.from_numpy(bandh).cuda()
s = S.Solver(p=p, precond=0)
s.set_third_stage(kb, perms)
for _ in range(2):
    s.setup(band, n, k)
torch.cuda.synchronize()
print(s.report()["t_spk"])
