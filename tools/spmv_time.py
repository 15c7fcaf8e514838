"""Banded SpMV (the Krylov A-operator) timing at config 2: us per call and achieved HBM GB/s."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_1509_07919_b200 as S  # noqa: E402

n, k = 200000, 200
band_h, rhs_h = S.random_banded(n, k, 1.0, 1)
band = torch.from_numpy(band_h).cuda()
x = torch.from_numpy(rhs_h).cuda()
y = torch.empty_like(x)
s = S.Solver(p=50, precond=S.PrecondKind.none)
s.setup(band, n, k)
for _ in range(5):
    s.matvec(x, y)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(50):
    s.matvec(x, y)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / 50
gb = (8.0 * n * (2 * k + 1) + 16.0 * n) / (us * 1e-6) / 1e9
print(f"banded SpMV: {us:.1f} us per call, {gb:.0f} GB/s algorithmic")
