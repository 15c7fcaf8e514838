"""Third-stage setup + solve timing at config-2 size (N = 200 000, K = 200, P = 50, SaP-C), against the
plain truncated-SPIKE setup. Cases: identity blocks at K_b = K (full spikes at w = 200: the worst case
for the full-spike solve) and a scrambled band whose blocks Cuthill-McKee narrows (oracle.scrambled_banded
is too slow in Python at this size, so the scrambled case is built here with numpy)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_07919_b200 as S  # noqa: E402

n, k, p = 200000, 200, 50


def timed(s, band, rhs, reps=4):
    stream = torch.cuda.Stream()
    s.set_stream(stream)
    best = None
    with torch.cuda.stream(stream):
        for i in range(reps):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            s.setup(band, n, k)
            x, st = s.solve(rhs)
            e1.record(stream)
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1)
            if i and (best is None or t < best[0]):
                best = (t, s.report(), st)
    return best


def show(name, best):
    t, r, st = best
    print(f"{name}: {t:.3f} ms  t_lu {r['t_lu'] * 1e3:.3f}  t_bc {r['t_bc'] * 1e3:.3f}  t_spk {r['t_spk'] * 1e3:.3f}  "
          f"t_lurdcd {r['t_lurdcd'] * 1e3:.3f}  t_kry {r['t_kry'] * 1e3:.3f}  it {st.iterations}  "
          f"res {st.final_relative_residual:.2e}", flush=True)


band_h, rhs_h = S.random_banded(n, k, 1.0, 1)
band = torch.from_numpy(band_h).cuda()
rhs = torch.from_numpy(rhs_h).cuda()
for kind in (0, 1):
    s = S.Solver(p=p, precond=kind)
    show(f"{'SaP-C' if kind == 0 else 'SaP-D'} plain", timed(s, band, rhs))
    s.set_third_stage(np.full(p, k, np.int32), None)
    show(f"{'SaP-C' if kind == 0 else 'SaP-D'} third stage, identity blocks K_b = K", timed(s, band, rhs))
    # every block reversed (a permutation that keeps the bandwidth): exercises the permuted paths at w = K
    lay = S.make_partition_layout(n, p, k)
    perms = [np.arange(m, dtype=np.int32)[::-1].copy() for m in lay.sizes]
    s.set_third_stage(np.full(p, k, np.int32), perms)
    show(f"{'SaP-C' if kind == 0 else 'SaP-D'} third stage, reversed blocks K_b = K", timed(s, band, rhs))
    s.close()

# scrambled band (oracle.scrambled_banded's construction, vectorized): kn = 10 band, windows of 40
# reversed, stored at K = 200; sap::third_stage (compiled reference) narrows every block back to 10
import oracle as O  # noqa: E402  (tools only: the reference's third_stage computes the permutations)

if O.has_ref():
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
        pi, pj = perm[i], perm[i + d]
        bandh[pj * (2 * k + 1) + (pi - pj + k)] = v
    bandh[perm * (2 * k + 1) + k] = rowsum
    kb, hp, pm = O.ref_third_stage(n, k, bandh, p, 0)
    lay = S.make_partition_layout(n, p, k)
    perms = [pm[o:o + m] if h else None for o, m, h in zip(lay.offsets, lay.sizes, hp)]
    print(f"scrambled: K_b {sorted(set(kb.tolist()))}, permuted blocks {int(hp.sum())}/{p}", flush=True)
    bandd = torch.from_numpy(bandh).cuda()
    for kind in (0, 1):
        s = S.Solver(p=p, precond=kind)
        show(f"{'SaP-C' if kind == 0 else 'SaP-D'} plain (scrambled)", timed(s, bandd, rhs))
        s.set_third_stage(kb, perms)
        show(f"{'SaP-C' if kind == 0 else 'SaP-D'} third stage (scrambled)", timed(s, bandd, rhs))
        s.close()
