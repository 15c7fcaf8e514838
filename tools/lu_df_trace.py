"""Timeline of one k_band_lu_df launch (per work item: grab, dependencies met, end) for config 2.

    python tools/lu_df_trace.py [C|D] [n k p]    (traces the dataflow kernel's streamed/early-start launch)
"""
import ctypes as C
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1509_07919_b200 as S  # noqa: E402
from paper_1509_07919_b200 import _lib  # noqa: E402


def decode(item, J, K, m_max, G=3):
    S = -(-m_max // 32)
    if item < S * J:
        return ("chain", item % J, item // J, 0)
    o = item - S * J
    w = 0
    while True:
        R = min(K, m_max - 32 * (w + 1))
        ng = ((R + 31) // 32 - 1 + G - 1) // G
        wn = J * ng
        if o < wn:
            return ("strip", o // ng, w, 1 + G * (o % ng))
        o -= wn
        w += 1


def main():
    kind = sys.argv[1] if len(sys.argv) > 1 else "C"
    n, k, p = (int(x) for x in sys.argv[2:5]) if len(sys.argv) > 4 else (200000, 200, 50)
    _lib.load().sap_dev_lu_df_trace_mode(1)
    G = int(os.environ.get("DF_GROUP", "0"))  # strips per worker item (lu.cu A.grp); 0: the launcher's choice
    _lib.load().sap_dev_lu_df_group(G)
    if G == 0:
        G = 2 if (kind == "D" and p <= 59) else 3  # launch_band_lu_df: exclusive panel SMs -> 2
    band, rhs = S.random_banded(n, k, 1.0, 1)
    src = torch.from_numpy(band).cuda()
    pk = S.PrecondKind.coupled if kind == "C" else S.PrecondKind.decoupled
    with S.Solver(p=p, precond=pk, device=0, lu_kernel=2) as s:
        for _ in range(3):
            s.setup(src, n, k)
        s.synchronize()
        print("t_factor_kernel ms", s.report()["t_factor_kernel"] * 1e3)
    lib = _lib.load()
    lib.sap_dev_lu_df_trace.restype = C.c_longlong
    cap = 1_000_000
    REC = 22  # lu.cu kDfRec: grab/end ns, grab/ready/marks 1-4/end clock, SM|CTA, panel_diag groups 0-8, rows end, chain stores done, release done
    buf = np.zeros(REC * cap, np.uint64)
    cnt = lib.sap_dev_lu_df_trace(buf.ctypes.data_as(C.POINTER(C.c_ulonglong)), cap)
    t = buf[: REC * cnt].reshape(cnt, REC).astype(np.int64)
    out = os.path.join(ROOT, "gpurun_out")
    os.makedirs(out, exist_ok=True)
    np.save(os.path.join(out, f"dftrace_{kind}.npy"), t)
    J = 2 * p if kind == "C" else p
    m_max = -(-n // p)
    valid = t[:, 1] > 0
    GHZ = 1.965  # clock64 -> ns
    t0 = t[valid, 0].min()
    grab, end = t[:, 0] - t0, t[:, 1] - t0
    ready = grab + (t[:, 3] - t[:, 2]) / GHZ  # dependencies met, from the SM clock
    print(f"items {cnt}, traced {valid.sum()}, span {(end[valid].max())/1e3:.1f} us")
    types = {}
    for i in range(cnt):
        if not valid[i]:
            continue
        ty, job, st, j = decode(i, J, k, m_max, G)
        skipped = t[i, 3] == 0
        d = types.setdefault(ty, [0, 0.0, 0.0, 0, np.zeros(5)])
        d[0] += 1
        if skipped:
            d[3] += 1
            continue
        d[1] += (ready[i] - grab[i]) / 1e3
        d[2] += (end[i] - ready[i]) / 1e3
        marks = [t[i, 3]] + [t[i, 4 + q] if t[i, 4 + q] > 0 else t[i, 3] for q in range(4)] + [t[i, 8]]
        d[4] += np.diff(marks) / GHZ / 1e3
    for ty, (c, wsum, ksum, sk, ph) in types.items():
        c2 = max(c - sk, 1)
        print(f"{ty:7s} n={c:6d} skipped={sk:5d} wait avg {wsum / c2:7.2f} us  work avg {ksum / c2:7.2f} us  "
              f"total work {ksum/1e3:.2f} ms; phases (us) " + " ".join(f"{x / c2:.2f}" for x in ph))
    # per CTA: busy (work) vs waiting vs idle
    ncta = int((t[valid, 9] & 0xffffffff).max()) + 1
    span = end[valid].max()
    work = sum((end[i] - ready[i]) for i in range(cnt) if valid[i] and t[i, 3] > 0)
    wait = sum((ready[i] - grab[i]) for i in range(cnt) if valid[i] and t[i, 3] > 0)
    print(f"CTAs {ncta}: work {work / (ncta * span):.2%}, dependency wait {wait / (ncta * span):.2%} of CTA-time")
    # critical path sample: job 0's panels
    ps = sorted((decode(i, J, k, m_max, G)[2], ready[i], end[i]) for i in range(cnt)
                if valid[i] and decode(i, J, k, m_max, G)[:2] == ("chain", 0))
    if len(ps) > 4:
        steps = np.diff([x[2] for x in ps])
        print(f"job 0 panel-to-panel: median {np.median(steps)/1e3:.2f} us, panel work median "
              f"{np.median([x[2]-x[1] for x in ps])/1e3:.2f} us")
    s0 = [(decode(i, J, k, m_max, G)[2], grab[i], ready[i], end[i]) for i in range(cnt)
          if valid[i] and decode(i, J, k, m_max, G)[:2] == ("strip", 0) and decode(i, J, k, m_max, G)[3] == 1]
    if s0:
        print("job 0 strip1 work median %.2f us, wait median %.2f us" % (
            np.median([x[3] - x[2] for x in s0]) / 1e3, np.median([x[2] - x[1] for x in s0]) / 1e3))
    for w in (5, 50, 100):
        sel = [i for i in range(cnt) if valid[i] and decode(i, J, k, m_max, G)[2] == w]
        if sel:
            print(f"step {w}: items {len(sel)} grab [{grab[sel].min()/1e3:.1f}, {grab[sel].max()/1e3:.1f}] "
                  f"end [{end[sel].min()/1e3:.1f}, {end[sel].max()/1e3:.1f}] us")


if __name__ == "__main__":
    main()
