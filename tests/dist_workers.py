"""Worker bodies for the multi-process tests (spawned; importable by name).

CPU workers (gloo, host buffers) check the host side of the multi-GPU path:
the sap_comm callbacks and a numpy model of the distributed SaP-C apply that
follows the same interface-slot plan as api.cu (left cross, local, right
cross; cross interfaces solved on both ranks; one g-halo exchange per apply).
GPU workers run the real DistributedSolver, several ranks sharing one GPU.
"""
from __future__ import annotations

import ctypes as C
import os
import sys
import traceback

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port, backend="gloo"):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group(backend, rank=rank, world_size=world)
    return dist


def run(fn, rank, world, port, q, *args):
    try:
        q.put((rank, fn(rank, world, port, *args)))
    except BaseException:  # noqa: BLE001
        q.put((rank, "ERROR\n" + traceback.format_exc()))


# ---------------------------------------------------------------------------
def comm_callbacks(rank, world, port):
    """Drive the sap_comm function pointers (through their ctypes thunks) on host buffers."""
    dist = _init(rank, world, port)
    from paper_1509_07919_b200.distributed import TorchComm
    comm = TorchComm(host_buffers=True)
    s = comm.struct
    out = {}
    v = np.array([rank + 1.0, 10.0 * rank, -1.0])
    rc = s.allreduce_sum(None, v.ctypes.data_as(C.POINTER(C.c_double)), 3)
    out["allreduce"] = (rc, v.tolist())
    n = 5
    sl = np.full(n, 100.0 * rank + 1)   # to the left neighbour
    sr = np.full(n, 100.0 * rank + 2)   # to the right neighbour
    rl, rr = np.zeros(n), np.zeros(n)
    hl, hr = rank > 0, rank < world - 1
    ptr = lambda a, on: a.ctypes.data if on else None  # noqa: E731
    rc = s.exchange(None, ptr(sl, hl), n if hl else 0, ptr(sr, hr), n if hr else 0, ptr(rl, hl), n if hl else 0,
                    ptr(rr, hr), n if hr else 0)
    out["exchange"] = (rc, rl.tolist(), rr.tolist())
    out["calls"] = dict(comm.calls)
    dist.barrier()
    dist.destroy_process_group()
    return out


# ---------------------------------------------------------------------------
def _local_band(band, k, lo, hi):
    """The global band's columns [lo, hi): the diagonal blocks of rows [lo, hi) (entries outside ignored)."""
    w = 2 * k + 1
    return np.ascontiguousarray(band[lo * w:hi * w])


def dist_apply_model(rank, world, port, n, k, p, d, seed):
    """Numpy model of apply_m_dist (api.cu) on the oracle's factors; returns this rank's rows of M^{-1} r."""
    dist = _init(rank, world, port)
    import oracle as O
    from paper_1509_07919_b200.distributed import TorchComm
    comm = TorchComm(host_buffers=True)
    band, rhs = O.random_banded(n, k, d, seed)
    sizes, offs = O.partition_layout(n, p, k)
    offs = list(offs)
    pb, pe = rank * p // world, (rank + 1) * p // world
    lo, hi = offs[pb], offs[pe]
    nl, pl, w = hi - lo, pe - pb, k
    sp = O.spikes(n, k, band, p)
    blk = lambda a, t: a[t * w * w:(t + 1) * w * w].reshape(w, w)  # noqa: E731
    has_l, has_r = lo > 0, hi < n
    lc, rc = int(has_l), int(has_r)
    # interface slots [left cross?, local..., right cross?] -> global interface index and own-row position
    slots = []
    for t in range(lc + pl - 1 + rc):
        li = t - lc  # -1: left cross, pl-1: right cross
        slots.append((pb - lc + t, 0 if li < 0 else offs[pb + li + 1] - lo))
    loc_band = _local_band(band, k, lo, hi)
    dinv = lambda v: O.apply(nl, k, loc_band, pl, 1, v)  # noqa: E731 - decoupled = D^{-1} on own blocks
    r = rhs[lo:hi].copy()
    g = np.zeros(nl + 2 * w)
    g[w:w + nl] = dinv(r)
    gv = g[w:w + nl]
    # one exchange: my first / last w rows of g to the neighbours, halos back
    sl, sr = gv[:w].copy(), gv[nl - w:].copy()
    rl, rr = np.zeros(w), np.zeros(w)
    ptr = lambda a, on: a.ctypes.data if on else None  # noqa: E731
    rcode = comm.struct.exchange(None, ptr(sl, has_l), w if has_l else 0, ptr(sr, has_r), w if has_r else 0,
                                 ptr(rl, has_l), w if has_l else 0, ptr(rr, has_r), w if has_r else 0)
    assert rcode == 0
    g[:w], g[w + nl:] = rl, rr
    b2 = r.copy()
    for t, (gi, e) in enumerate(slots):
        W, V, B, Cc = blk(sp["wt"], gi), blk(sp["vb"], gi), blk(sp["B"], gi), blk(sp["C"], gi)
        rbar = np.eye(w) - W @ V
        ge = w + e  # position of the interface in g
        xt = np.linalg.solve(rbar, g[ge:ge + w] - W @ g[ge - w:ge])
        xb = g[ge - w:ge] - V @ xt
        if not (t == 0 and has_l):  # the B update lands on the left rank's rows
            b2[e - w:e] -= B @ xt
        if not (t == len(slots) - 1 and has_r):  # the C update lands on the right rank's rows
            b2[e:e + w] -= Cc @ xb
    out = dinv(b2)
    dist.barrier()
    dist.destroy_process_group()
    return out.tolist()


# ---------------------------------------------------------------------------
def gpu_dist_solve(rank, world, port, n, k, p, d, seed, precond):
    """The real DistributedSolver (gloo, ranks share cuda:0): setup, apply, matvec, solve."""
    dist = _init(rank, world, port)
    import torch
    import oracle as O
    from paper_1509_07919_b200 import KrylovOptions, PrecondKind
    from paper_1509_07919_b200.distributed import DistributedSolver, TorchComm
    torch.cuda.set_device(0)
    comm = TorchComm()
    band, rhs = O.random_banded(n, k, d, seed)
    s = DistributedSolver(comm, p=p, precond=PrecondKind(precond), krylov=KrylovOptions())
    s.setup_from_global(band, n, k)
    lo, hi = s.row_lo, s.row_hi
    res = {"rows": (lo, hi)}
    res["apply"] = s.apply_preconditioner(rhs[lo:hi].copy()).tolist()
    xg = np.sin(np.arange(n) * 0.37)
    res["matvec"] = s.matvec(xg[lo:hi].copy()).tolist()
    # device-pointer path too
    rd = torch.tensor(rhs[lo:hi], device="cuda:0")
    torch.cuda.synchronize()
    dev = s.apply_preconditioner(rd).cpu().numpy()
    res["apply_dev_equal"] = bool(np.array_equal(dev, np.array(res["apply"])))
    x, st = s.solve(rhs[lo:hi].copy())
    res["x"] = x.tolist()
    res["iterations"] = st.iterations
    res["converged"] = st.converged
    res["report"] = s.report()
    res["calls"] = dict(comm.calls)
    s.close()
    dist.barrier()
    dist.destroy_process_group()
    return res


def gpu_nccl_solve(rank, world, port, n, k, p, d, seed, precond):
    """The native NCCL data plane (sap_create_distributed_nccl; torch.distributed only bootstraps the id):
    one rank per GPU. On a one-GPU box world = 1 (NCCL refuses two ranks on one device)."""
    dist = _init(rank, world, port)
    import torch
    import oracle as O
    from paper_1509_07919_b200 import KrylovOptions, PrecondKind
    from paper_1509_07919_b200.distributed import DistributedSolver, NcclComm
    torch.cuda.set_device(rank)
    comm = NcclComm()
    band, rhs = O.random_banded(n, k, d, seed)
    s = DistributedSolver(comm, p=p, precond=PrecondKind(precond), krylov=KrylovOptions(), device=rank)
    s.setup_from_global(band, n, k)
    lo, hi = s.row_lo, s.row_hi
    res = {"rows": (lo, hi)}
    res["apply"] = s.apply_preconditioner(rhs[lo:hi].copy()).tolist()
    xg = np.sin(np.arange(n) * 0.37)
    res["matvec"] = s.matvec(xg[lo:hi].copy()).tolist()
    x, st = s.solve(rhs[lo:hi].copy())
    res["x"] = x.tolist()
    res["iterations"] = st.iterations
    res["converged"] = st.converged
    res["history"] = list(st.residual_history)
    s.close()
    dist.barrier()
    dist.destroy_process_group()
    return res
