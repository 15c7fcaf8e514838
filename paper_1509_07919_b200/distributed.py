"""Multi-GPU SaP over torch.distributed: one process per GPU.

The partitions of ``make_partition_layout(n, p, k)`` are sharded across ranks
in order — rank r owns partitions ``[r*p/world, (r+1)*p/world)`` and the
matching rows (``rank_rows``). Factorization is rank-local; at setup the
neighbours swap one w x w spike tip each way, and every rank-crossing
interface's reduced block is built and factored on both of its ranks. Every
preconditioner apply then needs ONE neighbour exchange of w = k rows each way,
every operator apply one k-row halo exchange, and every Krylov reduction a
scalar allreduce (the reference's single-process spike.hpp:304-351 /
krylov.hpp:110-442 data flow, cut at partition boundaries).

``NcclComm`` selects the library's native data plane (``sap_create_distributed_nccl``): grouped
ncclSend / ncclRecv on the handle's stream for every exchange and device-side ncclAllReduce for the Krylov
dots, no Python on the data path; the torch.distributed group only carries the 128-byte NCCL id once.

``TorchComm`` supplies the ``sap_comm`` callbacks of include/sap_gpu.h instead (the CPU tests and the
several-ranks-on-one-GPU GPU tests, where NCCL cannot run):

* backend ``nccl``: device buffers are sent as-is (``batch_isend_irecv``),
* backend ``gloo``: device buffers are staged through host tensors — the way
  the CPU tests and the several-ranks-on-one-GPU GPU tests run.

``host_buffers=True`` makes ``exchange`` treat the pointers as host memory
(the CPU tests drive the callbacks without a GPU that way).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .solver import KrylovOptions, PartitionLayout, PrecondKind, Solver, _check, _is_cuda_tensor, make_partition_layout


def rank_rows(n: int, p: int, k: int, rank: int, world: int) -> tuple[int, int]:
    """[row_lo, row_hi) of `rank` (sap_rank_rows)."""
    lo, hi = C.c_int(), C.c_int()
    _check(L.load().sap_rank_rows(n, p, k, rank, world, C.byref(lo), C.byref(hi)))
    return lo.value, hi.value


def band_slice_columns(n: int, k: int, row_lo: int, row_hi: int) -> tuple[int, int]:
    """Global band columns a rank's slice must hold: [max(0, row_lo-k), min(n, row_hi+k))."""
    return max(0, row_lo - k), min(n, row_hi + k)


class _CudaArray:
    """A raw device pointer as a __cuda_array_interface__ object (no copy)."""

    def __init__(self, ptr: int, count: int):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": "<f8", "data": (ptr, False), "version": 3,
                                         "strides": None}


class TorchComm:
    """sap_comm callbacks over a torch.distributed process group."""

    def __init__(self, group=None, host_buffers: bool = False):
        import torch
        import torch.distributed as dist
        self._torch = torch
        self._dist = dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = str(dist.get_backend(group))
        self.host_buffers = host_buffers
        self.error: BaseException | None = None
        self.calls = {"allreduce": 0, "exchange": 0}
        # keep the ctypes thunks alive as long as this object
        self._ar = L.ALLREDUCE_FN(self._allreduce)
        self._ex = L.EXCHANGE_FN(self._exchange)
        self.struct = L.sap_comm(None, self.rank, self.world, self._ar, self._ex)

    def _peer(self, r: int) -> int:
        return r if self.group is None else self._dist.get_global_rank(self.group, r)

    # -- callbacks (return 0 = ok; an exception is recorded and reported as a failure) --------
    def _allreduce(self, _ctx, ptr, count):
        try:
            self.calls["allreduce"] += 1
            torch = self._torch
            host = torch.from_numpy(np.ctypeslib.as_array(ptr, shape=(count,)))
            if self.backend == "nccl":
                t = host.to(f"cuda:{torch.cuda.current_device()}")
                self._dist.all_reduce(t, group=self.group)
                host.copy_(t.cpu())
            else:
                self._dist.all_reduce(host, group=self.group)
            return 0
        except BaseException as e:  # noqa: BLE001 - must not unwind through C
            self.error = e
            return 1

    def _view(self, ptr, count):
        torch = self._torch
        if self.host_buffers:
            return torch.from_numpy(np.ctypeslib.as_array(C.cast(ptr, C.POINTER(C.c_double)), shape=(count,)))
        return torch.as_tensor(_CudaArray(ptr, count), device=f"cuda:{torch.cuda.current_device()}")

    def _exchange(self, _ctx, sl, n_sl, sr, n_sr, rl, n_rl, rr, n_rr):
        try:
            self.calls["exchange"] += 1
            dist, torch = self._dist, self._torch
            left, right = self._peer(self.rank - 1), self._peer(self.rank + 1)
            plan = []  # (op, device view, peer)
            if n_rl:
                plan.append((dist.irecv, self._view(rl, n_rl), left))
            if n_rr:
                plan.append((dist.irecv, self._view(rr, n_rr), right))
            if n_sl:
                plan.append((dist.isend, self._view(sl, n_sl), left))
            if n_sr:
                plan.append((dist.isend, self._view(sr, n_sr), right))
            if not plan:
                return 0
            staged = self.backend != "nccl" and not self.host_buffers
            bufs = [v.cpu() if staged else v for _, v, _ in plan]
            if self.backend == "nccl":
                reqs = dist.batch_isend_irecv([dist.P2POp(op, b, peer, group=self.group)
                                               for (op, _, peer), b in zip(plan, bufs)])
            else:
                reqs = [op(b, peer, group=self.group) for (op, _, peer), b in zip(plan, bufs)]
            for q in reqs:
                q.wait()
            if staged:
                for (op, v, _), b in zip(plan, bufs):
                    if op is dist.irecv:
                        v.copy_(b)
            if not self.host_buffers and torch.cuda.is_available():
                torch.cuda.current_stream().synchronize()
            return 0
        except BaseException as e:  # noqa: BLE001
            self.error = e
            return 1


class NcclComm:
    """The library's own NCCL communicator (one process per GPU). Collective: every rank of `group`
    constructs it; rank 0's ``sap_nccl_get_unique_id`` reaches the others through torch.distributed."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.error: BaseException | None = None
        uid = np.zeros(128, np.uint8)
        if self.rank == 0:
            _check(L.load().sap_nccl_get_unique_id(uid.ctypes.data))
        t = torch.from_numpy(uid)
        if str(dist.get_backend(group)) == "nccl":
            t = t.to(f"cuda:{torch.cuda.current_device()}")
        src = 0 if group is None else dist.get_global_rank(group, 0)
        dist.broadcast(t, src=src, group=group)
        self.uid = np.ascontiguousarray(t.cpu().numpy(), np.uint8)


class DistributedSolver(Solver):
    """Solver whose partitions are sharded over the ranks of a TorchComm.

    Vectors passed to apply_preconditioner / matvec / solve are this rank's
    rows [row_lo, row_hi); ``factor(part)`` / ``spike(t)`` take GLOBAL
    partition / interface indices owned by (or crossing into) this rank.
    """

    def __init__(self, comm: "TorchComm | NcclComm", p: int, precond: PrecondKind = PrecondKind.coupled,
                 boost_eps: float = 1e-10, krylov: KrylovOptions | None = None, device: int = 0):
        self.comm = comm
        super().__init__(p=p, precond=precond, boost_eps=boost_eps, krylov=krylov, device=device)
        self.row_lo = self.row_hi = 0

    def _create(self) -> None:
        if isinstance(self.comm, NcclComm):
            _check(L.load().sap_create_distributed_nccl(C.byref(self.options), self.comm.uid.ctypes.data,
                                                        self.comm.rank, self.comm.world, C.byref(self._h)))
        else:
            _check(L.load().sap_create_distributed(C.byref(self.options), C.byref(self.comm.struct),
                                                   C.byref(self._h)))

    def rows(self, n: int, k: int) -> tuple[int, int]:
        return rank_rows(n, self.p, k, self.comm.rank, self.comm.world)

    def setup(self, band_slice, n: int, k: int) -> None:  # noqa: D401 - same name as Solver.setup
        """Collective. band_slice = global band columns band_slice_columns(n, k, *rows(n, k))."""
        lo, hi = self.rows(n, k)
        c0, c1 = band_slice_columns(n, k, lo, hi)
        if not _is_cuda_tensor(band_slice):
            band_slice = np.ascontiguousarray(band_slice, dtype=np.float64).reshape(-1)
        size = int(band_slice.numel() if _is_cuda_tensor(band_slice) else band_slice.size)
        if size != (c1 - c0) * (2 * k + 1):
            raise ValueError("setup: band slice must hold the columns [max(0,row_lo-k), min(n,row_hi+k))")
        ptr, dev = self._ptr(band_slice)
        rc = L.load().sap_setup_banded_dist(self._h, n, k, lo, hi, ptr, dev)
        self._raise_comm()
        _check(rc)
        self.n, self.k, self.row_lo, self.row_hi = n, k, lo, hi
        self.layout = make_partition_layout(n, self.p, k)

    def setup_from_global(self, band, n: int, k: int) -> None:
        """Slice this rank's columns out of the full band (host array or CUDA tensor) and set up."""
        lo, hi = self.rows(n, k)
        c0, c1 = band_slice_columns(n, k, lo, hi)
        w = 2 * k + 1
        self.setup(band[c0 * w:c1 * w], n, k)

    def local_partitions(self) -> range:
        pb = self.layout.offsets.index(self.row_lo)
        pe = self.layout.offsets.index(self.row_hi)
        return range(pb, pe)

    def factors(self, which: int = 0):
        parts = [self.factor(i, which) for i in self.local_partitions()]
        return (np.concatenate([q[0] for q in parts]), np.array([q[1] for q in parts], np.int32),
                np.array([q[2] for q in parts]))

    def _raise_comm(self):
        if self.comm.error is not None:
            e, self.comm.error = self.comm.error, None
            raise RuntimeError(f"communication callback failed: {e!r}") from e

    def _op(self, fn, x, out):
        try:
            return super()._op(fn, x, out)
        finally:
            self._raise_comm()

    def solve(self, b, x=None, history_capacity: int | None = None):
        try:
            return super().solve(b, x, history_capacity)
        finally:
            self._raise_comm()


__all__ = ["TorchComm", "NcclComm", "DistributedSolver", "rank_rows", "band_slice_columns", "PartitionLayout"]
