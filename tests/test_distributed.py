"""Multi-GPU path: partitions sharded over ranks.

CPU (gloo, world_size 2 and 3): rank row assignment, the sap_comm callbacks,
and a numpy model of the distributed SaP-C apply — the same interface-slot
plan as api.cu — against the oracle's single-process apply.
GPU: the real DistributedSolver with several ranks sharing cuda:0 over gloo;
the distributed apply and matvec must equal the single-GPU ones bit for bit
(same kernels on the same blocks), the solve must converge like it.
"""
import multiprocessing as mp
import socket

import numpy as np
import pytest

import dist_workers as W


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _spawn(fn, world, *args, timeout=240):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=W.run, args=(fn, r, world, port, q, *args)) for r in range(world)]
    for p in procs:
        p.start()
    out = {}
    try:
        for _ in range(world):
            r, v = q.get(timeout=timeout)
            out[r] = v
    finally:
        for p in procs:
            p.join(timeout=30)
            if p.is_alive():
                p.kill()
    for r, v in out.items():
        assert not (isinstance(v, str) and v.startswith("ERROR")), f"rank {r}:\n{v}"
    return [out[r] for r in range(world)]


@pytest.mark.parametrize("n,p,k,world", [(1000, 4, 10, 2), (1001, 7, 10, 3), (200000, 50, 200, 8),
                                         (97, 3, 0, 3), (5000, 16, 31, 4)])
def test_rank_rows_partition_cover(sap, n, p, k, world):
    from paper_1509_07919_b200.distributed import rank_rows
    lay = sap.make_partition_layout(n, p, k)
    prev = 0
    for r in range(world):
        lo, hi = rank_rows(n, p, k, r, world)
        assert lo == prev and hi > lo
        assert lo in lay.offsets and hi in lay.offsets
        prev = hi
    assert prev == n


def test_rank_rows_errors(sap):
    from paper_1509_07919_b200.distributed import rank_rows
    with pytest.raises(ValueError, match="fewer partitions than ranks"):
        rank_rows(1000, 2, 10, 0, 4)
    with pytest.raises(ValueError, match="rank out of range"):
        rank_rows(1000, 4, 10, 4, 4)
    with pytest.raises(ValueError, match="largest feasible p"):
        rank_rows(100, 8, 10, 0, 2)


@pytest.mark.parametrize("world", [2, 3])
def test_comm_callbacks_gloo(world):
    res = _spawn(W.comm_callbacks, world)
    for r, o in enumerate(res):
        rc, v = o["allreduce"]
        assert rc == 0
        assert v == [sum(q + 1.0 for q in range(world)), sum(10.0 * q for q in range(world)), -1.0 * world]
        rc, rl, rr = o["exchange"]
        assert rc == 0
        if r > 0:
            assert rl == [100.0 * (r - 1) + 2] * 5  # left neighbour's send_right
        if r < world - 1:
            assert rr == [100.0 * (r + 1) + 1] * 5  # right neighbour's send_left
        assert o["calls"] == {"allreduce": 1, "exchange": 1}


@pytest.mark.parametrize("n,k,p,d,world", [(2000, 8, 4, 1.0, 2), (3001, 12, 6, 0.6, 3), (2400, 10, 5, 0.3, 2)])
def test_distributed_apply_model_matches_oracle(oracle, n, k, p, d, world):
    res = _spawn(W.dist_apply_model, world, n, k, p, d, 7)
    got = np.concatenate([np.array(v) for v in res])
    band, rhs = oracle.random_banded(n, k, d, 7)
    ref = oracle.apply(n, k, band, p, 0, rhs)
    assert got.shape == ref.shape
    np.testing.assert_allclose(got, ref, rtol=0, atol=1e-9 * np.abs(ref).max())


# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("n,k,p,d,world,precond", [(20000, 20, 8, 1.0, 2, 0), (30001, 16, 12, 0.6, 3, 0),
                                                   (20000, 20, 8, 1.0, 2, 1), (24000, 8, 8, 0.5, 4, 0)])
def test_gpu_distributed_matches_single(sap, oracle, n, k, p, d, world, precond):
    res = _spawn(W.gpu_dist_solve, world, n, k, p, d, 11, precond, timeout=600)
    band, rhs = oracle.random_banded(n, k, d, 11)
    single = sap.Solver(p=p, precond=sap.PrecondKind(precond))
    single.setup(band, n, k)
    ap = single.apply_preconditioner(rhs)
    xg = np.sin(np.arange(n) * 0.37)
    mv = single.matvec(xg)
    x1, st1 = single.solve(rhs)
    rows = [tuple(r["rows"]) for r in res]
    assert rows[0][0] == 0 and rows[-1][1] == n
    # same kernels on the same blocks and interfaces: bitwise equal
    np.testing.assert_array_equal(np.concatenate([r["apply"] for r in res]), ap)
    np.testing.assert_array_equal(np.concatenate([r["matvec"] for r in res]), mv)
    assert all(r["apply_dev_equal"] for r in res)
    # Krylov dots are summed over ranks in a different order: same convergence, not bitwise
    its = {r["iterations"] for r in res}
    assert len(its) == 1, its
    assert all(r["converged"] for r in res) and st1.converged
    assert abs(res[0]["iterations"] - st1.iterations) <= 0.5
    x = np.concatenate([r["x"] for r in res])
    assert np.linalg.norm(x - x1) <= 1e-8 * np.linalg.norm(x1)
    rep = res[0]["report"]
    assert rep["partitions"] == p and rep["n"] == n
    assert all(r["calls"]["exchange"] > 0 for r in res)


@pytest.mark.gpu
@pytest.mark.parametrize("precond", [0, 1])
def test_gpu_native_nccl_world1_matches_single(sap, oracle, precond):
    """The library's own NCCL communicator (ncclCommInitRank from an id broadcast over torch.distributed,
    exchanges as ncclSend/ncclRecv on the handle's stream, Krylov dots as device ncclAllReduce) at the world
    size one GPU allows: bitwise the single-GPU setup, apply, operator and solve."""
    n, k, p, d = 20000, 20, 8, 1.0
    res = _spawn(W.gpu_nccl_solve, 1, n, k, p, d, 11, precond, timeout=600)[0]
    band, rhs = oracle.random_banded(n, k, d, 11)
    single = sap.Solver(p=p, precond=sap.PrecondKind(precond))
    single.setup(band, n, k)
    assert tuple(res["rows"]) == (0, n)
    np.testing.assert_array_equal(np.array(res["apply"]), single.apply_preconditioner(rhs))
    np.testing.assert_array_equal(np.array(res["matvec"]), single.matvec(np.sin(np.arange(n) * 0.37)))
    x1, st1 = single.solve(rhs)
    assert res["converged"] and res["iterations"] == st1.iterations
    assert np.linalg.norm(np.array(res["x"]) - x1) <= 1e-12 * np.linalg.norm(x1)
