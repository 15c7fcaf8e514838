"""Host-side mirror of the reference SaP interface over the C ABI.

Names, argument meaning and error behaviour follow /root/reference/proj:

* ``make_partition_layout`` / ``max_feasible_partitions``  — partition.hpp:34-69
  (``ValueError`` ≙ ``std::invalid_argument`` with the reference's message)
* ``PrecondKind``, ``KrylovMethod``, ``KrylovFailure``    — spike.hpp:14, krylov.hpp:16-18
* ``KrylovOptions``, ``SolveStats``                       — krylov.hpp:20-41
* ``Solver.setup``      ≙ ``detail::build_precond_op``   — pipeline.hpp:140-202
* ``Solver.apply_preconditioner`` / ``Solver.matvec``     — the M / A ``LinearOp`` (krylov.hpp:14)
* ``Solver.solve``      ≙ ``run_krylov``                 — krylov.hpp:434-442
* ``PreconditionerError`` ≙ ``sap::PreconditionerError``  — errors.hpp:17-20

Vectors may be numpy arrays (host) or CUDA tensors (``torch.Tensor`` on the
handle's device, passed as device pointers: no host round trip).
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass, field

import numpy as np

from . import _lib as L


class PreconditionerError(RuntimeError):
    """sap::PreconditionerError (errors.hpp:17-20)."""


class StateError(RuntimeError):
    """Call made out of order (e.g. solve before setup)."""


class CudaError(RuntimeError):
    pass


class PrecondKind(enum.IntEnum):
    coupled = 0
    decoupled = 1
    diagonal = 2
    none = 3


class KrylovMethod(enum.IntEnum):
    bicgstab_l = 0
    cg = 1
    automatic = 2


class KrylovFailure(enum.IntEnum):
    none = 0
    max_iterations = 1
    breakdown = 2
    non_finite = 3
    indefinite_operator = 4


def _check(rc: int) -> None:
    if rc == 0:
        return
    msg = L.load().sap_last_error().decode()
    if rc == 1:
        raise ValueError(msg)
    if rc == 2:
        raise PreconditionerError(msg)
    if rc == 5:
        raise StateError(msg)
    raise CudaError(f"{L.load().sap_status_string(rc).decode()}: {msg}")


@dataclass
class PartitionLayout:
    p: int
    sizes: list
    offsets: list
    remainder: int
    per_partition_k: list

    def total(self) -> int:
        return self.offsets[-1] if self.offsets else 0


def max_feasible_partitions(n: int, k: int) -> int:
    return int(L.load().sap_max_feasible_partitions(n, k))


def make_partition_layout(n: int, p: int, k: int) -> PartitionLayout:
    sizes = (C.c_int * max(p, 1))()
    offs = (C.c_int * (max(p, 1) + 1))()
    _check(L.load().sap_partition_layout(n, p, k, sizes, offs))
    return PartitionLayout(p=p, sizes=list(sizes)[:p], offsets=list(offs)[:p + 1], remainder=n % p,
                           per_partition_k=[k] * p)


def random_banded(n: int, k: int, d: float, seed: int, with_rhs: bool = True):
    """testsup::random_banded (+ random_rhs) with the reference's mt19937 stream."""
    band = np.zeros(n * (2 * k + 1))
    rhs = np.zeros(n) if with_rhs else None
    _check(L.load().sap_random_banded(n, k, d, seed, band.ctypes.data, rhs.ctypes.data if with_rhs else None))
    return (band, rhs) if with_rhs else band


@dataclass
class KrylovOptions:
    method: KrylovMethod = KrylovMethod.bicgstab_l
    ell: int = 2
    rel_tol: float = 1e-10
    abs_tol: float = 0.0
    max_iterations: int = 500
    mixed_precision: bool = False
    caller_asserts_spd: bool = False


@dataclass
class SolveStats:
    iterations: float = 0.0
    residual_history: list = field(default_factory=list)
    converged: bool = False
    final_relative_residual: float = 0.0
    failure: KrylovFailure = KrylovFailure.none


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(x.is_cuda)


class Solver:
    """SaP setup()/solve() over libsap_gpu (one handle, one CUDA stream)."""

    def __init__(self, p: int = 1, precond: PrecondKind = PrecondKind.coupled, boost_eps: float = 1e-10,
                 krylov: KrylovOptions | None = None, device: int = 0, triangle_solve: int = 0,
                 lu_kernel: int = 0, tip_solve: int = 0):
        kr = krylov or KrylovOptions()
        o = L.sap_options()
        L.load().sap_options_default(C.byref(o))
        o.p, o.precond, o.boost_eps = int(p), int(precond), float(boost_eps)
        o.method, o.ell, o.rel_tol, o.abs_tol = int(kr.method), int(kr.ell), float(kr.rel_tol), float(kr.abs_tol)
        o.max_iterations, o.mixed_precision = int(kr.max_iterations), int(kr.mixed_precision)
        o.caller_asserts_spd, o.device = int(kr.caller_asserts_spd), int(device)
        o.triangle_solve = int(triangle_solve)  # 0 automatic, 1 chunk inverses, 2 substitution
        o.lu_kernel = int(lu_kernel)  # 0 automatic, 1 one CTA per job, 2 dataflow (bitwise-equal factors)
        o.tip_solve = int(tip_solve)  # SaP-C first block solve: 0 automatic (LU + UL tip sweeps), 1 full LU solve
        self.options = o
        self._h = C.c_void_p()
        self._create()
        self.n = 0
        self.k = 0
        self.p = int(p)
        self.layout: PartitionLayout | None = None

    def _create(self) -> None:
        _check(L.load().sap_create(C.byref(self.options), C.byref(self._h)))

    def close(self) -> None:
        if self._h:
            L.load().sap_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- helpers --------------------------------------------------------
    @staticmethod
    def _ptr(x):
        if _is_cuda_tensor(x):
            return C.c_void_p(x.data_ptr()), 1
        if not (isinstance(x, np.ndarray) and x.dtype == np.float64 and x.flags.c_contiguous):
            raise TypeError("expected a C-contiguous float64 numpy array or a CUDA tensor")
        return C.c_void_p(x.ctypes.data), 0

    def set_stream(self, stream) -> None:
        """Run on an external CUDA stream (torch.cuda.Stream or raw handle int)."""
        raw = getattr(stream, "cuda_stream", stream)
        _check(L.load().sap_set_stream(self._h, C.c_void_p(raw or None)))

    def synchronize(self) -> None:
        _check(L.load().sap_synchronize(self._h))

    # -- setup ≙ build_precond_op ---------------------------------------
    def setup(self, band, n: int, k: int) -> None:
        if not _is_cuda_tensor(band):
            band = np.ascontiguousarray(band, dtype=np.float64).reshape(-1)
        if int(band.numel() if _is_cuda_tensor(band) else band.size) != n * (2 * k + 1):
            raise ValueError("setup: band must hold n*(2k+1) entries")
        ptr, dev = self._ptr(band)
        self._arm_third_stage(n, k)
        _check(L.load().sap_setup_banded(self._h, n, k, ptr, dev))
        self.n, self.k = n, k
        if self.options.precond in (PrecondKind.coupled, PrecondKind.decoupled):
            self.layout = make_partition_layout(n, self.p, k)

    def setup_from_csr(self, row_ptr, col_idx, values, k: int) -> None:
        """assemble_banded (pipeline.hpp:103-115) on the device + setup; entries outside k raise ValueError."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        n = len(rp) - 1
        self._arm_third_stage(n, k)
        _check(L.load().sap_setup_banded_from_csr(self._h, n, k, len(ci), rp.ctypes.data, ci.ctypes.data,
                                                  v.ctypes.data, 0))
        self.n, self.k = n, k
        if self.options.precond in (PrecondKind.coupled, PrecondKind.decoupled):
            self.layout = make_partition_layout(n, self.p, k)

    def setup_from_csr_drop(self, row_ptr, col_idx, values, drop_tol: float) -> int:
        """drop_off (pipeline.hpp:59-99) + assemble_banded + setup on the device; returns k_after."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        n = len(rp) - 1
        ka = C.c_int()
        if getattr(self, "_ts", None):
            raise ValueError("setup_from_csr_drop: arm the third stage after the bandwidth is known "
                             "(use setup_from_csr with k_after)")
        _check(L.load().sap_setup_from_csr_drop(self._h, n, len(ci), rp.ctypes.data, ci.ctypes.data, v.ctypes.data,
                                                float(drop_tol), 0, C.byref(ka)))
        self.n, self.k = n, ka.value
        if self.options.precond in (PrecondKind.coupled, PrecondKind.decoupled):
            self.layout = make_partition_layout(n, self.p, self.k)
        return ka.value

    def set_third_stage(self, block_k, block_perms=None) -> None:
        """Arm the third stage (PipelineConfig::third_stage, pipeline.hpp:312-319) with
        sap::third_stage's result (ThirdStageResult, reorder_cm.hpp:227-231): block_k[p] per-partition
        half-bandwidths and block_perms[p] (an int array per block, or None / empty for identity).
        Applies to every following setup; ``set_third_stage(None)`` disarms."""
        if block_k is None:
            self._ts = None
            _check(L.load().sap_set_third_stage(self._h, 0, None, None, None, 0))
            return
        kb = np.ascontiguousarray(block_k, dtype=np.int32)
        perms = list(block_perms) if block_perms is not None else [None] * len(kb)
        if len(perms) != len(kb):
            raise ValueError("set_third_stage: one permutation (or None) per block")
        self._ts = (kb, perms)

    def _arm_third_stage(self, n: int, k: int) -> None:
        """Hand the armed third stage to the library; perm[n] is indexed by global row, so it is
        expanded over the partition layout the coming setup uses."""
        if not getattr(self, "_ts", None):
            return
        kb, perms = self._ts
        has = np.array([0 if q is None or len(q) == 0 else 1 for q in perms], np.int32)
        full = np.zeros(max(n, 1), np.int32)
        if has.any():
            lay = make_partition_layout(n, self.p, k)
            if lay.p != len(kb):
                raise ValueError("third stage: block count does not match the partition layout")
            for b, (q, h) in enumerate(zip(perms, has)):
                if h:
                    full[lay.offsets[b]:lay.offsets[b] + lay.sizes[b]] = np.asarray(q, np.int32)
        _check(L.load().sap_set_third_stage(self._h, len(kb), kb.ctypes.data, has.ctypes.data, full.ctypes.data, n))

    def full_spike(self, t: int):
        """(V_t, W_t) of the third stage (SpikeSet::v_full / w_full, spike.hpp:258-296): column-major
        sizes[t] x w_t and sizes[t+1] x w_t, returned as (m, w) numpy arrays."""
        kb = self._ts[0]
        w = int(max(kb[t], kb[t + 1]))
        mt, mn = self.layout.sizes[t], self.layout.sizes[t + 1]
        v = np.zeros(mt * w)
        wv = np.zeros(mn * w)
        _check(L.load().sap_get_full_spike(self._h, t, v.ctypes.data, wv.ctypes.data))
        return v.reshape(w, mt).T, wv.reshape(w, mn).T

    def set_operator_csr(self, row_ptr, col_idx, values) -> None:
        rp = np.ascontiguousarray(row_ptr, dtype=np.int32)
        ci = np.ascontiguousarray(col_idx, dtype=np.int32)
        v = np.ascontiguousarray(values, dtype=np.float64)
        _check(L.load().sap_set_operator_csr(self._h, len(rp) - 1, len(ci), rp.ctypes.data, ci.ctypes.data,
                                             v.ctypes.data, 0))

    # -- the two LinearOps ----------------------------------------------
    @staticmethod
    def _check_out(name, buf, like):
        """The library writes len(like) float64 values through buf's raw pointer: a caller-supplied
        output must be exactly that (the reference's std::span length check, spike.hpp:311-318)."""
        if _is_cuda_tensor(like):
            import torch
            ok = (_is_cuda_tensor(buf) and buf.dtype == torch.float64 and buf.is_contiguous()
                  and buf.numel() == like.numel() and buf.device == like.device)
        else:
            ok = (isinstance(buf, np.ndarray) and buf.dtype == np.float64 and buf.flags.c_contiguous
                  and buf.flags.writeable and buf.size == like.size)
        if not ok:
            raise ValueError(f"{name}: output must be a writable C-contiguous float64 buffer of length "
                             f"{like.numel() if _is_cuda_tensor(like) else like.size} on the input's device")

    def _op(self, fn, x, out):
        if _is_cuda_tensor(x):
            import torch
            if x.dtype != torch.float64 or not x.is_contiguous():
                raise ValueError("input must be a contiguous float64 tensor")
            if out is None:
                out = torch.empty_like(x)
            else:
                self._check_out("apply", out, x)
            _check(fn(self._h, C.c_void_p(x.data_ptr()), C.c_void_p(out.data_ptr()), 1))
            return out
        x = np.ascontiguousarray(x, dtype=np.float64)
        if out is None:
            out = np.empty_like(x)
        else:
            self._check_out("apply", out, x)
        _check(fn(self._h, x.ctypes.data, out.ctypes.data, 0))
        return out

    def apply_preconditioner(self, x, out=None):
        """out = M^{-1} x (apply_preconditioner, spike.hpp:304-351)."""
        return self._op(L.load().sap_apply_preconditioner, x, out)

    def matvec(self, x, out=None):
        """out = A x (BandedMatrix::matvec or the CSR operator)."""
        return self._op(L.load().sap_apply_operator, x, out)

    # -- solve ≙ run_krylov ---------------------------------------------
    def solve(self, b, x=None, history_capacity: int | None = None):
        cap = history_capacity if history_capacity is not None else 8 * max(self.options.max_iterations, 1) + 8
        hist = (C.c_double * cap)()
        st = L.sap_solve_stats()
        st.history = C.cast(hist, C.POINTER(C.c_double))
        st.history_capacity = cap
        if _is_cuda_tensor(b):
            import torch
            if b.dtype != torch.float64 or not b.is_contiguous():
                raise ValueError("solve: b must be a contiguous float64 tensor")
            if x is None:
                x = torch.empty_like(b)
            else:
                self._check_out("solve", x, b)
            _check(L.load().sap_solve(self._h, C.c_void_p(b.data_ptr()), C.c_void_p(x.data_ptr()), 1, C.byref(st)))
        else:
            b = np.ascontiguousarray(b, dtype=np.float64)
            if x is None:
                x = np.zeros_like(b)
            else:
                self._check_out("solve", x, b)
            _check(L.load().sap_solve(self._h, b.ctypes.data, x.ctypes.data, 0, C.byref(st)))
        stats = SolveStats(iterations=st.iterations, residual_history=list(hist[:min(st.history_len, cap)]),
                           converged=bool(st.converged), final_relative_residual=st.final_relative_residual,
                           failure=KrylovFailure(st.failure))
        return x, stats

    # -- reports and parity accessors -------------------------------------
    def report(self) -> dict:
        r = L.sap_report()
        _check(L.load().sap_get_report(self._h, C.byref(r)))
        return {f: getattr(r, f) for f, _ in L.sap_report._fields_}

    def factor(self, part: int, which: int = 0):
        """(band, boosts, block_norm) of block `part`; which 0 = LU, 1 = UL."""
        m = self.layout.sizes[part]
        ts = getattr(self, "_ts", None)
        out = np.zeros(m * (2 * (int(ts[0][part]) if ts else self.k) + 1))
        b = C.c_int()
        nrm = C.c_double()
        _check(L.load().sap_get_factor(self._h, part, which, out.ctypes.data, C.byref(b), C.byref(nrm)))
        return out, b.value, nrm.value

    def factors(self, which: int = 0):
        """All blocks concatenated (the reference's BlockFactors lu / ul vectors back to back)."""
        parts = [self.factor(i, which) for i in range(self.layout.p)]
        return (np.concatenate([q[0] for q in parts]), np.array([q[1] for q in parts], np.int32),
                np.array([q[2] for q in parts]))

    def spike(self, t: int) -> dict:
        ts = getattr(self, "_ts", None)
        w = int(max(ts[0][t], ts[0][t + 1])) if ts else self.k
        arrs = {q: np.zeros(w * w) for q in ("B", "C", "vb", "wt", "rbar")}
        rb = C.c_int()
        _check(L.load().sap_get_spike(self._h, t, arrs["B"].ctypes.data, arrs["C"].ctypes.data,
                                      arrs["vb"].ctypes.data, arrs["wt"].ctypes.data, arrs["rbar"].ctypes.data,
                                      C.byref(rb)))
        arrs["rbar_boosts"] = rb.value
        return arrs
