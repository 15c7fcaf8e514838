"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU oracle.

Two libraries live here, both checkers, never the product:

* ``libsap_oracle.so`` — the plain-C restatement of the reference algorithm
  (``oracle/sap_oracle.c``; each function cites the reference file:line it
  follows).
* ``_ref/libsapref.so`` — the unmodified reference headers compiled in place
  (``oracle/ref_shim.cpp``, ``oracle/Makefile``). Present in the build
  container and shipped prebuilt to the GPU box; ``has_ref()`` says whether it
  is loadable.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline /
reference legs may import this package.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
_ORACLE = os.path.join(HERE, "libsap_oracle.so")
_REF = os.path.join(HERE, "_ref", os.environ.get("SAP_REF_LIB", "libsapref.so"))  # tools may pick libsapref_fma.so

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"oracle error {code}: {msg}")
        self.code = code


def build() -> None:
    """Compile the C restatement (and the reference shim where the sources exist)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Stats(C.Structure):
    _fields_ = [("iterations", C.c_double), ("converged", C.c_int), ("final_relative_residual", C.c_double),
                ("failure", C.c_int), ("hist_len", C.c_int)]


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_ORACLE):
            build()
        L = C.CDLL(_ORACLE)
        L.sapo_random_banded.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint32, _dp, C.c_void_p]
        L.sapo_uniform_stream.argtypes = [C.c_uint32, C.c_int, _dp]
        L.sapo_partition_layout.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip]
        L.sapo_max_feasible_partitions.argtypes = [C.c_int, C.c_int]
        L.sapo_band_matvec.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
        L.sapo_csr_matvec.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp]
        L.sapo_band_lu_inplace.argtypes = [C.c_int, C.c_int, _dp, C.c_double, C.c_double]
        L.sapo_band_ul_inplace.argtypes = [C.c_int, C.c_int, _dp, C.c_double, C.c_double]
        L.sapo_band_lu_solve.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.sapo_band_ul_solve.argtypes = [C.c_int, C.c_int, _dp, _dp]
        L.sapo_factor_blocks.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, C.c_void_p,
                                         _ip, C.c_void_p, C.c_void_p]
        L.sapo_dense_lu_nopivot_boosted.argtypes = [C.c_int, _dp, C.c_double]
        L.sapo_dense_lu_solve.argtypes = [C.c_int, _dp, _dp]
        L.sapo_extract_coupling.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip, _dp, _dp]
        L.sapo_spike_tips.argtypes = [C.c_int, C.c_int, _ip, _ip, _dp, _dp, _dp, _dp, C.c_double, _dp, _dp, _dp,
                                      _ip]
        L.sapo_apply.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, _dp]
        L.sapo_solve_banded.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_int,
                                        C.c_double, C.c_double, C.c_int, _dp, C.POINTER(_Stats), _dp, C.c_int]
        L.sapo_krylov_csr_identity.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp,
                                               C.POINTER(_Stats), _dp, C.c_int]
        _lib = L
    return _lib


def has_ref() -> bool:
    try:
        ref()
        return True
    except OSError:
        return False


def ref():
    global _ref
    if _ref is None:
        R = C.CDLL(_REF)
        R.sapref_last_error.restype = C.c_char_p
        R.sapref_random_banded.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, _dp, C.c_void_p]
        R.sapref_partition_layout.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip]
        R.sapref_band_matvec.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp]
        R.sapref_factor_blocks.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, C.c_void_p,
                                           _ip, C.c_void_p, C.c_void_p]
        R.sapref_spikes.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_double, _dp, _dp, _dp, _dp, _dp, _ip]
        R.sapref_factor_blocks_f32.argtypes = R.sapref_factor_blocks.argtypes
        R.sapref_spikes_f32.argtypes = R.sapref_spikes.argtypes
        R.sapref_apply_f32.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, _dp]
        R.sapref_apply.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_int, C.c_double, _dp, _dp]
        R.sapref_solve_banded.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, C.c_int, C.c_double, C.c_int,
                                          C.c_double, C.c_double, C.c_int, C.c_int, _dp,
                                          C.POINTER(C.c_double), C.POINTER(C.c_int), C.POINTER(C.c_double),
                                          C.POINTER(C.c_int), _dp, C.c_int, C.POINTER(C.c_int), _dp]
        R.sapref_krylov_csr_identity.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_int, C.c_double, C.c_int, _dp,
                                                 C.POINTER(C.c_double), C.POINTER(C.c_int),
                                                 C.POINTER(C.c_double), C.POINTER(C.c_int), _dp, C.c_int,
                                                 C.POINTER(C.c_int)]
        R.sapref_solve_sparse.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_double, C.c_int, C.c_double, C.c_uint, C.c_int, C.c_double, C.c_int,
                                          C.c_int, _dp, _dp, C.POINTER(C.c_double), C.POINTER(C.c_int),
                                          C.POINTER(C.c_double), C.POINTER(C.c_int)]
        R.sapref_host_stage.argtypes = [C.c_int, _ip, _ip, _dp, _dp, C.c_int, C.c_int, C.c_int, C.c_uint, _ip, _ip,
                                        _dp, _dp, _ip, _dp, _dp]
        _ref = R
    return _ref


def _ref_check(rc: int) -> None:
    if rc:
        raise OracleError(rc, ref().sapref_last_error().decode())


# ---------------------------------------------------------------------------
# C restatement (the checker)

def random_banded(n: int, k: int, d: float, seed: int, with_rhs: bool = True):
    band = np.zeros(n * (2 * k + 1))
    rhs = np.zeros(n) if with_rhs else None
    lib().sapo_random_banded(n, k, d, seed, band, rhs.ctypes.data if with_rhs else None)
    return (band, rhs) if with_rhs else band


def uniform_stream(seed: int, count: int) -> np.ndarray:
    out = np.zeros(count)
    lib().sapo_uniform_stream(seed, count, out)
    return out


def partition_layout(n: int, p: int, k: int):
    sizes = np.zeros(max(p, 1), np.int32)
    offs = np.zeros(max(p, 1) + 1, np.int32)
    if lib().sapo_partition_layout(n, p, k, sizes, offs):
        raise OracleError(1, "make_partition_layout: infeasible")
    return sizes, offs


def band_matvec(n, k, band, x):
    y = np.zeros(n)
    lib().sapo_band_matvec(n, k, band, np.ascontiguousarray(x, np.float64), y)
    return y


def csr_matvec(n, rp, ci, v, x):
    y = np.zeros(n)
    lib().sapo_csr_matvec(n, rp, ci, v, np.ascontiguousarray(x, np.float64), y)
    return y


def factor_blocks(n, k, band, p, lu_and_ul, boost_eps=1e-10):
    lu = np.zeros(n * (2 * k + 1))
    ul = np.zeros(n * (2 * k + 1)) if lu_and_ul else None
    boosts = np.zeros(p, np.int32)
    bul = np.zeros(p, np.int32)
    norms = np.zeros(p)
    rc = lib().sapo_factor_blocks(n, k, band, p, int(lu_and_ul), boost_eps, lu,
                                  ul.ctypes.data if lu_and_ul else None, boosts, bul.ctypes.data,
                                  norms.ctypes.data)
    if rc:
        raise OracleError(rc, "factor_blocks")
    return dict(lu=lu, ul=ul, boosts=boosts, boosts_ul=bul, norms=norms)


def spikes(n, k, band, p, boost_eps=1e-10):
    """extract_coupling + compute_spike_tips (+ rbar) on the oracle's own factors."""
    f = factor_blocks(n, k, band, p, True, boost_eps)
    sizes, offs = partition_layout(n, p, k)
    ww = max(p - 1, 0) * k * k
    B, Cb, vb, wt, rb = (np.zeros(max(ww, 1)) for _ in range(5))
    rbo = np.zeros(max(p - 1, 1), np.int32)
    lib().sapo_extract_coupling(n, k, band, p, offs, B, Cb)
    rc = lib().sapo_spike_tips(k, p, sizes, offs, f["lu"], f["ul"], B, Cb, boost_eps, vb, wt, rb, rbo)
    if rc:
        raise OracleError(rc, "spike tips not finite")
    cut = slice(0, ww)
    return dict(B=B[cut], C=Cb[cut], vb=vb[cut], wt=wt[cut], rbar=rb[cut], rbar_boosts=rbo[:max(p - 1, 0)],
                **f)


def apply(n, k, band, p, kind, x, boost_eps=1e-10):
    out = np.zeros(n)
    rc = lib().sapo_apply(n, k, band, p, kind, boost_eps, np.ascontiguousarray(x, np.float64), out)
    if rc:
        raise OracleError(rc, "apply")
    return out


def solve_banded(n, k, band, rhs, p, kind, boost_eps=1e-10, ell=2, rel_tol=1e-10, abs_tol=0.0, max_iterations=500):
    x = np.zeros(n)
    st = _Stats()
    cap = 4 * 2 * max(max_iterations, 1) + 8
    hist = np.zeros(cap)
    rc = lib().sapo_solve_banded(n, k, band, rhs, p, kind, boost_eps, ell, rel_tol, abs_tol, max_iterations, x,
                                 C.byref(st), hist, cap)
    if rc:
        raise OracleError(rc, "solve_banded")
    return x, dict(iterations=st.iterations, converged=bool(st.converged),
                   final_relative_residual=st.final_relative_residual, failure=st.failure,
                   residual_history=hist[:min(st.hist_len, cap)].copy())


# ---------------------------------------------------------------------------
# The compiled reference (oracle/_ref)

def ref_random_banded(n, k, d, seed):
    band = np.zeros(n * (2 * k + 1))
    rhs = np.zeros(n)
    _ref_check(ref().sapref_random_banded(n, k, d, seed, band, rhs.ctypes.data))
    return band, rhs


def ref_factor_blocks(n, k, band, p, lu_and_ul, boost_eps=1e-10):
    lu = np.zeros(n * (2 * k + 1))
    ul = np.zeros(n * (2 * k + 1))
    boosts = np.zeros(p, np.int32)
    bul = np.zeros(p, np.int32)
    norms = np.zeros(p)
    _ref_check(ref().sapref_factor_blocks(n, k, band, p, int(lu_and_ul), boost_eps, lu, ul.ctypes.data, boosts,
                                          bul.ctypes.data, norms.ctypes.data))
    return dict(lu=lu, ul=ul if lu_and_ul else None, boosts=boosts, boosts_ul=bul, norms=norms)


def ref_spikes(n, k, band, p, boost_eps=1e-10):
    ww = max(p - 1, 0) * k * k
    B, Cb, vb, wt, rb = (np.zeros(max(ww, 1)) for _ in range(5))
    rbo = np.zeros(max(p - 1, 1), np.int32)
    _ref_check(ref().sapref_spikes(n, k, band, p, boost_eps, B, Cb, vb, wt, rb, rbo))
    cut = slice(0, ww)
    return dict(B=B[cut], C=Cb[cut], vb=vb[cut], wt=wt[cut], rbar=rb[cut], rbar_boosts=rbo[:max(p - 1, 0)])


def ref_apply(n, k, band, p, kind, x, boost_eps=1e-10):
    out = np.zeros(n)
    _ref_check(ref().sapref_apply(n, k, band, p, kind, boost_eps, np.ascontiguousarray(x, np.float64), out))
    return out


def ref_factor_blocks_f32(n, k, band, p, lu_and_ul, boost_eps=1e-10):
    """factor_blocks<float> on banded_cast<float>(band) (build_precond_op<float>), widened to double."""
    lu = np.zeros(n * (2 * k + 1))
    ul = np.zeros(n * (2 * k + 1))
    boosts = np.zeros(p, np.int32)
    bul = np.zeros(p, np.int32)
    norms = np.zeros(p)
    _ref_check(ref().sapref_factor_blocks_f32(n, k, band, p, int(lu_and_ul), boost_eps, lu, ul.ctypes.data, boosts,
                                              bul.ctypes.data, norms.ctypes.data))
    return dict(lu=lu, ul=ul if lu_and_ul else None, boosts=boosts, boosts_ul=bul, norms=norms)


def ref_spikes_f32(n, k, band, p, boost_eps=1e-10):
    ww = max(p - 1, 0) * k * k
    B, Cb, vb, wt, rb = (np.zeros(max(ww, 1)) for _ in range(5))
    rbo = np.zeros(max(p - 1, 1), np.int32)
    _ref_check(ref().sapref_spikes_f32(n, k, band, p, boost_eps, B, Cb, vb, wt, rb, rbo))
    cut = slice(0, ww)
    return dict(B=B[cut], C=Cb[cut], vb=vb[cut], wt=wt[cut], rbar=rb[cut], rbar_boosts=rbo[:max(p - 1, 0)])


def ref_apply_f32(n, k, band, p, kind, x, boost_eps=1e-10):
    out = np.zeros(n)
    _ref_check(ref().sapref_apply_f32(n, k, band, p, kind, boost_eps, np.ascontiguousarray(x, np.float64), out))
    return out


def ref_solve_banded(n, k, band, rhs, p, kind, boost_eps=1e-10, ell=2, rel_tol=1e-10, abs_tol=0.0,
                     max_iterations=500, mixed_precision=False):
    x = np.zeros(n)
    it, conv, res, fail, hl = C.c_double(), C.c_int(), C.c_double(), C.c_int(), C.c_int()
    cap = 4 * 2 * max(max_iterations, 1) + 8
    hist = np.zeros(cap)
    tim = np.zeros(5)
    _ref_check(ref().sapref_solve_banded(n, k, band, rhs, p, kind, boost_eps, ell, rel_tol, abs_tol,
                                         max_iterations, int(mixed_precision), x, C.byref(it), C.byref(conv),
                                         C.byref(res), C.byref(fail), hist, cap, C.byref(hl), tim))
    return x, dict(iterations=it.value, converged=bool(conv.value), final_relative_residual=res.value,
                   failure=fail.value, residual_history=hist[:min(hl.value, cap)].copy(),
                   t_lu=tim[0], t_bc=tim[1], t_spk=tim[2], t_lurdcd=tim[3], t_kry=tim[4])


def ref_host_stage(n, row_ptr, col_idx, vals, rhs, use_db=True, db_scaling=True, use_cm=True, seed=0):
    """solve_sparse's host stage (pipeline.hpp:228-266) run by the compiled reference: db_reorder + scaling,
    cm_reorder. Returns the reordered CSR (rp, ci, v), rhs, the CM permutation and column scaling that map
    the solution back (x[i] = z[cm_perm[i]] * col_scale[i]), and (t_db, t_cm) in seconds."""
    nnz = int(row_ptr[n])
    rp, ci, v = np.zeros(n + 1, np.int32), np.zeros(nnz, np.int32), np.zeros(nnz)
    r, perm, cs, tim = np.zeros(n), np.zeros(n, np.int32), np.zeros(n), np.zeros(2)
    _ref_check(ref().sapref_host_stage(n, np.ascontiguousarray(row_ptr, np.int32),
                                       np.ascontiguousarray(col_idx, np.int32), np.ascontiguousarray(vals, np.float64),
                                       np.ascontiguousarray(rhs, np.float64), int(use_db), int(db_scaling),
                                       int(use_cm), seed, rp, ci, v, r, perm, cs, tim))
    return dict(rp=rp, ci=ci, v=v, rhs=r, cm_perm=perm, col_scale=cs, t_db=tim[0], t_cm=tim[1])


def convection_diffusion_3d(s):
    """3-D 7-point upwind convection-diffusion on an s^3 grid (natural order), diagonal
    6.3, -1.3 on the x-1 / y-1 / z-1 neighbours, -0.7 on +1 (a builder-defined 3-D analog of
    proj/tests/acceptance.cpp:442-454). Returns n, row_ptr, col_idx, values (CSR, ascending columns)."""
    n = s ** 3
    idx = np.arange(n, dtype=np.int64)
    z, y, x = idx // (s * s), (idx // s) % s, idx % s
    cols, vals = [], []
    for off, cond, val in ((-s * s, z > 0, -1.3), (-s, y > 0, -1.3), (-1, x > 0, -1.3), (0, None, 6.3),
                           (1, x < s - 1, -0.7), (s, y < s - 1, -0.7), (s * s, z < s - 1, -0.7)):
        m = np.ones(n, bool) if cond is None else cond
        c = np.where(m, idx + off, -1)
        cols.append(c)
        vals.append(np.where(m, val, 0.0))
    C_ = np.stack(cols, 1)
    V_ = np.stack(vals, 1)
    keep = C_ >= 0
    rp = np.concatenate([[0], np.cumsum(keep.sum(1))]).astype(np.int32)
    return n, rp, C_[keep].astype(np.int32), V_[keep].astype(np.float64)


def manufactured_solution(n):
    """benchmark.hpp:23-34: x_j = 1 + 399 (1 - t^2), t = 2 j / (n - 1) - 1."""
    if n == 1:
        return np.array([400.0])
    t = 2.0 * np.arange(n) / (n - 1) - 1.0
    return 1.0 + 399.0 * (1.0 - t * t)


def ref_solve_sparse(n, row_ptr, col_idx, vals, rhs, p, kind, use_db=False, db_scaling=True, use_cm=False,
                     third_stage=False, drop_tol=0.0, boost_eps=1e-10, seed=0, ell=2, rel_tol=1e-10,
                     max_iterations=500, mixed_precision=False):
    """The reference's solve_sparse (pipeline.hpp:213-369) end to end; report = t_db, t_cm, t_drop, t_asmbl,
    t_bc, t_lu, t_spk, t_lurdcd, t_kry, k (after drop-off)."""
    x = np.zeros(n)
    rep = np.zeros(10)
    it, conv, res, fail = C.c_double(), C.c_int(), C.c_double(), C.c_int()
    _ref_check(ref().sapref_solve_sparse(n, np.ascontiguousarray(row_ptr, np.int32),
                                         np.ascontiguousarray(col_idx, np.int32),
                                         np.ascontiguousarray(vals, np.float64), np.ascontiguousarray(rhs, np.float64),
                                         int(use_db), int(db_scaling), int(use_cm), int(third_stage), p, drop_tol,
                                         kind, boost_eps, seed, ell, rel_tol, max_iterations, int(mixed_precision),
                                         x, rep, C.byref(it), C.byref(conv), C.byref(res), C.byref(fail)))
    return x, dict(iterations=it.value, converged=bool(conv.value), final_relative_residual=res.value,
                   failure=fail.value, k_after=int(rep[9]), report=rep)


# ---------------------------------------------------------------------------
# Third stage (per-block reordering) through the compiled reference. The C restatement does not
# cover it: these wrappers ARE the checker for the third-stage path (the reference's own
# third_stage / factor_blocks(perms) / compute_full_spikes / apply / build_precond_op code).

def _ts_args(p, block_k, has_perm, perm, n):
    kb = np.ascontiguousarray(block_k, np.int32)
    hp = np.ascontiguousarray(has_perm if has_perm is not None else np.zeros(p), np.int32)
    pm = np.ascontiguousarray(perm if perm is not None else np.zeros(max(n, 1)), np.int32)
    return kb, hp, pm


def ref_third_stage(n, k, band, p, seed=0):
    """sap::third_stage (reorder_cm.hpp:233-274): (block_k[p], has_perm[p], perm[n])."""
    kb = np.zeros(p, np.int32)
    hp = np.zeros(p, np.int32)
    pm = np.zeros(max(n, 1), np.int32)
    R = ref()
    R.sapref_third_stage.argtypes = [C.c_int, C.c_int, _dp, C.c_int, C.c_uint, _ip, _ip, _ip]
    _ref_check(R.sapref_third_stage(n, k, band, p, seed, kb, hp, pm))
    return kb, hp, pm[:n]


def ref_third_setup(n, k, band, p, block_k, has_perm, perm, coupled=True, boost_eps=1e-10):
    """factor_blocks(perms, K_b) + extract_coupling + compute_full_spikes; per-block / per-interface lists."""
    kb, hp, pm = _ts_args(p, block_k, has_perm, perm, n)
    sizes, offsets = partition_layout(n, p, k)
    lu = np.zeros(sum(int(sizes[b]) * (2 * int(kb[b]) + 1) for b in range(p)))
    boosts = np.zeros(p, np.int32)
    norms = np.zeros(p)
    wid = [int(max(kb[t], kb[t + 1])) for t in range(p - 1)]
    ww = max(sum(w * w for w in wid), 1)
    B, Cb, vb, wt, rb = (np.zeros(ww) for _ in range(5))
    rbo = np.zeros(max(p - 1, 1), np.int32)
    vf = np.zeros(max(sum(int(sizes[t]) * wid[t] for t in range(p - 1)), 1))
    wf = np.zeros(max(sum(int(sizes[t + 1]) * wid[t] for t in range(p - 1)), 1))
    R = ref()
    R.sapref_third_setup.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip, _ip, _ip, C.c_double, C.c_int, _dp, _ip,
                                     _dp, _dp, _dp, _dp, _dp, _dp, _ip, _dp, _dp]
    _ref_check(R.sapref_third_setup(n, k, band, p, kb, hp, pm, boost_eps, int(coupled), lu, boosts, norms, B, Cb, vb,
                                    wt, rb, rbo, vf, wf))
    out = dict(lu=[], boosts=boosts, norms=norms, B=[], C=[], vb=[], wt=[], rbar=[], rbar_boosts=rbo[:p - 1],
               v_full=[], w_full=[], widths=wid)
    o = 0
    for b in range(p):
        ln = int(sizes[b]) * (2 * int(kb[b]) + 1)
        out["lu"].append(lu[o:o + ln])
        o += ln
    o = ov = ow = 0
    for t, w in enumerate(wid):
        for key, arr in (("B", B), ("C", Cb), ("vb", vb), ("wt", wt), ("rbar", rb)):
            out[key].append(arr[o:o + w * w].reshape(w, w))
        o += w * w
        mt, mn = int(sizes[t]), int(sizes[t + 1])
        out["v_full"].append(vf[ov:ov + mt * w].reshape(w, mt).T)
        out["w_full"].append(wf[ow:ow + mn * w].reshape(w, mn).T)
        ov += mt * w
        ow += mn * w
    return out


def ref_third_apply(n, k, band, p, block_k, has_perm, perm, kind, x, boost_eps=1e-10):
    kb, hp, pm = _ts_args(p, block_k, has_perm, perm, n)
    out = np.zeros(n)
    R = ref()
    R.sapref_third_apply.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip, _ip, _ip, C.c_int, C.c_double, _dp, _dp]
    _ref_check(R.sapref_third_apply(n, k, band, p, kb, hp, pm, kind, boost_eps, np.ascontiguousarray(x, np.float64),
                                    out))
    return out


def ref_third_solve_banded(n, k, band, rhs, p, block_k, has_perm, perm, kind, boost_eps=1e-10, ell=2,
                           rel_tol=1e-10, max_iterations=500, mixed_precision=False):
    kb, hp, pm = _ts_args(p, block_k, has_perm, perm, n)
    x = np.zeros(n)
    it, conv, res, fail = C.c_double(), C.c_int(), C.c_double(), C.c_int()
    R = ref()
    R.sapref_third_solve_banded.argtypes = [C.c_int, C.c_int, _dp, _dp, C.c_int, _ip, _ip, _ip, C.c_int, C.c_double,
                                            C.c_int, C.c_double, C.c_int, C.c_int, _dp, C.POINTER(C.c_double),
                                            C.POINTER(C.c_int), C.POINTER(C.c_double), C.POINTER(C.c_int)]
    _ref_check(R.sapref_third_solve_banded(n, k, band, np.ascontiguousarray(rhs, np.float64), p, kb, hp, pm, kind,
                                           boost_eps, ell, rel_tol, max_iterations, int(mixed_precision), x,
                                           C.byref(it), C.byref(conv), C.byref(res), C.byref(fail)))
    return x, dict(iterations=it.value, converged=bool(conv.value), final_relative_residual=res.value,
                   failure=fail.value)


def scrambled_banded(n, kn, window, k, d, seed):
    """Test input for the third stage: a random diagonally dominant band of half-bandwidth kn,
    symmetrically permuted by reversing every `window` consecutive indices (bandwidth grows to at most
    2*window - 1 + kn <= k), stored at half-bandwidth k. Cuthill-McKee recovers a narrow band per block."""
    rng = np.random.default_rng(seed)
    pos = np.arange(n)
    w0 = (pos // window) * window
    perm = np.minimum(w0 + window - 1, n - 1) - (pos - w0)  # new index of old index i
    if n % window:  # tail window reversed within its own length
        t0 = (n // window) * window
        perm[t0:] = n - 1 - (pos[t0:] - t0)
    band = np.zeros(n * (2 * k + 1))
    rows, cols, vals = [], [], []
    for i in range(n):
        off = 0.0
        for j in range(max(0, i - kn), min(n, i + kn + 1)):
            if j == i:
                continue
            v = rng.uniform(-1, 1) or 0.5
            rows.append(i); cols.append(j); vals.append(v)
            off += abs(v)
        rows.append(i); cols.append(i); vals.append(d * off)
    for i, j, v in zip(rows, cols, vals):
        pi, pj = int(perm[i]), int(perm[j])
        assert abs(pi - pj) <= k
        band[pj * (2 * k + 1) + (pi - pj + k)] = v
    return band


def ref_drop_off(n, row_ptr, col_idx, vals, tol):
    """sap::drop_off (pipeline.hpp:59-99) through the compiled reference: (k_after, nnz kept)."""
    R = ref()
    R.sapref_drop_off.argtypes = [C.c_int, _ip, _ip, _dp, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_int)]
    ka, nk = C.c_int(), C.c_int()
    _ref_check(R.sapref_drop_off(n, np.ascontiguousarray(row_ptr, np.int32), np.ascontiguousarray(col_idx, np.int32),
                                 np.ascontiguousarray(vals, np.float64), tol, C.byref(ka), C.byref(nk)))
    return ka.value, nk.value
