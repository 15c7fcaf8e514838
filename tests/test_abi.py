"""CPU-side checks of the C ABI library (no device work):

* libsap_gpu.so loads and exports every function include/sap_gpu.h declares;
* host logic mirrors the reference: options defaults (pipeline.hpp:21-32,
  krylov.hpp:20-28), make_partition_layout / max_feasible_partitions
  (partition.hpp:34-69, messages included), and the synthetic generator
  (testsup::random_banded) bit for bit against the oracle.
"""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "sap_gpu.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sap_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(sap):
    lib = sap.load()
    names = _declared()
    assert len(names) >= 19
    for name in names:
        assert hasattr(lib, name), name
    from paper_1509_07919_b200._lib import SIGNATURES
    assert sorted(SIGNATURES) == names


def test_library_is_sm100a(sap):
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", sap.LIB_PATH], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "-sass", sap.LIB_PATH], capture_output=True,
                          text=True).stdout
    assert "DMMA" in sass  # FP64 tensor-core trailing updates are present


def test_options_defaults_match_reference(sap):
    import ctypes as C
    from paper_1509_07919_b200 import _lib as L
    o = L.sap_options()
    sap.load().sap_options_default(C.byref(o))
    assert (o.p, o.precond, o.boost_eps, o.method, o.ell) == (1, 0, 1e-10, 0, 2)
    assert (o.rel_tol, o.abs_tol, o.max_iterations, o.mixed_precision, o.caller_asserts_spd) == (1e-10, 0.0, 500, 0, 0)
    assert (o.triangle_solve, o.lu_kernel, o.tip_solve) == (0, 0, 0)  # implementation choices, automatic by default


def test_partition_layout_matches_reference(sap, oracle):
    lay = sap.make_partition_layout(10, 3, 1)
    assert lay.sizes == [4, 3, 3] and lay.offsets == [0, 4, 7, 10] and lay.remainder == 1 and lay.total() == 10
    assert sap.make_partition_layout(12, 4, 1).sizes == [3, 3, 3, 3]
    assert sap.make_partition_layout(7, 1, 3).per_partition_k == [3]
    with pytest.raises(ValueError, match="largest feasible p is 2"):
        sap.make_partition_layout(10, 3, 2)
    with pytest.raises(ValueError, match="empty matrix"):
        sap.make_partition_layout(0, 1, 1)
    with pytest.raises(ValueError, match="partition count must be positive"):
        sap.make_partition_layout(5, 0, 1)
    with pytest.raises(ValueError, match="negative bandwidth"):
        sap.make_partition_layout(5, 1, -1)
    assert [sap.max_feasible_partitions(*a) for a in [(10, 2), (10, 0), (7, 3), (12, 3), (5, 3)]] == [2, 10, 1, 2, 0]
    for n, p, k in [(200000, 50, 200), (2000000, 512, 128), (10001, 7, 10), (37, 37, 0)]:
        s, o = oracle.partition_layout(n, p, k)
        lay = sap.make_partition_layout(n, p, k)
        assert lay.sizes == list(s) and lay.offsets == list(o)


def test_generator_matches_oracle_and_reference(sap, oracle):
    for (n, k, d, seed) in [(300, 7, 0.1, 2), (1000, 20, 1.0, 1), (64, 0, 1.3, 9)]:
        b1, r1 = sap.random_banded(n, k, d, seed)
        b2, r2 = oracle.random_banded(n, k, d, seed)
        assert np.array_equal(b1, b2) and np.array_equal(r1, r2)


def test_errors_map_to_reference_exceptions(sap):
    import ctypes as C
    lib = sap.load()
    rc = lib.sap_partition_layout(10, 3, 2, None, None)
    assert rc == 1 and b"largest feasible p is 2" in lib.sap_last_error()
    assert lib.sap_status_string(2) == b"preconditioner error"
    assert lib.sap_create(None, None) == 1  # null output -> invalid argument, not a crash
