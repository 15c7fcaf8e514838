"""The two band LU implementations (sap_options::lu_kernel: 1 = one CTA per job; 2 = the dataflow kernel
k_band_lu_df) give BITWISE equal factors, boost counts and reduced blocks where the one-CTA
kernel is k_band_lu_res (the dataflow kernel performs every element's operations in the same order), across the
shapes the dispatch can route either way: odd K, unequal blocks, a host band (streamed upload), low dominance,
and K = 300 beyond it. At K = 224 k_band_lu_res does not fit shared memory and the one-CTA kernel is the staged
k_band_lu_seq, whose panel multiplies by a reciprocal (l = a (1/p)): there the two agree within the SURVEY 8c
factor tolerance (1e-13 normwise), boost counts equal. The automatic choice (0) equals one of them."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

BITWISE = {0, 1, 2, 3, 5}
CASES = [  # n, k, d, p, coupled, host band
    (3000, 64, 1.0, 3, True, False),
    (20011, 77, 1.0, 7, True, False),
    (20000, 100, 0.5, 5, True, True),
    (40000, 200, 0.06, 10, True, False),
    (40000, 224, 1.0, 8, False, True),
    (40000, 300, 1.0, 8, True, False),
]


def _factors(sap, case, lu_kernel):
    import torch
    n, k, d, p, coupled, host = case
    band, rhs = sap.random_banded(n, k, d, 7)
    kind = sap.PrecondKind.coupled if coupled else sap.PrecondKind.decoupled
    with sap.Solver(p=p, precond=kind, lu_kernel=lu_kernel) as s:
        s.setup(band if host else torch.from_numpy(band).cuda(), n, k)
        out = {"lu": s.factors(0)}
        if coupled:
            out["ul"] = s.factors(1)
            sp = [s.spike(t) for t in range(p - 1)]
            out["rbar"] = np.concatenate([x["rbar"] for x in sp])
            out["rbar_boosts"] = [x["rbar_boosts"] for x in sp]
        x, st = s.solve(rhs)
        out["it"] = st.iterations
    return out


@pytest.mark.parametrize("ci", range(len(CASES)))
def test_dataflow_lu_is_bitwise_the_single_cta_lu(sap, ci):
    case = CASES[ci]
    a, b, c = (_factors(sap, case, lk) for lk in (1, 2, 0))
    if ci not in BITWISE:
        for key in ("lu", "ul"):
            if key in a:
                den = np.max(np.abs(a[key][0]))
                assert np.max(np.abs(a[key][0] - b[key][0])) <= 1e-13 * den and np.array_equal(a[key][1], b[key][1])
        assert abs(a["it"] - b["it"]) <= 1.0
        a = b  # the automatic choice is the dataflow kernel here
    for key in a:
        for other in ((b, c) if ci in BITWISE else (c,)):
            if key in ("lu", "ul"):
                assert np.array_equal(a[key][0], other[key][0]) and np.array_equal(a[key][1], other[key][1]), key
            elif key == "rbar":
                assert np.array_equal(a[key], other[key])
            else:
                assert a[key] == other[key], key


SCHEDULES = [  # (job owners, strips per worker item): the dataflow kernel's schedule knobs (lu.cu DfArgs)
    (0, 3), (1, 1), (1, 2), (1, 3), (0, 1),
]


@pytest.mark.parametrize("case", [(40000, 200, 1.0, 10, True, False), (40000, 224, 0.5, 8, False, True),
                                  (30000, 300, 1.0, 5, True, False)])
def test_dataflow_schedules_are_bitwise_equal(sap, case):
    """The dataflow kernel's work split (chain items on job-owner CTAs or the shared queue; 1-3 strips per worker
    item) changes only who computes what and when, never an element's operations: factors, boosts and reduced
    blocks are bitwise the same for every schedule."""
    from paper_1509_07919_b200 import _lib
    lib = _lib.load()
    ref = None
    try:
        for owners, grp in SCHEDULES:
            lib.sap_dev_lu_df_owners(owners)
            lib.sap_dev_lu_df_group(grp)
            out = _factors(sap, case, 2)
            if ref is None:
                ref = out
                continue
            for key in ref:
                if key in ("lu", "ul"):
                    assert np.array_equal(ref[key][0], out[key][0]) and np.array_equal(ref[key][1], out[key][1]), key
                elif key == "rbar":
                    assert np.array_equal(ref[key], out[key])
                else:
                    assert ref[key] == out[key], key
    finally:
        lib.sap_dev_lu_df_owners(1)
        lib.sap_dev_lu_df_group(0)
