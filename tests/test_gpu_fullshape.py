"""Full-shape factor / spike parity at the BASELINE sizes (SURVEY §8c tolerances, d = 1):

* config 2 (N=200000, K=200, P=50): every block's LU and UL and every interface's B, C, V^b, W^t,
  R-bar against the oracle run on the whole system;
* config 5 (N=2000000, K=128, P=512): sampled blocks and interfaces (first, last, around the
  N mod P boundary where block sizes change) against the oracle run on the two-partition
  sub-system of each interface (a block's factors and an interface's tips depend only on the two
  diagonal blocks and their coupling corners, spike.hpp:95-254).
"""
import numpy as np
import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def nrel(a, b):
    den = np.max(np.abs(b))
    return np.max(np.abs(a - b)) / (den if den > 0 else 1.0)


def _check_interface(s, t, want, ti, k):
    got = s.spike(t)
    assert np.array_equal(got["B"], want["B"][ti * k * k:(ti + 1) * k * k]), t
    assert np.array_equal(got["C"], want["C"][ti * k * k:(ti + 1) * k * k]), t
    for q in ("vb", "wt", "rbar"):
        assert nrel(got[q], want[q][ti * k * k:(ti + 1) * k * k]) <= 1e-12, (t, q)
    assert got["rbar_boosts"] == want["rbar_boosts"][ti], t


def test_config2_all_blocks_and_interfaces(sap, oracle):
    n, k, p = 200000, 200, 50
    band, _ = sap.random_banded(n, k, 1.0, 1)
    s = sap.Solver(p=p, precond=sap.PrecondKind.coupled)
    s.setup(band, n, k)
    want = oracle.spikes(n, k, band, p)
    w = 2 * k + 1
    lay = s.layout
    for b in range(p):
        lo, hi = lay.offsets[b] * w, (lay.offsets[b] + lay.sizes[b]) * w
        lu, bl, nrm = s.factor(b, 0)
        ul, bu, _ = s.factor(b, 1)
        assert nrel(lu, want["lu"][lo:hi]) <= 1e-13, b
        assert nrel(ul, want["ul"][lo:hi]) <= 1e-13, b
        assert bl == want["boosts"][b] and bu == want["boosts_ul"][b] and nrm == want["norms"][b]
    for t in range(p - 1):
        _check_interface(s, t, want, t, k)
    s.close()


def _sub_system(band, n, k, lo, hi):
    """Rows [lo, hi) of the tall-thin band as a stand-alone system (entries reaching outside zeroed)."""
    w = 2 * k + 1
    sub = band[lo * w:hi * w].copy()
    m = hi - lo
    cols = np.repeat(np.arange(m), w)
    rows = cols - k + np.tile(np.arange(w), m)
    sub[(rows < 0) | (rows >= m)] = 0.0
    return sub


def test_config5_sampled_blocks_and_interfaces(sap, oracle):
    torch = pytest.importorskip("torch")
    n, k, p = 2000000, 128, 512
    band, _ = sap.random_banded(n, k, 1.0, 1)
    s = sap.Solver(p=p, precond=sap.PrecondKind.coupled)
    s.setup(torch.from_numpy(band).cuda(), n, k)
    lay = s.layout
    rem = n % p  # blocks [0, rem) have one row more (partition.hpp:42-69)
    w = 2 * k + 1
    for t in sorted({0, 1, rem - 2, rem - 1, rem, 300, p - 2}):
        lo = lay.offsets[t]
        hi = lay.offsets[t + 2]
        m0 = lay.sizes[t]
        want = oracle.spikes(hi - lo, k, _sub_system(band, n, k, lo, hi), 2)
        for j, b in enumerate((t, t + 1)):
            seg = slice(0, m0 * w) if j == 0 else slice(m0 * w, (hi - lo) * w)
            lu, bl, _ = s.factor(b, 0)
            ul, bu, _ = s.factor(b, 1)
            assert nrel(lu, want["lu"][seg]) <= 1e-13, b
            assert nrel(ul, want["ul"][seg]) <= 1e-13, b
            assert bl == want["boosts"][j] and bu == want["boosts_ul"][j]
        _check_interface(s, t, want, 0, k)
    s.close()
