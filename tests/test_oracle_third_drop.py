"""CPU checks of the third-stage / drop-off checker (the compiled reference behind oracle.ref_third_* and
oracle.ref_drop_off) and of the scrambled test input: no GPU, a few seconds."""
import numpy as np
import pytest


@pytest.fixture(scope="module")
def ref(oracle):
    if not oracle.has_ref():
        pytest.skip("compiled reference absent")
    return oracle


def test_scrambled_band_is_narrowed_by_third_stage(ref):
    n, k, p = 2000, 20, 2
    band = ref.scrambled_banded(n, 2, 8, k, 1.0, 1)
    kb, hp, pm = ref.ref_third_stage(n, k, band, p, 0)
    assert hp.all() and (kb == 2).all()
    sizes, offs = ref.partition_layout(n, p, k)
    for b in range(p):  # every block permutation is a permutation
        assert np.array_equal(np.sort(pm[offs[b]:offs[b] + sizes[b]]), np.arange(sizes[b]))


def test_third_stage_identity_equals_plain_factors(ref):
    """Identity permutations at K_b = k: factor_blocks with block_perms equals the plain LU (the
    reference's own code paths agree), and the full spikes' ends are the truncated tips."""
    n, k, p = 1200, 6, 3
    band, _ = ref.random_banded(n, k, 1.0, 3)
    sizes, offs = ref.partition_layout(n, p, k)
    kb = np.full(p, k, np.int32)
    hp = np.ones(p, np.int32)
    pm = np.concatenate([np.arange(m, dtype=np.int32) for m in sizes])
    got = ref.ref_third_setup(n, k, band, p, kb, hp, pm)
    plain = ref.ref_factor_blocks(n, k, band, p, False)
    assert np.array_equal(np.concatenate(got["lu"]), plain["lu"][:sum(len(x) for x in got["lu"])])
    tips = ref.ref_spikes(n, k, band, p)
    for t in range(p - 1):
        vb = tips["vb"][t * k * k:(t + 1) * k * k].reshape(k, k)
        assert np.max(np.abs(got["vb"][t] - vb)) <= 1e-13 * max(1.0, np.max(np.abs(vb)))
        assert np.allclose(got["v_full"][t][-k:], got["vb"][t], rtol=0, atol=0)


def test_drop_off_k_monotone_in_tolerance(ref):
    rng = np.random.default_rng(2)
    n = 1500
    rp, ci, v = [0], [], []
    for i in range(n):
        js = sorted({i} | {int(x) for x in np.clip(i + rng.integers(-80, 81, 5), 0, n - 1)})
        ci += js
        v += [7.0 if j == i else rng.uniform(-1, 1) for j in js]
        rp.append(len(ci))
    ks = [ref.ref_drop_off(n, rp, ci, v, t)[0] for t in (0.0, 0.01, 0.05, 0.1, 0.3, 1.0)]
    assert ks == sorted(ks, reverse=True) and ks[-1] == 0
    with pytest.raises(ref.OracleError, match="tolerance"):
        ref.ref_drop_off(n, rp, ci, v, 1.5)
