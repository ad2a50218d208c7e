"""Host-side planning invariants of the layer scheduler (step a0), checked on CPU through the ABI's
planning introspection (mps_plan_regime; no device work): every theta shape lands in an SVD regime
whose bucket parameters exist -- lane groups are powers of two in [4, 32], rows per lane cover the
rows, the QR regime's one-pair-per-group CTA fits, the large regime pads n to the 64-column panels.
A shape outside every bucket would silently skip its SVD (config 5 layer 7, m = 98, n = 106)."""
import numpy as np
import pytest


def _plan(m, n):
    import paper_2307_16870_b200 as pk
    return pk.mps_plan_regime(m, n)


def test_plan_invariants_over_shapes():
    shapes = [(m, n) for m in list(range(2, 130, 2)) + [196, 256, 400, 512, 1024, 4096]
              for n in list(range(2, 130, 2)) + [140, 200, 256, 300, 512, 2048, 8192]]
    seen = set()
    for m, n in shapes:
        reg, gt, rpl, npad = _plan(m, n)
        seen.add(reg)
        if reg == 1:
            assert npad % 64 == 0 and npad >= n > 0, (m, n, npad)
            continue
        assert npad == n
        assert gt in (4, 8, 16, 32), (m, n, reg, gt)
        assert rpl in (0, 1, 2, 4, 8, 16), (m, n, reg, rpl)
        if reg == 3:
            assert m >= n and 64 <= n <= 256 and (n // 2) * gt <= 512 and rpl > 0 and n <= rpl * gt, (m, n, gt, rpl)
        elif rpl > 0:
            assert m <= rpl * gt and n <= rpl * gt, (m, n, reg, gt, rpl)
    assert seen == {0, 1, 2, 3}


def test_config5_layer7_shape_is_bucketed():
    reg, gt, rpl, _ = _plan(98, 106)
    assert reg == 0 and gt in (4, 8, 16, 32)


@pytest.mark.parametrize("m,n,reg", [(32, 32, 0), (128, 128, 3), (64, 144, 2), (512, 512, 1), (2048, 2048, 1)])
def test_config2_regimes(m, n, reg):
    assert _plan(m, n)[0] == reg


def test_plan_rejects_bad_shapes():
    import paper_2307_16870_b200 as pk
    with pytest.raises(pk.EampsError):
        pk.mps_plan_regime(0, 4)
