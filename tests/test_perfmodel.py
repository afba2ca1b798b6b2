"""Pins of the performance model (§III-B/C) against closed forms and hand-computed values."""
import math

import numpy as np
import pytest

from paper_1506_09067_b200 import perfmodel as pm


def test_speedup_single_unit_is_one():
    assert pm.speedup(1, 2, 3, 4, 5, 6, 7, i=100, it=10, ep=3, p=1) == pytest.approx(1.0, abs=1e-15)


def test_speedup_no_sequential_work_is_linear_up_to_the_image_counts():
    # a = b = c = d = 0: S_p = p while p <= it <= i
    for p in (1, 2, 7, 10):
        assert pm.speedup(0, 0, 0, 0, 5, 6, 7, i=100, it=10, ep=3, p=p) == pytest.approx(p, rel=1e-12)


def test_speedup_clamps_p_to_the_image_counts():
    # p beyond i (and it): p_i = i, p_it = it, so the speed-up stops growing
    s100 = pm.speedup(0, 0, 0, 0, 1, 1, 1, i=100, it=10, ep=1, p=100)
    s1000 = pm.speedup(0, 0, 0, 0, 1, 1, 1, i=100, it=10, ep=1, p=1000)
    assert s100 == pytest.approx(s1000, rel=1e-15)
    # between it and i the test term saturates: hand-computed (2*100 + 10) / (2*100/50 + 10/10) = 42
    assert pm.speedup(0, 0, 0, 0, 1, 1, 1, i=100, it=10, ep=1, p=50) == pytest.approx(210 / 5, rel=1e-12)


def test_speedup_hand_value():
    # a..g = 1, i = 4, it = 2, ep = 2, p = 2: T1 = (4+2+1) + (1+4+4+2)*2 = 29;
    # Tp = 7 + (1 + 2 + 2 + 1)*2 = 19
    assert pm.speedup(1, 1, 1, 1, 1, 1, 1, i=4, it=2, ep=2, p=2) == pytest.approx(29 / 19, rel=1e-15)


def test_predict_time_rows():
    # hand-computed rows (2)-(5) with s = 2, CPI*OF = 3, contention 0.5
    i, it, ep, p, s = 8, 4, 2, 4, 2.0
    prep, fprop, bprop = 6.0, 10.0, 20.0
    rows = pm.t_comp_terms(i, it, ep, p, s, prep, fprop, bprop)
    assert rows["prep"] == pytest.approx((6 + 32 + 8 + 20) / 2)
    assert rows["train"] == pytest.approx(30 / 2 * (8 / 4) * 2)
    assert rows["validation"] == pytest.approx(10 / 2 * 2 * 2)
    assert rows["test"] == pytest.approx(10 / 2 * 1 * 2)
    t = pm.predict_time(i, it, ep, p, s, prep, fprop, bprop, 3.0, 0.5)
    assert t == pytest.approx(sum(rows.values()) * 3 + 0.5 * 8 * 2 / 4)


def test_t_mem_and_alpha():
    assert pm.t_mem(15, 60000, 244, 2e-6) == pytest.approx(2e-6 * 60000 * 15 / 244)
    assert pm.alpha(110.0, 100.0) == pytest.approx(10.0)
    assert pm.alpha(100.0, 100.0) == 0.0


def test_calibrate_recovers_known_constants():
    i, it, ep, s = 60000, 10000, 1, 1.9e9
    fprop, bprop = 3.5e6, 2.0e6
    cpi_opf, prep, mc = 0.37, 4.0e7, 4e-7
    pts = [(p, pm.predict_time(i, it, ep, p, s, prep, fprop, bprop, cpi_opf, mc, parts=("prep", "train")))
           for p in (1, 4, 16, 64, 592)]
    cal = pm.calibrate(pts, i, it, ep, s, fprop, bprop, contention=mc)
    assert cal.cpi_opf == pytest.approx(cpi_opf, rel=1e-9)
    assert cal.prep == pytest.approx(prep, rel=1e-6)
    assert cal.residual < 1e-9
    tab = pm.what_if(cal, s, fprop, bprop, [(592, 60000, 10000, 15), (1184, 120000, 10000, 15)])
    assert len(tab) == 2 and all(math.isfinite(r["seconds"]) and r["seconds"] > 0 for r in tab)
    assert np.isclose(tab[0]["seconds"], pm.predict_time(60000, 10000, 15, 592, s, prep, fprop, bprop, cpi_opf, mc))
