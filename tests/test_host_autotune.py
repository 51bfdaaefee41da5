"""Host autotuner (Controller, AT1..AT3b) replays the reference step for step.

Golden streams (tests/golden/controller.npz) were produced by the compiled
reference Controller (proj/src/autotune.cpp); the live test feeds fresh
random streams to both."""
import numpy as np
import pytest

from conftest import load_golden
from oracle import oracle as O
from paper_1311_1006_b200 import fmm as F

KINDS = ["none", "at1", "at2", "at3a", "at3b"]


def _cc(cf, ci):
    return F.ControllerConfig(theta_min=cf[0], theta_max=cf[1], base_thetastep=cf[2], cap=cf[3],
                              nl_min=int(ci[0]), nl_max=int(ci[1]), theta_every=int(ci[2]),
                              nl_every=int(ci[3]), filter_window=int(ci[4]),
                              init_fiblength=int(ci[5]), max_fiblength=int(ci[6]))


def test_controller_matches_reference_golden():
    g = load_golden("controller.npz")
    for c in range(int(g["count"])):
        kind = KINDS[int(g[f"{c}_kind"])]
        out, ev = F.controller_run(kind, _cc(g[f"{c}_cf"], g[f"{c}_ci"]), 0.5, 5,
                                   int(g[f"{c}_seed"]), g[f"{c}_meas"])
        assert np.array_equal(out, g[f"{c}_out"]), (c, kind)
        assert np.array_equal(ev, g[f"{c}_ev"]), (c, kind)


@pytest.mark.skipif(not O.ref_available(), reason="reference library not built here")
@pytest.mark.parametrize("kind", range(5))
def test_controller_matches_live_reference(kind):
    rng = np.random.default_rng(kind + 50)
    for trial in range(4):
        n = 600
        # V-shaped landscape in the step index plus noise and wait signs
        t = 1.0 + 0.3 * rng.random(n) + 0.2 * np.sin(np.arange(n) / 30.0) ** 2
        w = np.where(rng.random(n) < 0.5, 0.02 * rng.random(n), 0.0)
        meas = np.stack([t, w, np.full(n, float(trial % 2))], 1)
        cf = np.array([0.3, 0.7, 0.02, [0.1, 0.0, 0.3, 0.05][trial]])
        ci = np.array([2, 9, 2, [10, 4, 7, 3][trial], [3, 1, 2, 5][trial], 3, 8], dtype=np.int32)
        out_r = np.empty((n, 2))
        ev_r = np.empty((n, 3), dtype=np.int32)
        assert O.ref_lib().fmmref_controller_run(kind, cf, ci, 0.45, 6, 7 + trial, n, meas.ravel(),
                                                 out_r.ravel(), ev_r.ravel()) == 0
        out, ev = F.controller_run(KINDS[kind], _cc(cf, ci), 0.45, 6, 7 + trial, meas)
        assert np.array_equal(out, out_r)
        assert np.array_equal(ev, ev_r)


def test_at3a_follows_wait_signal_and_equals_at2_without_it():
    n = 200
    cc = F.ControllerConfig(nl_every=2, theta_every=1000)
    t = np.ones(n)
    up = np.stack([t, np.full(n, 0.01), np.ones(n)], 1)  # CPU waits -> deeper tree
    out, _ = F.controller_run("at3a", cc, 0.5, 4, 1, up)
    assert out[:, 1].max() > 4
    nowait = np.stack([t + 0.001 * np.arange(n), np.zeros(n), np.zeros(n)], 1)
    a, _ = F.controller_run("at3a", cc, 0.5, 4, 1, nowait)
    b, _ = F.controller_run("at2", cc, 0.5, 4, 1, nowait)
    assert np.array_equal(a, b)


def test_controller_validation():
    with pytest.raises(F.InvalidParameter):
        F.controller_run("at2", F.ControllerConfig(cap=-1.0), 0.5, 4, 1, np.ones((3, 3)))
    with pytest.raises(F.InvalidInput):
        F.controller_run("at2", F.ControllerConfig(), 0.5, 4, 1, np.zeros((3, 3)))
