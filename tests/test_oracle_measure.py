"""Pins for oracle M1: Alg. 4 lines 1-9, adaptive feature measurement (SURVEY 8f
row 3), with a recorded trace as the simulated sampling backend (reading R6).

Pinned to hand evaluations: a session that starts with enough samples of a stationary trace
stops after one Alg. 3 call (Diff = 0 -> SmpDur_next = -1); a session started at exactly
2 T_init samples takes Alg. 3's early exit (SmpDur = 2T - 1 < c_measure T -> SmpDur_next =
2T - (2T - 1) = 1), waits one sample and stops in round 2 with 2T + 1 samples; a recording
too short for the requested wait ends UNSTABLE; the measurement window is [n, n + T_iter).
"""
import numpy as np
import pytest

import oracle as O
import tracegen as tg


def _square(N, L0, duty=7):
    n = np.arange(N)
    return (np.where((n % L0) < duty, 1.0, 0.0) + 0.01 * np.sin(0.37 * n)).astype(np.float32)[None]


def test_stationary_stops_after_one_round():
    x = tg.generate_host(tg.CFG1)[0]
    m = O.measure(x, O.params_for(tg.CFG1), 1024)
    assert m == dict(status=O.TRACE_OK, t_iter=37, rounds=1, samples=1024, measure_start=1024, measure_end=1061,
                     err_iter=m["err_iter"], amb=False)


@pytest.mark.parametrize("L0", [20, 33])
def test_early_exit_then_one_sample_more(L0):
    m = O.measure(_square(2048, L0), O.Params(2048, min_period=4, max_period=1024), 2 * L0)
    assert m["rounds"] == 2 and m["samples"] == 2 * L0 + 1 and m["t_iter"] == L0
    assert (m["measure_start"], m["measure_end"]) == (2 * L0 + 1, 3 * L0 + 1)


def test_recording_too_short_is_unstable():
    # 40 samples of period 20: the early exit asks for one more sample than the recording holds
    m = O.measure(_square(40, 20), O.Params(40, min_period=4, max_period=20), 40)
    assert m["status"] == O.TRACE_UNSTABLE and m["rounds"] == 1 and m["t_iter"] == 20


def test_too_short_for_min_period():
    m = O.measure(_square(64, 20), O.Params(64, min_period=10, max_period=32), 8)
    assert m["status"] == O.TRACE_INSUFFICIENT and m["t_iter"] == -1 and m["rounds"] == 1
