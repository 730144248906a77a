"""Pins for oracle R1: Alg. 3, the online robust period detection framework (
SURVEY 8f row 1), on a recorded trace under reading R5.

Pinned to hand evaluations of the algorithm's own formulas: the suffix starts
t_start = max(0, SmpDur - (2 + c_eval step) T_init) + j step T_init while
(SmpDur - t_start)/T_init >= c_measure (lines 7-13), the early exit of lines 3-6 with
SmpDur_next = c_measure T_init - SmpDur, and SmpDur_next = ceil(SmpDur/max T) max T - SmpDur
(lines 16-21); plus planted periods: a stationary trace (every T_j equals the planted
period, Diff = 0, stop sampling) and a mid-trace period change (the rolling suffixes see
only the new period, which T_iter reports although Alg. 1 on the whole trace found the old).
"""
import math

import numpy as np
import pytest

import oracle as O
import tracegen as tg


def _starts(N, L0, c_measure=2.0, step=0.5, c_eval=6.5):
    smpdur = N - 1
    t = max(0.0, smpdur - (2 + c_eval * step) * L0)
    out = []
    while (smpdur - t) / L0 >= c_measure:
        out.append(int(math.floor(t)))
        t += step * L0
    return out


def test_stationary_planted_period_config1():
    x = tg.generate_host(tg.CFG1)[0]
    r = O.rolling(x, O.params_for(tg.CFG1))
    assert r.status == O.TRACE_OK and r.t_init == 37 and not r.early
    # hand: t0 = 1023 - 5.25 * 37 = 828.75, step 18.5, last t <= 1023 - 74 = 949
    assert r.sub_start == [828, 847, 865, 884, 902, 921, 939] == _starts(1024, 37)
    assert r.sub_period == [37] * 7
    assert r.t_iter == 37 and r.diff == 0.0 and r.smpdur_next == -1.0


def test_early_exit_short_sampling():
    # period 64 in N = 128: SmpDur = 127 < 2 * 64 -> lines 3-6: T_iter = T_init,
    # SmpDur_next = 2 * 64 - 127 = 1, no rolling
    N = 128
    n = np.arange(N)
    y = (np.sin(2 * np.pi * n / 64 + 0.3) + 0.2 * np.sin(2 * np.pi * 3 * n / 64)).astype(np.float32)
    r = O.rolling(y[None], O.Params(N, min_period=4, max_period=64))
    assert r.early and r.t_init == 64 and r.t_iter == 64
    assert r.smpdur_next == 2 * 64 - 127 and r.sub_start == []


def test_period_change_mid_trace():
    # first half period 40, second half period 56 (with a harmonic): Alg. 1 on the whole trace
    # finds 40; the suffixes (the last 5.25 T_init samples) see only the second regime
    N = 2048
    n = np.arange(N)
    y = np.where(n < N // 2, np.sin(2 * np.pi * n / 40), np.sin(2 * np.pi * n / 56) + 0.5 * np.sin(4 * np.pi * n / 56))
    r = O.rolling(y[None].astype(np.float32), O.Params(N, min_period=8, max_period=512))
    assert r.t_init == 40
    assert r.sub_start == _starts(N, 40) == [1837, 1857, 1877, 1897, 1917, 1937, 1957]
    assert r.t_iter == 56
    assert r.sub_period.count(56) >= 5
    T = [t for t in r.sub_period if t > 0]
    assert r.diff == pytest.approx(abs(max(T) - min(T)) / np.mean(T))
    assert r.diff >= 0.05  # the suffixes disagree: keep sampling
    assert r.smpdur_next == math.ceil(2047 / max(T)) * max(T) - 2047


def test_aperiodic_whole_trace_no_rolling():
    x = np.full((1, 256), 7.0, np.float32)
    r = O.rolling(x, O.Params(256, min_period=4, max_period=128))
    assert r.status == O.TRACE_CONSTANT and r.t_iter == -1 and r.sub_start == []


@pytest.mark.parametrize("L0", [20, 37, 50])
def test_suffix_count_closed_form(L0):
    # J = floor((SmpDur - t0 - c_measure T) / (step T)) + 1 with t0 = SmpDur - 5.25 T (> 0):
    # (5.25 - 2) / 0.5 = 6.5 -> 7 suffixes whenever the trace is longer than 5.25 periods
    N = 1024
    n = np.arange(N)
    y = np.where((n % L0) < L0 // 3, 1.0, 0.0).astype(np.float32) + 0.01 * np.sin(n)
    r = O.rolling(y[None].astype(np.float32), O.Params(N, min_period=4, max_period=N // 2))
    assert r.t_init == L0
    assert len(r.sub_start) == 7 and r.sub_start == _starts(N, L0)
