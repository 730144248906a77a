"""Pins for the oracle's Alg. 1 end to end.

Planted truth (config 1 of BASELINE.json: period 37), brute force on tiny inputs
(exhaustive argmin over every L, O9), pure tones, statuses, and method accuracy on a
config-2-like suite as context (paper: mean 1.72 %, max 7.2 %).
"""
import numpy as np
import pytest

import oracle as O
import tracegen as tg


def test_config1_planted_37():
    x = tg.generate_host(tg.CFG1)
    d = O.detect(x[0], O.params_for(tg.CFG1))
    assert d.status == O.TRACE_OK
    assert d.period == 37
    assert d.local_lo <= 37 <= d.local_hi
    assert not d.ambiguous()


@pytest.mark.parametrize("noise", [0.02, 0.10])
def test_config1_planted_37_other_noise(noise):
    spec = tg.CFG1.with_(noise=noise)
    d = O.detect(tg.generate_host(spec)[0], O.params_for(spec))
    assert d.period == 37


def _piecewise_periodic(N, L0, rng):
    """Noiseless random profile (integer levels, NVML-like) with minimal period L0.
    Per-sample levels, not long constant runs: Alg. 2 gives Err = 0 to any L whose
    windows are all constant (Z13), so long flat segments would make tiny L tie at 0."""
    while True:
        prof = np.round(rng.uniform(0, 100, L0))
        # minimal period L0: no proper divisor d of L0 is a period of the profile
        if all(not np.array_equal(prof, np.roll(prof, d)) for d in range(1, L0) if L0 % d == 0):
            return np.tile(prof, N // L0 + 1)[:N].astype(np.float32)


@pytest.mark.parametrize("N,seed", [(64, 0), (64, 1), (128, 2), (128, 3), (256, 4), (256, 5), (256, 6)])
def test_exhaustive_tiny_inputs(N, seed):
    rng = np.random.default_rng(seed)
    L0 = int(rng.integers(3, N // 4 + 1))
    y = _piecewise_periodic(N, L0, rng)
    Lb, errs = O.exhaustive(y, 2, N // 2)
    assert Lb == L0  # Err(L0) = 0 exactly and ties go to the smaller L (Z17)
    assert errs[L0 - 2] == 0.0
    # Alg. 1 (FFT candidates + local search) returns L0 whenever the fundamental bin is a candidate
    d = O.detect(y[None, :], O.Params(N, 1, min_period=2, max_period=N // 2))
    if any(N // k in range(d.local_lo, d.local_hi + 1) and d.best_bin == k for k in [int(round(N / L0))]):
        assert d.period == L0
    if d.local_lo <= L0 <= d.local_hi:
        assert d.period == L0


@pytest.mark.parametrize("k0", [16, 40, 100])
def test_pure_tone_lands_in_local_range(k0):
    N = 4096
    n = np.arange(N)
    y = (50 + 10 * np.cos(2 * np.pi * k0 * n / N)).astype(np.float32)
    d = O.detect(y[None], O.Params(N, 1, min_period=4, max_period=1024))
    assert d.status == O.TRACE_OK
    assert d.n_candidates == 1 and d.cand_L[0] == N // k0
    assert d.local_lo <= d.period <= d.local_hi
    assert d.local_lo <= N // k0 <= d.local_hi


def test_statuses():
    N = 256
    d = O.detect(np.full((3, N), 7.0, np.float32), O.Params(N, 3, min_period=4, max_period=64))
    assert d.status == O.TRACE_CONSTANT and d.period == -1
    ramp = np.arange(N, dtype=np.float32)[None]  # |X_k| decreasing in k: no in-band peak
    d = O.detect(ramp, O.Params(N, 1, min_period=4, max_period=64))
    assert d.status == O.TRACE_APERIODIC
    with pytest.raises(ValueError):
        O.detect(ramp, O.Params(N, 1, min_period=4, max_period=200))  # L_max > N/2


def test_sample_interval_scales_seconds_only():
    x = tg.generate_host(tg.CFG1)[0]
    a = O.detect(x, O.params_for(tg.CFG1))
    b = O.detect(x, O.Params(1024, 1, sample_interval=0.1, min_period=4, max_period=512))
    assert a.period == b.period and a.error == b.error
    assert b.period_s == pytest.approx(0.1 * b.period)


def test_config2_accuracy_context():
    # Context, not parity: the method's accuracy on the config-2-like suite. The paper
    # reports mean 1.72 % / max 7.2 % on real traces; synthetic traces with
    # HF interference fool the c_peak gate sometimes (a property of the method).
    spec = tg.CFG2.with_(batch=24)
    X = tg.generate_host(spec)
    ds = O.detect_batch(X, O.params_for(spec))
    errs = []
    for i, d in enumerate(ds):
        t = tg.planted_period(spec, i)
        if np.isnan(t):
            continue
        errs.append(abs(d.period - t) / t)
    errs = np.array(errs)
    assert np.mean(errs < 0.05) >= 0.6


def test_given_candidates_and_forced_best_reproduce_alg1():
    # the parity harness's hooks: Alg. 1 from line 6 on a given candidate list (its own) and
    # with Tcand_opt forced to its own argmin give back exactly the same result
    x = tg.generate_host(tg.CFG2, 5, 1)[0]
    p = O.params_for(tg.CFG2)
    d = O.detect(x, p)
    assert d.status == O.TRACE_OK
    g = O.detect(x, p, given_k=d.cand_k)
    f = O.detect(x, p, force_kb=d.best_bin)
    for e in (g, f):
        assert (e.period, e.best_bin, e.local_lo, e.local_hi) == (d.period, d.best_bin, d.local_lo, d.local_hi)
        assert e.cand_err == d.cand_err and np.array_equal(e.local_err, d.local_err)
        assert np.array_equal(e.local_margin, d.local_margin)
    assert min(d.cand_margin + list(d.local_margin)) == d.margins["d_cem"]
    # forcing another candidate moves the local range to that candidate's bin
    if d.n_candidates > 1:
        other = [k for k in d.cand_k if k != d.best_bin][0]
        e = O.detect(x, p, force_kb=other)
        assert e.best_bin == other and (e.local_lo, e.local_hi) == O.local_range(8192, other, 10, 4096)
