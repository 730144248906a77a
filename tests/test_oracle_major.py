"""Pins for oracle S1, the spectral-only detector: T_iter = 1/f_major,
"the one with the largest amplitude is the major frequency component" (section
4.1.1; ODPP's method), under reading R3 (largest in-band Z5 peak, ties to the
smaller bin, integer period floor(N/k)).

Pinned to closed forms (pure and two-tone signals: the z-scored tone of amplitude A has
P = (A N / (2 sigma))^2), numpy.fft.rfft + scipy.signal.find_peaks on plateau-free
random spectra, the band rule (an out-of-band stronger tone is ignored, Z7), the
statuses, and the consistency with Alg. 1's first-ranked candidate (O3 uses the same
peak set and order).
"""
import numpy as np
import pytest
from scipy.signal import find_peaks

import oracle as O
import tracegen as tg


def _x(y):
    return np.asarray(y, np.float32)[None, :]


@pytest.mark.parametrize("N,k0", [(1024, 37), (4096, 5), (8192, 1000), (256, 64)])
def test_pure_tone_closed_form(N, k0):
    n = np.arange(N)
    y = 2.5 * np.cos(2 * np.pi * k0 * n / N + 0.4) + 7.0
    m = O.major(_x(y), O.Params(N, min_period=2, max_period=N // 2))
    assert m.status == O.TRACE_OK
    assert m.bin == k0 and m.period == N // k0
    # z-scored unit-variance tone: amplitude sqrt(2) -> P = (sqrt(2) N / 2)^2 = N^2 / 2
    assert m.power == pytest.approx(N * N / 2, rel=1e-6)


def test_two_tones_larger_wins_and_margin():
    N, A1, A2 = 2048, 3.0, 1.5
    n = np.arange(N)
    y = A1 * np.sin(2 * np.pi * 90 * n / N) + A2 * np.sin(2 * np.pi * 40 * n / N)
    m = O.major(_x(y), O.Params(N, min_period=4, max_period=N // 2))
    assert m.bin == 90 and m.period == N // 90
    assert m.d_major == pytest.approx(1 - (A2 / A1) ** 2, rel=1e-6)
    # swap amplitudes: the other bin wins
    y = A2 * np.sin(2 * np.pi * 90 * n / N) + A1 * np.sin(2 * np.pi * 40 * n / N)
    assert O.major(_x(y), O.Params(N, min_period=4, max_period=N // 2)).bin == 40


def test_out_of_band_tone_ignored():
    # Z7: the band [L_min, L_max] = [4, 64] excludes bin 10 (period 102); bin 50 (period 20) is in band
    N = 1024
    n = np.arange(N)
    y = 5.0 * np.cos(2 * np.pi * 10 * n / N) + 1.0 * np.cos(2 * np.pi * 50 * n / N)
    m = O.major(_x(y), O.Params(N, min_period=4, max_period=64))
    assert m.bin == 50 and m.period == 20


def test_equal_tones_reported_as_near_tie():
    # equal amplitudes: the two powers differ only by the fp32 rounding of y, and the
    # oracle reports the near-tie (Z27), so either bin is a valid answer
    N = 1024
    n = np.arange(N)
    y = np.cos(2 * np.pi * 30 * n / N) + np.cos(2 * np.pi * 60 * n / N)
    m = O.major(_x(y), O.Params(N, min_period=4, max_period=N // 2))
    assert m.bin in (30, 60)
    assert m.d_major < 1e-6 and m.ambiguous()


@pytest.mark.parametrize("seed", range(6))
def test_matches_numpy_scipy(seed):
    rng = np.random.default_rng(seed)
    N = 2048
    y = np.cumsum(rng.normal(size=N)).astype(np.float32)  # red-noise-like: many distinct peaks
    y += (2 * np.sin(2 * np.pi * rng.integers(20, 200) * np.arange(N) / N)).astype(np.float32)
    Lmin, Lmax = 8, 400
    m = O.major(_x(y), O.Params(N, min_period=Lmin, max_period=Lmax))
    # library: fp64 rfft of the same composite signal (O1, pinned separately); in-band
    # interior peaks by scipy; the largest (ties to the smaller bin)
    z = O.composite(_x(y))[0]
    assert np.allclose(z, (y - y.mean()) / y.std(), rtol=0, atol=1e-5)
    P = np.abs(np.fft.rfft(z.astype(np.float64))) ** 2
    ks = np.arange(N // 2 + 1)
    band = (ks >= 1) & (N // np.maximum(ks, 1) >= Lmin) & (N // np.maximum(ks, 1) <= Lmax)
    pk, _ = find_peaks(P)
    pk = [k for k in pk if band[k]]
    want = max(pk, key=lambda k: (P[k], -k))
    assert m.bin == want and m.period == N // want
    assert m.power == pytest.approx(P[want], rel=1e-9)


def test_statuses():
    N = 64
    P = O.Params(N, min_period=2, max_period=32)
    assert O.major(_x(np.full(N, 3.0)), P).status == O.TRACE_CONSTANT
    # floor(64/k) never equals 25 -> empty band
    assert O.major(_x(np.arange(N) % 7), O.Params(N, min_period=25, max_period=25)).status == O.TRACE_INSUFFICIENT
    # a strictly monotone ramp's spectrum decreases in k: no in-band peak
    r = O.major(_x(np.arange(N, dtype=np.float64)), O.Params(N, min_period=4, max_period=16))
    assert r.status == O.TRACE_APERIODIC and r.period == -1


def test_agrees_with_alg1_first_candidate():
    # O3 ranks the same in-band peaks by (P desc, k asc): its first candidate is f_major
    spec = tg.CFG2.with_(batch=6)
    X = tg.generate_host(spec)
    P = O.params_for(spec)
    for i in range(X.shape[0]):
        m = O.major(X[i], P)
        d = O.detect(X[i], P)
        assert m.status == d.status
        if d.status == O.TRACE_OK:
            assert d.cand_k[0] == m.bin


def test_band_only_dft_same_answer():
    spec = tg.CFG2.with_(batch=2)
    X = tg.generate_host(spec)
    a = O.major(X[0], O.params_for(spec))
    b = O.major(X[0], O.params_for(spec, dft_band_only=True))
    assert (a.bin, a.period, a.status) == (b.bin, b.period, b.status)
    assert a.power == b.power
