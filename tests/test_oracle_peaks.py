"""Pins for oracle O3 (peaks -> candidate integer periods, Alg. 1 l.3-5) and
O6's local range (Alg. 1 l.11-13).

Pinned to SPEC worked examples, scipy.signal.find_peaks on plateau-free
spectra, hand-built spectra, and the paper's own fractional formulas evaluated in fp64.
"""
import json
import os

import numpy as np
import pytest
from scipy.signal import find_peaks

import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def _hand_spectrum(N, peaks):
    """A smooth low floor with isolated peaks {bin: power}."""
    P = np.full(N // 2 + 1, 1e-6)
    P += 1e-9 * np.arange(N // 2 + 1)[::-1]  # strictly decreasing floor: no floor peaks
    for k, v in peaks.items():
        P[k] = v
    return P


def test_spec_threshold_examples():
    g = json.load(open(os.path.join(G, "candidates_spec.json")))
    N = 1024
    for case in g["cases"]:
        amps = case["peak_amplitudes"]
        P = _hand_spectrum(N, {20: amps[0] ** 2, 45: amps[1] ** 2})
        r = O.candidates(P, O.Params(N, min_period=4, max_period=512, c_peak=g["c_peak"]))
        assert r.n_candidates == case["n_candidates"]
        assert r.cand_k[0] == 20 and r.cand_L[0] == N // 20


def test_single_tone_single_candidate():
    # single-tone spectrum -> exactly one candidate = the tone's period
    N, k0 = 2048, 37
    n = np.arange(N)
    y = np.cos(2 * np.pi * k0 * n / N + 0.3).astype(np.float32)
    P = O.power_spectrum(y)
    r = O.candidates(P, O.Params(N, min_period=4, max_period=N // 2))
    assert r.n_candidates == 1
    assert r.cand_k[0] == k0 and r.cand_L[0] == N // k0


def test_no_peak_means_no_candidate():
    N = 256
    P = np.linspace(10, 1, N // 2 + 1)  # strictly decreasing: no local maxima in band
    r = O.candidates(P, O.Params(N, min_period=4, max_period=64))
    assert r.n_candidates == 0 and r.n_peaks == 0


@pytest.mark.parametrize("seed", range(5))
def test_peaks_match_scipy_on_plateau_free(seed):
    rng = np.random.default_rng(seed)
    N = 4096
    P = rng.exponential(1.0, N // 2 + 1)  # continuous: no plateaus w.p. 1
    lo_k, hi_k = 40, 400
    Lmin, Lmax = N // hi_k, N // lo_k
    r = O.candidates(P, O.Params(N, min_period=Lmin, max_period=Lmax, c_peak=1e-3, max_candidates=32))
    sp, _ = find_peaks(P)
    band = [k for k in sp if Lmin <= N // k <= Lmax]
    assert r.n_peaks == len(band)
    top = sorted(band, key=lambda k: (-P[k], k))[:32]
    # top-K by power, then integer period with dedupe (first in ranking order wins)
    want = []
    seen = set()
    for k in top:
        if N // k not in seen:
            seen.add(N // k)
            want.append(k)
    assert list(r.cand_k[:r.n_candidates]) == want


def test_plateau_takes_leftmost_and_mirrored_edges():
    N = 64
    P = np.full(N // 2 + 1, 0.1)
    P[10] = P[11] = 5.0  # flat top: P[k] > P[k-1] and P[k] >= P[k+1] selects k = 10 (Z5)
    P[N // 2] = 3.0      # Nyquist bin: mirrored neighbour P[N/2+1] = P[N/2-1] (Z5)
    r = O.candidates(P, O.Params(N, min_period=2, max_period=32, c_peak=0.5))
    ks = list(r.cand_k[:r.n_candidates])
    assert 10 in ks and 11 not in ks
    assert N // 2 in ks


def test_top_k_cap_and_dedupe():
    N = 8192
    peaks = {k: 100.0 - i for i, k in enumerate(range(300, 300 + 2 * 40, 2))}  # 40 peaks, all pass
    P = _hand_spectrum(N, peaks)
    r = O.candidates(P, O.Params(N, min_period=10, max_period=4096, max_candidates=16))
    assert r.n_passing == 40 and r.cap_binds
    ks = list(r.cand_k[:r.n_candidates])
    Ls = list(r.cand_L[:r.n_candidates])
    assert len(set(Ls)) == len(Ls)
    # the 16 strongest peaks, minus those whose floor(N/k) repeats an earlier one
    expect, seen = [], set()
    for k in range(300, 332, 2):
        if N // k not in seen:
            seen.add(N // k)
            expect.append(k)
    assert ks == expect


def test_max_is_in_band_only():
    # Z7: an out-of-band drift peak must not suppress valid candidates
    N = 1024
    P = _hand_spectrum(N, {2: 1000.0, 30: 1.0})
    r = O.candidates(P, O.Params(N, min_period=4, max_period=100))
    assert r.n_candidates == 1 and r.cand_k[0] == 30


def test_local_range_worked_example():
    g = json.load(open(os.path.join(G, "local_range_cfg1.json")))
    for c in g["cases"]:
        assert O.local_range(g["N"], c["k_b"], 4, 512) == (c["lo"], c["hi"])


@pytest.mark.parametrize("N", [64, 1024, 8192, 65536, 262144])
def test_local_range_matches_paper_fractional_formula(N):
    # P:320-322 in fp64: Tc = N/k (T_s = 1), N_T = (N-1)/Tc, T_low = Tc(1-1/(N_T+1)), T_up = Tc(1+1/(N_T-1))
    for k in list(range(2, 200)) + list(range(N // 8, N // 8 + 50)):
        if k > N // 2:
            continue
        Tc = N / k
        NT = (N - 1) / Tc
        lo_f = Tc * (1 - 1 / (NT + 1))
        hi_f = Tc * (1 + 1 / (NT - 1))
        lo, hi = O.local_range(N, k, 1, N)
        # integer formula == floor of the fractional one (unless fp64 sits on an integer)
        if abs(lo_f - round(lo_f)) > 1e-9:
            assert lo == int(np.floor(lo_f))
        if abs(hi_f - round(hi_f)) > 1e-9:
            assert hi == min(int(np.floor(hi_f)), N)
        assert lo <= N // k <= hi  # the candidate itself is always in its local range


def test_order_margin_of_tied_peaks():
    # two candidates with equal power: their rank order (and, for a shared L, the dedupe) is a
    # tie -- d_order = 0 (Z27); well-separated powers give the relative gap
    N = 1024
    r = O.candidates(_hand_spectrum(N, {20: 1.0, 45: 1.0}), O.Params(N, min_period=4, max_period=512))
    assert r.n_candidates == 2 and r.d_order == 0.0
    r = O.candidates(_hand_spectrum(N, {20: 1.0, 45: 0.8}), O.Params(N, min_period=4, max_period=512))
    assert r.d_order == pytest.approx(0.2, rel=1e-12)
