"""Pins for oracle O1 (composite) and O2 (DFT power spectrum).

O2 is the plain DFT definition (Alg. 1 l.1); pinned to closed forms (pure tone,
impulse, Parseval) and to a library routine (numpy.fft.rfft, fp64).
O1 (composite, reading Z1) is pinned to the textbook z-score and its invariants.
"""
import numpy as np
import pytest

import oracle as O


@pytest.mark.parametrize("N,k0,A", [(1024, 28, 3.0), (64, 5, 1.5), (8192, 221, 0.25), (96, 7, 2.0)])
def test_pure_tone_closed_form(N, k0, A):
    # y = A cos(2 pi k0 n / N)  =>  X_k0 = A N / 2, every other bin 0
    n = np.arange(N)
    y = (A * np.cos(2 * np.pi * k0 * n / N)).astype(np.float32)
    P = O.power_spectrum(y)
    Y = np.fft.rfft(y.astype(np.float64))  # the input really is fp32-rounded
    assert P[k0] == pytest.approx((A * N / 2) ** 2, rel=1e-6)
    others = np.delete(P, k0)
    assert others.max() <= 1e-10 * P[k0]
    assert np.argmax(P) == k0
    assert np.abs(P - np.abs(Y) ** 2).max() <= 1e-10 * P.max()


def test_impulse_is_flat():
    N = 256
    y = np.zeros(N, np.float32)
    y[0] = 1.0
    P = O.power_spectrum(y)
    np.testing.assert_allclose(P, 1.0, rtol=0, atol=1e-13)
    # delayed impulse: |X_k| = 1 for every k
    y = np.zeros(N, np.float32)
    y[37] = 2.0
    np.testing.assert_allclose(O.power_spectrum(y), 4.0, rtol=1e-12)


@pytest.mark.parametrize("N", [8, 64, 1000, 1024, 4096])
def test_parseval(N):
    rng = np.random.default_rng(N)
    y = rng.standard_normal(N).astype(np.float32)
    P = O.power_spectrum(y)
    # sum |y|^2 = (1/N) sum_{k<N} |X_k|^2, folded onto k = 0..N/2 for a real signal
    if N % 2 == 0:
        folded = P[0] + 2 * P[1:N // 2].sum() + P[N // 2]
    else:
        folded = P[0] + 2 * P[1:].sum()
    assert folded / N == pytest.approx(float(np.sum(y.astype(np.float64) ** 2)), rel=1e-11)


@pytest.mark.parametrize("N", [8, 100, 512, 2048, 8192])
def test_matches_numpy_rfft(N):
    rng = np.random.default_rng(7 + N)
    y = (rng.standard_normal(N) * 3 + np.sin(np.arange(N) * 0.3)).astype(np.float32)
    P = O.power_spectrum(y)
    ref = np.abs(np.fft.rfft(y.astype(np.float64))) ** 2
    assert np.abs(P - ref).max() <= 1e-12 * ref.max()


def test_composite_single_channel_is_textbook_zscore():
    x = (np.arange(100, dtype=np.float32) * 3 + 7)[None, :]
    y, mu, sg, const = O.composite(x)
    assert not const
    xd = x[0].astype(np.float64)
    ref = (xd - xd.mean()) / xd.std()  # population std (ddof=0), Z1
    assert mu[0] == pytest.approx(xd.mean(), rel=1e-15)
    assert sg[0] == pytest.approx(xd.std(), rel=1e-14)
    np.testing.assert_allclose(y, ref.astype(np.float32), rtol=2e-7, atol=1e-7)
    assert abs(float(np.mean(y.astype(np.float64)))) < 1e-6
    assert float(np.std(y.astype(np.float64))) == pytest.approx(1.0, rel=1e-6)


def test_composite_constant_channel_contributes_zero():
    rng = np.random.default_rng(3)
    p = np.round(rng.uniform(100, 300, 512)).astype(np.float32)
    x1 = p[None, :]
    x2 = np.stack([p, np.full(512, 55.0, np.float32)])
    y1, _, _, _ = O.composite(x1)
    y2, _, sg, _ = O.composite(x2)
    assert sg[1] == 0.0
    assert np.array_equal(y1, y2)  # S:261 "zero-variance channel drops out"
    _, _, _, const = O.composite(np.full((3, 64), 4.0, np.float32))
    assert const


def test_composite_weights_projection_and_affine_invariance():
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 100, (3, 300)).astype(np.float32)
    y_w, _, _, _ = O.composite(x, weights=(1.0, 0.0, 0.0))
    y_p, _, _, _ = O.composite(x[:1])
    assert np.array_equal(y_w, y_p)  # S:262 weights (1,0,0) -> normalised power
    # per-channel affine rescaling (a>0) leaves the composite unchanged
    xs = x.astype(np.float64) * np.array([[2.0], [0.5], [4.0]]) + np.array([[10.0], [-3.0], [0.25]])
    y_s, _, _, _ = O.composite(xs.astype(np.float32))
    y0, _, _, _ = O.composite(x)
    np.testing.assert_allclose(y_s, y0, atol=2e-5)


def test_composite_identical_sinusoids():
    # three identical sinusoid channels -> composite is a sinusoid of the same period
    n = np.arange(1024)
    s = (50 + 20 * np.sin(2 * np.pi * n / 64)).astype(np.float32)
    y, _, _, _ = O.composite(np.stack([s, s, s]))
    P = O.power_spectrum(y)
    assert int(np.argmax(P)) == 1024 // 64
    y1, _, _, _ = O.composite(s[None])
    np.testing.assert_allclose(y, 3 * y1, rtol=1e-6, atol=1e-6)


def test_band_only_dft_same_values():
    # the band-only evaluation computes the same per-bin arithmetic, only fewer bins
    rng = np.random.default_rng(1)
    y = rng.standard_normal(2048).astype(np.float32)
    P = O.power_spectrum(y)
    np.testing.assert_array_equal(O.power_spectrum_bins(y, 100, 300), P[100:301])
    x = (rng.standard_normal((1, 2048)) * 5 + np.sin(np.arange(2048) * 2 * np.pi / 41)).astype(np.float32)
    a = O.detect(x, O.Params(2048, 1, min_period=10, max_period=400))
    b = O.detect(x, O.Params(2048, 1, min_period=10, max_period=400, dft_band_only=True))
    assert a.period == b.period and a.cand_L == b.cand_L and a.error == b.error and a.margins == b.margins


def _fp32_rounding_is_clear(v64: float, rel=1e-12) -> bool:
    """False when v lies within rel of an fp32 rounding boundary (a midpoint between two
    adjacent fp32 values): there a rounding-once claim cannot be checked bit for bit."""
    r = np.float32(v64)
    if not np.isfinite(r) or v64 == 0.0:
        return True
    up = np.nextafter(r, np.float32(np.inf))
    dn = np.nextafter(r, np.float32(-np.inf))
    mids = [(float(r) + float(up)) / 2, (float(r) + float(dn)) / 2]
    return min(abs(v64 - m) for m in mids) > rel * abs(v64)


@pytest.mark.parametrize("F,weights,N", [(1, None, 257), (3, None, 257), (3, (1.0, 0.5, 2.0), 257), (2, (0.25, 1.0), 257),
                                         (1, None, 65536)])
def test_composite_is_the_exact_definition_rounded_once(F, weights, N):
    """Z23: y[n] is the exact value of the definition (Z1) sum_c w_c (x_c[n] - mu_c)
    / sigma_c rounded to fp32 once. Reference: a 50-digit decimal evaluation of the
    definition (no binary floating point in it), compared bit for bit wherever the exact
    value is not within 1e-12 of an fp32 rounding boundary. At N = 2^16 (config 3's length)
    on integer readings this also checks the statistics' accuracy (a plain running fp64 sum
    of the squares is up to ~1e-12 off at this length, which moves the rounding of a sample
    now and then)."""
    from decimal import Decimal, getcontext
    getcontext().prec = 50
    rng = np.random.default_rng(F + (0 if weights is None else 7))
    x = np.round(rng.uniform(0, 300, (F, N)) + 40 * np.sin(np.arange(N) * 0.07), 1).astype(np.float32)
    if N > 1000:  # NVML-like integer readings (the GPU composite test's data)
        x = np.round(rng.uniform(0, 300, (F, N)) + 50 * np.sin(np.arange(N) * 0.01)).astype(np.float32)
    y, _, _, _ = O.composite(x, weights=weights)
    w = [Decimal(float(np.float32(v))) for v in (weights or (1.0,) * F)]
    cols = []
    for c in range(F):
        xs = [Decimal(float(v)) for v in x[c]]
        mu = sum(xs) / N
        sigma = (sum((v - mu) ** 2 for v in xs) / N).sqrt()
        cols.append([(v - mu) / sigma * w[c] for v in xs])
    checked = 0
    for n in range(N):
        exact = float(sum(col[n] for col in cols))  # correctly rounded to fp64 (50 digits first)
        if not _fp32_rounding_is_clear(exact):
            continue
        assert y[n] == np.float32(exact), (n, y[n], exact)
        checked += 1
    assert checked >= N - 2
