"""Pins for the oracle's SMAPE (Alg. 2 l.14), the CEM reading of "Gauss" (Alg. 2 l.8,
reading Z12) and Alg. 2 itself.

CEM: SPEC examples; library special case (well-separated mixtures: same
partition as sklearn KMeans and sklearn GaussianMixture); fixed-point invariant (the
returned labels are the argmax of the Z12 score under the parameters re-estimated from
those labels); first-pass closed form (nearest equal-width centre).
Alg. 2: hand-derived 2-window values (tests/golden/alg2_hand.json), exact zeros on
exactly periodic input, Err(T) < Err(1.5T), HF-interference
robustness, affine and within-window-permutation invariance.
"""
import json
import os

import numpy as np
import pytest
from sklearn.cluster import KMeans
from sklearn.mixture import GaussianMixture

import oracle as O

G = os.path.join(os.path.dirname(__file__), "golden")


def test_smape_spec_values():
    for c in json.load(open(os.path.join(G, "smape_spec.json")))["cases"]:
        assert O.smape(c["a"], c["b"]) == pytest.approx(c["smape"], abs=1e-15)
    assert O.smape(-3.0, 3.0) == 2.0  # opposite signs: the [0, 2] upper bound (Z14)
    assert O.smape(5.0, -1.0) == O.smape(-1.0, 5.0)


def _groups(labels):
    out = {}
    for i, l in enumerate(labels):
        out.setdefault(int(l), []).append(i)
    return sorted(out.values())


def test_gmm_spec_examples():
    g = json.load(open(os.path.join(G, "gmm_spec.json")))
    for c in g["cases"]:
        lab, _, _ = O.gmm_cem(np.array(c["values"], np.float32), c["num_groups"])
        assert _groups(lab) == sorted(c["groups"])
    t = g["two_gaussians"]
    rng = np.random.default_rng(0)
    v = np.concatenate([rng.normal(m, t["sigma"], t["n_each"]) for m in t["mu"]]).astype(np.float32)
    truth = np.repeat([0, 1], t["n_each"])
    lab, _, _ = O.gmm_cem(v, 2)
    match = max(np.mean(lab == truth), np.mean(lab == 1 - truth))
    assert match >= t["min_match"]


@pytest.mark.parametrize("seed", range(8))
def test_cem_matches_library_on_separated_mixtures(seed):
    # Special case that reduces to library routines: k well-separated clusters whose
    # centres sit near the Z12 equal-width initial centres. Any correct 1-D mixture
    # clustering (CEM, Lloyd k-means, soft-EM GMM) returns the generating partition.
    rng = np.random.default_rng(100 + seed)
    k = int(rng.integers(2, 5))
    lo, w = rng.uniform(-50, 50), rng.uniform(5, 40)
    centres = lo + (np.arange(k) + 0.5) * w + rng.uniform(-0.1, 0.1, k) * w
    sizes = rng.integers(5, 40, k)
    v = np.concatenate([c + np.clip(rng.normal(0, 1, s), -3, 3) * rng.uniform(0.005, 0.04) * w
                        for c, s in zip(centres, sizes)])
    truth = np.repeat(np.arange(k), sizes)
    order = rng.permutation(v.size)
    v, truth = v[order].astype(np.float32), truth[order]
    lab, _, _ = O.gmm_cem(v, k)
    vd = v.reshape(-1, 1).astype(np.float64)
    km = KMeans(n_clusters=k, init=centres.reshape(-1, 1), n_init=1).fit(vd)
    gm = GaussianMixture(n_components=k, means_init=centres.reshape(-1, 1), random_state=0).fit(vd)
    assert _groups(lab) == _groups(truth)
    assert _groups(lab) == _groups(km.labels_)
    assert _groups(lab) == _groups(gm.predict(vd))


def _z12_params(v, lab, G, R):
    """M-step of Z12 from labels (numpy, fp64)."""
    out = []
    for j in range(G):
        m = lab == j
        if not m.any():
            out.append(None)
            continue
        mu = v[m].mean()
        var = max(((v[m] - mu) ** 2).mean(), 1e-6 * R * R)
        out.append((m.sum() / v.size, mu, var))
    return out


@pytest.mark.parametrize("seed", range(12))
def test_cem_fixed_point_invariant(seed):
    # Converged CEM labels are a fixed point: each sample's label maximises
    # ln pi_j - 1/2 ln var_j - (v - mu_j)^2 / (2 var_j) under the parameters re-estimated
    # from the labels themselves (classification EM, Z12).
    rng = np.random.default_rng(seed)
    L = int(rng.integers(20, 300))
    # NVML-like quantised levels with noise: unequal variances and weights
    levels = rng.uniform(0, 50, 3)
    v = np.round(rng.choice(levels, L, p=[0.5, 0.3, 0.2]) + rng.normal(0, rng.uniform(0.5, 4), L)).astype(np.float32)
    lab, passes, _ = O.gmm_cem(v, 4, 200)
    assert passes < 200  # converged
    vd = v.astype(np.float64)
    R = vd.max() - vd.min()
    prm = _z12_params(vd, lab, 4, R)
    for s in range(L):
        sc = [(-np.inf if p is None else np.log(p[0]) - 0.5 * np.log(p[2]) - (vd[s] - p[1]) ** 2 / (2 * p[2]))
              for p in prm]
        best = int(np.argmax(sc))
        assert lab[s] == best or sc[lab[s]] >= sc[best] - 1e-9 * (abs(sc[best]) + 1)


def test_cem_first_pass_is_nearest_equal_width_centre():
    # With max_iters = 1 only the initial assignment runs: equal pi and var, so the label
    # is the nearest of the centres min + (j + 1/2) R / G (Z12 init).
    rng = np.random.default_rng(9)
    v = rng.uniform(-5, 5, 501).astype(np.float32)
    lab, passes, _ = O.gmm_cem(v, 4, 1)
    assert passes == 1
    vd = v.astype(np.float64)
    edges = vd.min() + (vd.max() - vd.min()) * np.array([0.25, 0.5, 0.75])
    want = np.searchsorted(edges, vd, side="left")  # value on an edge -> lower group (ties -> lowest j)
    assert np.array_equal(lab, want)


def test_cem_degenerate():
    lab, passes, _ = O.gmm_cem(np.full(17, 3.5, np.float32), 4)
    assert passes == 0 and (lab == 0).all()  # Z13: all-equal window -> one group
    lab, _, _ = O.gmm_cem(np.array([1, 2], np.float32), 4)  # L < G -> <= L groups
    assert len(set(lab.tolist())) == 2


def test_alg2_hand_values():
    for c in json.load(open(os.path.join(G, "alg2_hand.json")))["cases"]:
        y = np.array(c["signal"], np.float32)
        assert O.similarity_error(y, c["L"], c["num_groups"]) == pytest.approx(c["err"], abs=1e-12)


def _periodic(L0, N, rng, levels=4):
    prof = np.round(rng.uniform(0, 100, L0)) if levels == 0 else rng.choice(rng.uniform(0, 100, levels), L0)
    return np.tile(prof, N // L0 + 1)[:N].astype(np.float32)


@pytest.mark.parametrize("seed", range(6))
def test_alg2_exact_zero_at_period_and_multiples(seed):
    rng = np.random.default_rng(seed)
    L0 = int(rng.integers(5, 60))
    y = _periodic(L0, 2000, rng)
    assert O.similarity_error(y, L0) == 0.0
    assert O.similarity_error(y, 2 * L0) == 0.0
    assert O.similarity_error(y, L0 + 1) > 0.0


def test_alg2_true_period_beats_1p5x():
    # S:180 square-plus-sine trace
    n = np.arange(4096)
    T = 64
    y = (np.where((n % T) < T // 3, 10.0, 2.0) + 0.7 * np.sin(2 * np.pi * n / T)).astype(np.float32)
    assert O.similarity_error(y, T) < O.similarity_error(y, 96)


def test_alg2_hf_interference_suppressed():
    # periodic signal + HF interference of period << T -> Err(T) <= 0.1
    n = np.arange(8192)
    T = 200
    base = np.where((n % T) < 100, 10.0, 2.0)
    y = (base + 0.8 * np.sin(2 * np.pi * n / 7.3)).astype(np.float32)
    assert O.similarity_error(y, T) <= 0.1
    # ... while a pointwise (Euclidean-style) comparison sees the interference
    assert O.similarity_error(y, T) < O.similarity_error(y, T + 3)


def test_alg2_affine_and_permutation_invariance():
    rng = np.random.default_rng(11)
    N, L = 3000, 50
    y = (_periodic(L, N, rng) + rng.normal(0, 3, N)).astype(np.float32)
    e0 = O.similarity_error(y, L)
    # y -> a y + b (a > 0): CEM is affine-equivariant, SMAPE scale-free
    e1 = O.similarity_error((y.astype(np.float64) * 4.0 + 17.0).astype(np.float32), L)
    assert e1 == pytest.approx(e0, rel=1e-4)
    # the same permutation of sample positions inside every window leaves Err unchanged
    perm = rng.permutation(L)
    M = N // L
    yp = y.copy()
    for i in range(M):
        yp[i * L:(i + 1) * L] = y[i * L:(i + 1) * L][perm]
    assert O.similarity_error(yp, L) == pytest.approx(e0, rel=1e-9)
    # reversing the pair order (time reversal of whole windows) changes which window is
    # clustered, so Err is NOT invariant in general: guards against clustering W_{i+1}
    yr = np.concatenate([y[i * L:(i + 1) * L] for i in reversed(range(M))])
    assert O.similarity_error(yr, L) != e0
