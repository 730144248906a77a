"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bars (BASELINE.json north star; the harness is tests/parity.py):
  * detected periods, candidate lists, best bins, local ranges, statuses: bit-exact;
  * spectra: normwise max|P_gpu - P_ref| <= 1e-4 max P_ref (Z29);
  * Alg. 2 scores of every candidate AND every local L: |Err_gpu - Err_ref| <= 1e-4 max(Err_ref, 1e-6)
    (Z30);
  * composite signal: the fp64 expression rounded once on both sides (Z23) -- bit-identical
    except where the two sides' fp64 statistics (summed in different orders) straddle an fp32
    rounding boundary: <= 1 ulp there, counted (expected ~1e-8 of the samples).
Where the oracle records a decision margin below what the precision difference between the
two sides can move (Z27), several answers are correct: the GPU's answer is then checked for
validity against the oracle (parity.py), and every such exclusion is counted with its reason.
"""
import numpy as np
import pytest

import torch  # noqa: E402

import oracle as O  # noqa: E402
import paper_2201_01684_b200 as g  # noqa: E402
import parity as PH  # noqa: E402
import tracegen as tg  # noqa: E402

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not torch.cuda.is_available(), reason="needs a CUDA device")]


def _to_dev(x: np.ndarray):
    """[B][F][N] -> device rows of trace_stride = F*N rounded up to 4 floats (the ABI's
    16-byte alignment rule; default_params uses the same stride)."""
    B = x.shape[0]
    flat = x.reshape(B, -1)
    stride = (flat.shape[1] + 3) & ~3
    rows = np.zeros((B, stride), np.float32)
    rows[:, :flat.shape[1]] = flat
    return torch.from_numpy(rows).cuda()


def _detect(x: np.ndarray, p):
    res, det, ws = g.detect_periods(_to_dev(x), p, detail=True)
    loc = g.local_scores(ws, p, x.shape[0])
    torch.cuda.synchronize()
    return g.results_numpy(res), g.detail_numpy(det), loc.cpu().numpy(), ws


def _check(x, op, got, label, ods=None, max_excluded_frac=0.1):
    """Alg. 1 records of the GPU (res, det, loc) against the oracle on x under op."""
    res, det, loc = got[:3]
    ods = ods if ods is not None else O.detect_batch(x, op)
    return PH.check_batch(x, op, res, det, loc, ods, label, max_excluded_frac)


# ---------------------------------------------------------------------------------------

@pytest.mark.parametrize("spec,idx", [(tg.CFG1, [0]), (tg.CFG2, list(range(71))),
                                      (tg.CFG3, [0, 1, 17, 9999, 99999]), (tg.CFG5, [0, 4321])])
def test_generator_bit_identical(spec, idx):
    cnt = len(idx)
    host = np.stack([tg.generate_host(spec, i, 1)[0] for i in idx])
    dev = torch.empty((cnt, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    for j, i in enumerate(idx):
        tg.generate_device(spec, dev[j:j + 1], first=i, count=1)
    torch.cuda.synchronize()
    assert np.array_equal(dev.cpu().numpy().reshape(host.shape).view(np.uint32), host.view(np.uint32))


@pytest.mark.parametrize("N,F", [(8, 1), (64, 2), (1024, 1), (1024, 3), (8192, 3), (65536, 3), (262144, 2)])
def test_composite_signal_matches_oracle(N, F):
    rng = np.random.default_rng(N + F)
    B = 3 if N <= 65536 else 1
    x = np.round(rng.uniform(0, 300, (B, F, N)) + 50 * np.sin(np.arange(N) * 0.01)).astype(np.float32)
    x[0, 0, :] = 17.0  # a constant channel contributes 0
    p = g.default_params(N, F)
    _, sig = g.power_spectrum(_to_dev(x), p)
    sig = sig.cpu().numpy()
    n_off = 0
    for b in range(B):
        y, _, _, _ = O.composite(x[b])
        diff = sig[b].view(np.int32).astype(np.int64) - y.view(np.int32).astype(np.int64)
        # the same fp64 expression rounded once (Z23) from fp64 statistics summed in another
        # order: bit-identical unless the value sits within their last-bit difference of an
        # fp32 rounding boundary -- then 1 ulp
        assert np.abs(diff).max() <= 1, np.abs(diff).max()
        n_off += np.count_nonzero(diff)
    print(f"[composite N={N} F={F}] samples={B * N} off-by-1ulp={n_off}")
    assert n_off <= max(2, B * N // 10**6)


@pytest.mark.parametrize("N", [8, 16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192, 16384, 32768, 65536])
def test_spectrum_matches_oracle_full(N):
    rng = np.random.default_rng(N)
    x = (rng.standard_normal((2, 1, N)) * 3 + np.cos(2 * np.pi * np.arange(N) * (N // 8 + 0.3) / N)).astype(np.float32)
    p = g.default_params(N, 1)
    spec, _ = g.power_spectrum(_to_dev(x), p)
    spec = spec.cpu().numpy().astype(np.float64)
    for b in range(2 if N <= 32768 else 1):
        y, _, _, _ = O.composite(x[b])
        ref = O.power_spectrum(y)
        err = np.abs(spec[b] - ref).max() / ref.max()
        assert err <= 1e-4, (N, b, err)
        assert err <= 2e-6  # fp32 FFT: typically ~1e-7


@pytest.mark.parametrize("N", [131072, 262144])
def test_spectrum_matches_oracle_sampled(N):
    # cluster FFT (4 and 8 CTAs): sampled bins computed one by one by the oracle
    rng = np.random.default_rng(N)
    x = (rng.standard_normal((1, 3, N)) * 3 + np.cos(2 * np.pi * np.arange(N) * 1234.5 / N)).astype(np.float32)
    p = g.default_params(N, 3)
    spec, _ = g.power_spectrum(_to_dev(x), p)
    spec = spec.cpu().numpy()[0].astype(np.float64)
    y, _, _, _ = O.composite(x[0])
    bins = sorted(set([0, 1, N // 2 - 1, N // 2, 1234, 1235, N // 4, N // 8 + 1] +
                      rng.integers(0, N // 2 + 1, 40).tolist()))
    ref = np.array([O.power_spectrum_bins(y, k, k)[0] for k in bins])
    pmax = O.power_spectrum_bins(y, 1234, 1235).max()
    assert np.abs(spec[bins] - ref).max() <= 1e-4 * pmax


def test_similarity_scores_match_oracle():
    x = tg.generate_host(tg.CFG2, 0, 6)
    ys = np.stack([O.composite(x[b])[0] for b in range(6)])
    rng = np.random.default_rng(0)
    Ls = sorted(set([2, 3, 5, 10, 16, 17, 31, 32, 33, 100, 255, 256, 257, 511, 512, 513, 700, 1024, 2047, 4096] +
                    rng.integers(10, 4097, 40).tolist()))
    ti = np.repeat(np.arange(6), len(Ls)).astype(np.int32)
    pe = np.tile(np.array(Ls, np.int32), 6)
    got = g.similarity_error(torch.from_numpy(ys).cuda(), ti, pe).cpu().numpy()
    bad = []
    for q in range(len(ti)):
        ref, margin = O.similarity_error(ys[ti[q]], int(pe[q]), with_margin=True)
        if margin < 1e-10:
            continue
        if abs(got[q] - ref) > 1e-4 * max(ref, 1e-6):
            bad.append((int(ti[q]), int(pe[q]), got[q], ref))
    assert not bad


@pytest.mark.parametrize("G,maxit", [(1, 32), (2, 32), (3, 5), (4, 1), (4, 2), (5, 32), (8, 32)])
def test_similarity_groups_and_caps(G, maxit):
    x = tg.generate_host(tg.CFG2, 3, 2)
    ys = np.stack([O.composite(x[b])[0] for b in range(2)])
    # team widths 1, 2, 4, 8, 16, 32 (the halving reduction runs on teams of >= pow2ceil(2G)
    # lanes, the butterfly on smaller ones) and both bucketed launches
    Ls = [7, 20, 64, 100, 200, 300, 600, 1500, 3000]
    ti = np.repeat(np.arange(2), len(Ls)).astype(np.int32)
    pe = np.tile(np.array(Ls, np.int32), 2)
    got = g.similarity_error(torch.from_numpy(ys).cuda(), ti, pe, num_groups=G, gmm_max_iters=maxit).cpu().numpy()
    for q in range(len(ti)):
        ref, margin = O.similarity_error(ys[ti[q]], int(pe[q]), G, maxit, with_margin=True)
        if margin < 1e-10:
            continue
        assert abs(got[q] - ref) <= 1e-4 * max(ref, 1e-6), (G, maxit, ti[q], pe[q], got[q], ref)
    if G == 1:
        assert (got == 0).all()


def test_similarity_long_windows_all_paths():
    # every scorer path on one signal: team (L < 513), mid bucketed (<= 2048), xl bucketed
    # (<= 8192) and the streaming warp path (L > 8192, labels in global scratch)
    x = tg.generate_host(tg.CFG2.with_(n_samples=32768, period_lo=3000.0, period_hi=9000.0), 0, 2)
    ys = np.stack([O.composite(x[b])[0] for b in range(2)])
    Ls = [100, 1200, 3000, 8192, 8193, 10000, 16384]
    ti = np.repeat(np.arange(2), len(Ls)).astype(np.int32)
    pe = np.tile(np.array(Ls, np.int32), 2)
    got = g.similarity_error(torch.from_numpy(ys).cuda(), ti, pe).cpu().numpy()
    for q in range(len(ti)):
        ref, margin = O.similarity_error(ys[ti[q]], int(pe[q]), with_margin=True)
        if margin < 1e-10:
            continue
        assert abs(got[q] - ref) <= 1e-4 * max(ref, 1e-6), (ti[q], pe[q], got[q], ref)


def test_similarity_exact_zero_on_periodic():
    rng = np.random.default_rng(5)
    rows, Ls = [], []
    for L0 in (3, 7, 40, 333, 600, 1500):
        prof = np.round(rng.uniform(0, 100, L0))
        rows.append(np.tile(prof, 8192 // L0 + 1)[:8192].astype(np.float32))
        Ls.append(L0)
    y = torch.from_numpy(np.stack(rows)).cuda()
    ti = np.concatenate([np.arange(6), np.arange(6)]).astype(np.int32)
    pe = np.array(Ls + [2 * L for L in Ls], np.int32)
    got = g.similarity_error(y, ti, pe).cpu().numpy()
    assert (got == 0.0).all()  # exactly 0 (Z28), so the (Err, L) tie-break picks the fundamental
    off = g.similarity_error(y, np.arange(6, dtype=np.int32), np.array([L + 1 for L in Ls], np.int32)).cpu().numpy()
    assert (off > 0).all()


def test_bounded_search_exact_ties_on_periodic():
    """Exactly periodic traces: Err is exactly 0 at the period and its multiples (Z28), so the
    bounded search's bound reaches 0; a query whose partial sum is still 0 must not stop (only a
    strictly larger Err may), and the tie-break to the smaller L (Z17) must hold as without it."""
    rng = np.random.default_rng(11)
    N, F = 8192, 3
    rows = []
    for L0 in (37, 120, 333, 700, 1500, 2500):
        prof = np.round(rng.uniform(0, 100, (F, L0)))
        rows.append(np.tile(prof, (1, N // L0 + 1))[:, :N].astype(np.float32))
    x = np.stack(rows)
    p1 = g.default_params(N, F, min_period=10, max_period=N // 2)
    p0 = g.default_params(N, F, min_period=10, max_period=N // 2, bounded_search=0)
    r1, d1, l1, _ = _detect(x, p1)
    r0, d0, l0, _ = _detect(x, p0)
    assert r1.tobytes() == r0.tobytes()
    ods = O.detect_batch(x, O.Params(N, F, min_period=10, max_period=N // 2))
    for i, od in enumerate(ods):
        assert r1[i]["status"] == od.status == 0 and r1[i]["period"] == od.period, (i, r1[i], od.period)
        assert (d1[i]["best_err"] == 0.0) == (od.error == 0.0), (i, d1[i]["best_err"], od.error)
    # every local L whose exhaustive Err is 0 finished with 0 (never stopped)
    zero = l0 == 0.0
    assert (l1[zero] == 0.0).all()


def test_detect_config1():
    x = tg.generate_host(tg.CFG1)
    got = _detect(x, g.params_for(tg.CFG1))
    assert got[0][0]["period"] == 37 and got[0][0]["status"] == 0
    t = _check(x, O.params_for(tg.CFG1), got, "cfg1")
    assert t.exact == 1


def test_detect_config2_all_71():
    x = tg.generate_host(tg.CFG2)
    t = _check(x, O.params_for(tg.CFG2), _detect(x, g.params_for(tg.CFG2)), "cfg2")
    assert t.exact >= 69


def test_detect_config3_shape_subset():
    spec = tg.CFG3
    idx = [0, 1, 2, 3, 5, 8, 13, 21, 34, 55, 89, 144, 233, 377, 610, 987]
    x = np.stack([tg.generate_host(spec, i, 1)[0] for i in idx])
    _check(x, O.params_for(spec, dft_band_only=True), _detect(x, g.params_for(spec)), "cfg3")


def test_detect_config5_first16():
    # BASELINE config 5 (2^18 samples, mid-trace period shift, harmonic aliasing): its first
    # 16 traces, every decision and score against the oracle (SURVEY 8(d) subset)
    spec = tg.CFG5
    x = tg.generate_host(spec, 0, 16)
    _check(x, O.params_for(spec, dft_band_only=True), _detect(x, g.params_for(spec)), "cfg5")


@pytest.mark.slow
def test_full_size_config5_sampled():
    """BASELINE.json config 5 at full size, in the launch configuration bench.py times (one call
    over 10^4 traces x 3 x 2^18 resident in HBM, bounded search on); 16 traces spread over the
    batch checked against the oracle one by one (every decision, every candidate and local
    score, stopped queries validated)."""
    spec = tg.CFG5
    B = spec.batch
    x = torch.empty((B, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    tg.generate_device(spec, x)
    p = g.params_for(spec)
    res, det, ws = g.detect_periods(x, p, detail=True)
    torch.cuda.synchronize()
    del x
    rng = np.random.default_rng(55)
    idx = sorted(set([0, B - 1] + rng.choice(np.arange(1, B - 1), 14, replace=False).tolist()))
    ti = torch.as_tensor(idx, device="cuda")
    loc = g.local_scores(ws, p, B)[ti].cpu().numpy()
    r = g.results_numpy(res)[idx]
    d = g.detail_numpy(det)[idx]
    xs = np.stack([tg.generate_host(spec, i, 1)[0] for i in idx])
    _check(xs, O.params_for(spec, dft_band_only=True), (r, d, loc), "cfg5-full")
    allr = g.results_numpy(res)
    assert (allr["status"] == 0).all()


def test_edge_cases_statuses_and_small_n():
    N = 64
    rng = np.random.default_rng(1)
    x = np.zeros((5, 2, N), np.float32)
    x[0] = 5.0                                       # constant -> CONSTANT
    x[1, 0] = np.arange(N)                           # ramp + constant channel -> APERIODIC
    x[1, 1] = 3.0
    x[2, 0] = np.tile([1, 9, 4, 4, 0, 2, 7], 10)[:N]  # period 7
    x[2, 1] = 1.0
    x[3] = np.round(rng.uniform(0, 10, (2, N)))
    x[4, 0] = np.tile([0, 10], N // 2)               # period 2 (L_min)
    x[4, 1] = np.tile([1, 3], N // 2)              # in phase (anti-phase would cancel)
    p = g.default_params(N, 2, min_period=2, max_period=32)
    got = _detect(x, p)
    res = got[0]
    assert res[0]["status"] == g.TRACE_CONSTANT and res[0]["period"] == -1
    assert res[1]["status"] == g.TRACE_APERIODIC
    assert res[2]["period"] == 7 and res[4]["period"] == 2
    _check(x, O.Params(N, 2, min_period=2, max_period=32), got, "edge")


@pytest.mark.parametrize("N", [8, 16, 32])
def test_tiny_n(N):
    rng = np.random.default_rng(N)
    x = np.round(rng.uniform(0, 50, (4, 1, N))).astype(np.float32)
    x[0, 0] = np.tile([1, 5, 2], N)[:N]
    _check(x, O.Params(N, 1), _detect(x, g.default_params(N, 1)), f"tiny{N}")


@pytest.mark.parametrize("kw", [dict(max_candidates=1), dict(num_groups=2), dict(num_groups=8), dict(gmm_max_iters=1),
                                dict(c_peak=0.3), dict(min_period=200, max_period=200), dict(weights=(1.0, 0.5, 2.0))])
def test_parameter_variants(kw):
    spec = tg.CFG2.with_(batch=12)
    x = tg.generate_host(spec)
    okw = dict(kw)
    if "min_period" not in kw:
        okw.update(min_period=spec.min_period, max_period=spec.max_period)
    got = _detect(x, g.default_params(spec.n_samples, 3, **({**dict(min_period=spec.min_period,
                                                                    max_period=spec.max_period), **kw})))
    _check(x, O.Params(spec.n_samples, 3, **okw), got, str(kw))


def test_deterministic_and_batch_order_invariant():
    spec = tg.CFG2.with_(batch=24)
    x = tg.generate_host(spec)
    # every score to the end: the debug surfaces are bit-reproducible too (with the bounded
    # search only the results are -- which queries stop depends on timing)
    p = g.params_for(spec, bounded_search=0)
    r1, d1, l1, _ = _detect(x, p)
    r2, d2, l2, _ = _detect(x, p)
    assert r1.tobytes() == r2.tobytes() and d1.tobytes() == d2.tobytes() and l1.tobytes() == l2.tobytes()
    perm = np.random.default_rng(0).permutation(24)
    r3, d3, l3, _ = _detect(x[perm], p)
    assert r3.tobytes() == r1[perm].tobytes() and d3.tobytes() == d1[perm].tobytes()
    assert l3.tobytes() == l1[perm].tobytes()


@pytest.mark.parametrize("spec,some_stop", [(tg.CFG2, True), (tg.CFG3.with_(batch=48), True),
                                            (tg.CFG5.with_(batch=4), False)])
def test_bounded_search_same_results(spec, some_stop):
    """Bounded search (gpoeo_params.bounded_search = 1, the default) against every query scored
    to the end, both on the GPU: identical result records and best_err, identical scores where
    a query finished, and every stopped query's full score strictly above its trace's winner
    (what the stop proved)."""
    x = tg.generate_host(spec)
    B = x.shape[0]
    r0, d0, l0, _ = _detect(x, g.params_for(spec, bounded_search=0))
    stopped = 0
    for rep in range(2):
        r1, d1, l1, ws = _detect(x, g.params_for(spec))
        assert r1.tobytes() == r0.tobytes(), rep
        assert d1["best_err"].tobytes() == d0["best_err"].tobytes()
        c0, c1 = d0["cand_err"], d1["cand_err"]
        cinf = np.isposinf(c1)
        assert c1[~cinf].tobytes() == c0[~cinf].tobytes()
        best_c = np.array([row[:n].min() if n else 0.0 for row, n in zip(c0, d0["n_candidates"])])
        assert (c0[cinf] > np.repeat(best_c[:, None], c0.shape[1], 1)[cinf]).all()
        fin = np.isfinite(l1) | np.isnan(l1)
        # a stopped candidate inside the local range is copied there as +inf (memoised)
        same = fin & np.isfinite(l0)
        assert l1[same].tobytes() == l0[same].tobytes()
        inf = np.isposinf(l1)
        assert (l0[inf] > np.repeat(d0["best_err"][:, None], l0.shape[1], 1)[inf]).all()
        c = g.read_counters(ws, g.params_for(spec), B)
        # stopped queries: candidates + local ones (a memoised copy is not a query)
        n_memo_inf = sum(int(np.isin(d1["cand_L"][i][:d1["n_candidates"][i]][cinf[i][:d1["n_candidates"][i]]],
                                     np.arange(d1["local_lo"][i], d1["local_hi"][i] + 1)).sum())
                         for i in range(B) if r1["status"][i] == 0)
        assert c["n_pruned_queries"] == int(cinf.sum()) + int(inf.sum()) - n_memo_inf
        stopped += int(inf.sum()) + int(cinf.sum())
    print(f"[bounded {spec.name}] stopped {stopped / 2:.0f} of {int(np.isfinite(l0).sum())} local + candidate scores per call")
    assert stopped > 0 or not some_stop  # 4 traces: every query starts before any finishes


def test_host_entry_point_matches_device():
    spec = tg.CFG2.with_(batch=40)
    x = tg.generate_host(spec)
    p = g.params_for(spec)
    r1 = _detect(x, p)[0]
    pinned = torch.from_numpy(x.reshape(40, -1)).pin_memory()
    r2 = g.detect_periods_host(pinned, p, chunk=7)
    assert r2.tobytes() == r1.tobytes()


def test_work_counters():
    spec = tg.CFG2.with_(batch=10)
    x = tg.generate_host(spec)
    p = g.params_for(spec)
    res, det, _, ws = _detect(x, p)
    c = g.read_counters(ws, p, 10)
    assert c["n_candidate_queries"] == int(det["n_candidates"][res["status"] == 0].sum())
    # local queries = the local ranges minus candidates already scored (memoised, as in the oracle)
    want = 0
    for i in np.nonzero(res["status"] == 0)[0]:
        cands = set(det["cand_L"][i][:det["n_candidates"][i]].tolist())
        want += sum(1 for L in range(det["local_lo"][i], det["local_hi"][i] + 1) if L not in cands)
    assert c["n_local_queries"] == want
    assert c["cem_sample_passes"] > 0
    assert 0 <= c["n_pruned_queries"] <= c["n_local_queries"] + c["n_candidate_queries"]


@pytest.mark.slow
def test_full_size_config3_sampled():
    """BASELINE.json config 3 at full size, in the launch configuration bench.py times
    (one call over 10^5 traces x 3 x 2^16 resident in HBM); sampled traces checked
    against the oracle one by one."""
    spec = tg.CFG3
    B = spec.batch
    x = torch.empty((B, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    tg.generate_device(spec, x)
    p = g.params_for(spec)
    res, det, ws = g.detect_periods(x, p, detail=True)
    torch.cuda.synchronize()
    del x
    # 64 traces spread over the whole 10^5 batch (first, last, and 60 seeded picks)
    rng = np.random.default_rng(2024)
    idx = sorted(set([0, 1, 99998, 99999] + rng.choice(np.arange(2, 99998), 60, replace=False).tolist()))
    ti = torch.as_tensor(idx, device="cuda")
    loc = g.local_scores(ws, p, B)[ti].cpu().numpy()
    r = g.results_numpy(res)[idx]
    d = g.detail_numpy(det)[idx]
    xs = np.stack([tg.generate_host(spec, i, 1)[0] for i in idx])
    _check(xs, O.params_for(spec, dft_band_only=True), (r, d, loc), "cfg3-full")
    allr = g.results_numpy(res)
    assert set(np.unique(allr["status"])) <= {0, 1}
    assert (allr["period"][allr["status"] == 0] >= spec.min_period).all()


def test_similarity_stress_few_levels_and_outliers():
    # NVML-like coarse quantisation (few distinct values, many exact ties), a lone outlier
    # that squeezes every other value into one bucket, and a two-level square wave
    rng = np.random.default_rng(12)
    N = 8192
    rows = [
        np.round(rng.normal(50, 1.5, N)).astype(np.float32),                       # ~10 levels
        np.where(rng.random(N) < 0.5, 3.0, 7.0).astype(np.float32),                # 2 levels
        np.concatenate([[1e4], np.round(rng.normal(20, 2, N - 1))]).astype(np.float32),  # outlier
        (np.where((np.arange(N) % 700) < 300, 10.0, 2.0) + np.round(rng.normal(0, 0.6, N))).astype(np.float32),
    ]
    y = np.stack(rows)
    Ls = [3, 16, 100, 256, 300, 512, 513, 700, 1024, 2000, 4096]
    ti = np.repeat(np.arange(len(rows)), len(Ls)).astype(np.int32)
    pe = np.tile(np.array(Ls, np.int32), len(rows))
    got = g.similarity_error(torch.from_numpy(y).cuda(), ti, pe).cpu().numpy()
    bad = []
    for q in range(len(ti)):
        ref, margin = O.similarity_error(y[ti[q]], int(pe[q]), with_margin=True)
        if margin < 1e-10:
            continue
        if abs(got[q] - ref) > 1e-4 * max(ref, 1e-6):
            bad.append((int(ti[q]), int(pe[q]), got[q], ref))
    assert not bad


# ---- spectral-only detector (oracle S1, reading R3) ------------------

def _major_compare(x, spec, label):
    p = g.params_for(spec)
    res, _ = g.detect_major_periods(_to_dev(x), p)
    torch.cuda.synchronize()
    r = g.major_numpy(res)
    op = O.params_for(spec, dft_band_only=spec.n_samples > 8192)
    ms = O.major_batch(x, op)
    n_amb = 0
    for i, m in enumerate(ms):
        assert r[i]["status"] == m.status, (label, i)
        if m.status != O.TRACE_OK:
            assert r[i]["period"] == -1 and r[i]["bin"] == -1
            continue
        if r[i]["bin"] != m.bin:
            # Z27: only a near-tie of the two largest peaks (or a peak test) may move f_major;
            # the GPU's bin must then be an in-band peak within 1e-5 P_major of the maximum on
            # the oracle's own DFT values
            assert m.ambiguous(), (label, i, r[i]["bin"], m.bin, m.d_major, m.d_peak)
            y = O.composite(x[i], weights=op.weights)[0]
            pm, pk, pp = PH._p3(y, int(r[i]["bin"]))
            eps = O.THR_SPEC * m.power
            assert pk >= m.power - eps and pk > pm - eps and pk >= pp - eps, (label, i)
            n_amb += 1
        assert r[i]["period"] == spec.n_samples // r[i]["bin"]
        assert r[i]["period_s"] == np.float32(r[i]["period"] * op.sample_interval)
    print(f"[major {label}] traces={len(ms)} justified-exclusions={n_amb}")
    assert n_amb <= max(1, len(ms) // 10), (label, n_amb)
    return r


@pytest.mark.parametrize("spec,n", [(tg.CFG1, 1), (tg.CFG2, 71), (tg.CFG3, 6), (tg.CFG5, 2)])
def test_major_matches_oracle(spec, n):
    x = tg.generate_host(spec.with_(batch=n))
    _major_compare(x, spec, spec.name)


@pytest.mark.parametrize("N,F", [(8, 1), (64, 2), (4096, 3), (65536, 1), (65536, 2), (131072, 3)])
def test_major_shapes(N, F):
    lo = 2 if N <= 8192 else N // 256  # keep the oracle's O(N * band) DFT short
    spec = tg.CFG2.with_(batch=3, n_samples=N, n_features=F, min_period=lo, max_period=N // 2)
    x = tg.generate_host(spec)
    _major_compare(x, spec, f"N{N}F{F}")


def test_major_equals_alg1_first_candidate():
    # the first-ranked Alg. 1 candidate is f_major (same peaks, same order)
    spec = tg.CFG3.with_(batch=64)
    xd = torch.empty((64, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
    tg.generate_device(spec, xd)
    p = g.params_for(spec)
    res, _ = g.detect_major_periods(xd, p)
    _, det, _ = g.detect_periods(xd, p, detail=True)
    torch.cuda.synchronize()
    r, d = g.major_numpy(res), g.detail_numpy(det)
    ok = r["status"] == 0
    assert ok.sum() > 40
    assert (r["bin"][ok] == d["cand_k"][ok, 0]).all()


def test_major_statuses():
    N = 1024
    x = np.zeros((3, 1, N), np.float32)
    x[1, 0] = np.arange(N)                          # monotone ramp: no in-band peak for [4, 16]
    x[2, 0] = np.cos(2 * np.pi * 100 * np.arange(N) / N)  # period 10: in the band [4, 16]
    spec = tg.CFG1.with_(batch=3, min_period=4, max_period=16)
    p = g.params_for(spec)
    res, _ = g.detect_major_periods(_to_dev(x), p)
    r = g.major_numpy(res)
    assert list(r["status"]) == [O.TRACE_CONSTANT, O.TRACE_APERIODIC, O.TRACE_OK]
    assert r["bin"][2] == 100 and r["period"][2] == N // 100


# ---- N not a power of two (band-limited DFT path) -------------------------------------

@pytest.mark.parametrize("N", [999, 1000, 3001, 6000])
def test_non_pow2_spectrum_matches_oracle(N):
    spec = tg.CFG2.with_(batch=2, n_samples=N, period_lo=15.0, period_hi=N / 4, min_period=2, max_period=N // 2)
    x = tg.generate_host(spec)
    p = g.params_for(spec)
    spec_d, sig = g.power_spectrum(_to_dev(x), p)
    spec_d, sig = spec_d.cpu().numpy(), sig.cpu().numpy()
    for b in range(2):
        y, _, _, _ = O.composite(x[b])
        assert (sig[b].view(np.int32) == y.view(np.int32)).all()
        ref = O.power_spectrum(y)
        assert np.abs(spec_d[b] - ref).max() <= 1e-4 * ref.max()


@pytest.mark.parametrize("N,F", [(1000, 3), (2999, 1), (5000, 3)])
def test_non_pow2_detect_matches_oracle(N, F):
    spec = tg.CFG2.with_(batch=12, n_samples=N, n_features=F, period_lo=20.0, period_hi=N / 6, min_period=10,
                         max_period=N // 3)
    x = tg.generate_host(spec)
    _check(x, O.params_for(spec), _detect(x, g.params_for(spec)), f"N{N}")
    _major_compare(x, spec, f"major-N{N}")


# ---- Alg. 3 rolling detector (oracle R1, reading R5) ------------------

def _rolling_compare(x, spec, label, weights=None):
    p = g.params_for(spec)
    if weights is not None:
        for c, v in enumerate(weights):
            p.feature_weights[c] = v
    r = g.detect_rolling(_to_dev(x), p)
    op = O.params_for(spec, dft_band_only=True, weights=weights)
    n_amb = 0
    for i in range(x.shape[0]):
        o = O.rolling(x[i], op)
        assert r[i]["status"] == o.status, (label, i)
        if o.status != O.TRACE_OK:
            assert r[i]["t_iter"] == -1
            continue
        want_next = np.float32(o.smpdur_next * 1.0) if o.smpdur_next >= 0 else np.float32(-1.0)
        got = (int(r[i]["t_init"]), bool(r[i]["early"]), int(r[i]["n_sub"]), int(r[i]["t_iter"]),
               float(r[i]["smpdur_next_s"]))
        want = (o.t_init, o.early, len(o.sub_start), o.t_iter, float(want_next))
        if got != want:
            # Z27: only a call whose oracle records a decision margin below the thresholds
            # (an ambiguous Alg. 1 on the whole trace or a suffix, a line-14 near-tie, Diff
            # at the threshold) may take another valid trajectory
            assert o.amb, (label, i, got, want, o.sub_period)
            n_amb += 1
            continue
        if np.isfinite(o.diff):
            assert abs(r[i]["diff"] - o.diff) <= 1e-6 * max(1.0, o.diff)
    print(f"[rolling {label}] traces={x.shape[0]} justified-exclusions={n_amb}")
    assert n_amb <= max(1, x.shape[0] // 5), (label, n_amb)


def test_rolling_config1():
    x = tg.generate_host(tg.CFG1)
    r = g.detect_rolling(_to_dev(x), g.params_for(tg.CFG1))
    assert r[0]["t_init"] == 37 and r[0]["t_iter"] == 37 and r[0]["n_sub"] == 7 and r[0]["smpdur_next_s"] == -1.0
    _rolling_compare(x, tg.CFG1, "cfg1")


def test_rolling_config2_slice():
    spec = tg.CFG2.with_(batch=16)
    _rolling_compare(tg.generate_host(spec), spec, "cfg2")


def test_rolling_period_shift():
    # mid-trace period change (config 5's structure at N = 8192): the suffixes see the new period
    spec = tg.CFG5.with_(batch=6, n_samples=8192, period_lo=30.0, period_hi=200.0, max_period=2048)
    _rolling_compare(tg.generate_host(spec), spec, "shift")


# ---- Alg. 4 adaptive measurement (oracle M1, reading R6) ----------------

def _measure_compare(x, spec, init, label, weights=None):
    p = g.params_for(spec)
    if weights is not None:
        for c, v in enumerate(weights):
            p.feature_weights[c] = v
    r = g.measure_adaptive(_to_dev(x), p, init)
    op = O.params_for(spec, dft_band_only=True, weights=weights)
    n_amb = 0
    for i in range(x.shape[0]):
        o = O.measure(x[i], op, init)
        got = (int(r[i]["status"]), int(r[i]["t_iter"]), int(r[i]["rounds"]), int(r[i]["samples"]),
               int(r[i]["measure_start"]), int(r[i]["measure_end"]))
        want = (o["status"], o["t_iter"], o["rounds"], o["samples"], o["measure_start"], o["measure_end"])
        if got != want:
            # Z27: a near-tie inside some round's Alg. 3 call (recorded by the oracle) may
            # legitimately change the session's trajectory; nothing else may
            assert o["amb"], (label, i, got, want)
            n_amb += 1
    print(f"[measure {label}] sessions={x.shape[0]} justified-exclusions={n_amb}")
    assert n_amb <= max(1, x.shape[0] // 5), (label, n_amb)
    return r


def test_measure_config1_and_closed_form():
    r = _measure_compare(tg.generate_host(tg.CFG1), tg.CFG1, 1024, "cfg1")
    assert (r[0]["t_iter"], r[0]["rounds"], r[0]["samples"]) == (37, 1, 1024)
    n = np.arange(2048)
    x = (np.where((n % 20) < 7, 1.0, 0.0) + 0.01 * np.sin(0.37 * n)).astype(np.float32)[None, None]
    spec = tg.CFG1.with_(n_samples=2048, min_period=4, max_period=1024)
    r = g.measure_adaptive(_to_dev(x), g.params_for(spec), 40)
    assert (r[0]["rounds"], r[0]["samples"], r[0]["t_iter"], r[0]["measure_start"]) == (2, 41, 20, 41)


def test_measure_config2_slice():
    spec = tg.CFG2.with_(batch=16)
    _measure_compare(tg.generate_host(spec), spec, 2048, "cfg2")


def test_measure_period_shift():
    spec = tg.CFG5.with_(batch=6, n_samples=8192, period_lo=30.0, period_hi=200.0, max_period=2048)
    _measure_compare(tg.generate_host(spec), spec, 2048, "shift")


# ---- gear local search (oracle G1, reading R7) ---------------------------

def test_gear_search_matches_oracle():
    rng = np.random.default_rng(3)
    sm = np.arange(510, 1966, 15, dtype=np.float64)
    mem = np.array([405.0, 810.0, 1600.0, 2619.0, 3996.0])
    n = 400
    wl = np.zeros(n, dtype=g.GEAR_WORKLOAD_DTYPE)
    wl["compute_work"] = rng.uniform(0.5e9, 3e9, n)
    wl["memory_work"] = np.where(rng.random(n) < 0.5, 1e6, rng.uniform(0.5e9, 3e9, n))
    wl["overhead"] = rng.uniform(0.01, 0.1, n)
    wl["p_static"] = rng.uniform(60, 150, n)
    wl["c_sm"] = rng.uniform(2e-4, 1e-3, n)
    wl["c_mem"] = rng.uniform(0.005, 0.03, n)
    wl["u_c"] = rng.uniform(0.2, 1.0, n)
    wl["u_m"] = rng.uniform(0.2, 1.0, n)
    wl["noise"] = np.where(rng.random(n) < 0.5, 0.0, 0.01)
    wl["seed"] = rng.integers(0, 1 << 62, n, dtype=np.uint64)
    ps = rng.integers(0, len(sm), n).astype(np.int32)
    pm = rng.integers(0, len(mem), n).astype(np.int32)
    r = g.gear_search(wl, sm, mem, 0.05, ps, pm)
    n_amb = 0
    for i in range(n):
        w = O.gear_workload(**{k: (int(wl[k][i]) if k == "seed" else float(wl[k][i])) for k in wl.dtype.names})
        o = O.gear_search(w, sm, mem, 0.05, int(ps[i]), int(pm[i]))
        got = (int(r[i]["sm_gear"]), int(r[i]["mem_gear"]), int(r[i]["probes_sm"]), int(r[i]["probes_mem"]))
        if got != (o["sm_gear"], o["mem_gear"], o["probes_sm"], o["probes_mem"]):
            # Z27: the two sides' pow() differ in the last ulps (CUDA libdevice vs glibc), so only
            # a search decision the oracle took on a relative margin below 1e-12 (two objective
            # values, or the fitted curvature's sign) or a vertex within 1e-9 of a rounding
            # boundary may go the other way
            assert o["margin_rel"] < 1e-12 or o["margin_round"] < 1e-9, (i, got, o)
            n_amb += 1
            continue
        assert abs(r[i]["objective"] - o["objective"]) <= 1e-12 * abs(o["objective"])
    print(f"[gear] workloads={n} justified-exclusions={n_amb}")
    assert n_amb <= 4, n_amb


def test_rolling_and_measure_non_pow2_weighted():
    # N not a power of two, three channels with unequal weights (Z1): Alg. 3 and Alg. 4
    spec = tg.CFG2.with_(batch=8, n_samples=3000, period_lo=20.0, period_hi=300.0, min_period=10, max_period=1000)
    x = tg.generate_host(spec)
    w = (1.0, 0.5, 2.0)
    _rolling_compare(x, spec, "non-pow2-weighted", weights=w)
    _measure_compare(x, spec, 600, "non-pow2-weighted", weights=w)


def test_measure_prefix_lengths_not_multiple_of_4():
    # ragged Alg. 4 prefixes whose channel stride (the recording length, 3001) is not a
    # multiple of 4 while some prefix lengths are: the composite must not take the 128-bit
    # path on misaligned rows
    spec = tg.CFG2.with_(batch=6, n_samples=3001, period_lo=20.0, period_hi=300.0, min_period=10, max_period=1000)
    x = tg.generate_host(spec)
    _measure_compare(x, spec, 600, "n3001")


def test_rolling_n_not_multiple_of_4_large_batch():
    # suffix chunks of a recording whose length is not a multiple of 4, at a batch large
    # enough that the chunk layout used to outgrow its workspace section
    spec = tg.CFG2.with_(batch=40, n_samples=2049, period_lo=20.0, period_hi=200.0, min_period=10, max_period=1024)
    _rolling_compare(tg.generate_host(spec), spec, "n2049-b40")


def test_sharded_detect_nccl_world1():
    # row e on the device: shard.detect_sharded through a real NCCL process group (world 1 on
    # the one GPU a test box has): the all-gathered records equal the unsharded call's bytes
    import os
    import socket

    import torch.distributed as dist

    from paper_2201_01684_b200 import shard

    spec = tg.CFG2.with_(batch=12)
    x = tg.generate_host(spec)
    p = g.params_for(spec)
    r1 = _detect(x, p)[0]
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        out, _ = shard.detect_sharded(_to_dev(x), spec.batch, p)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == r1.tobytes()
        # config 4's streamed shard: the same traces through a 5-trace resident buffer in
        # chunks (generated on the device per chunk), then the all-gather
        xb = torch.empty((5, spec.n_features * spec.n_samples), dtype=torch.float32, device="cuda")
        res = torch.empty(spec.batch * shard.RESULT_BYTES, dtype=torch.uint8, device="cuda")
        shard.detect_shard_chunked(lambda xv, f, n: tg.generate_device(spec, xv, first=f, count=n), 0, spec.batch,
                                   5, p, xb, res)
        out2 = shard.gather_results(res, spec.batch)
        torch.cuda.synchronize()
        assert out2.cpu().numpy().tobytes() == r1.tobytes()
    finally:
        dist.destroy_process_group()


def test_measure_empty_band_prefix():
    # the first prefix's band is empty (L_max clipped to 2500 < L_min = 3000): INSUFFICIENT,
    # without the band DFT writing past its shared-memory slots
    spec = tg.CFG2.with_(batch=3, n_samples=20000, period_lo=3200.0, period_hi=4000.0, min_period=3000,
                         max_period=10000)
    r = _measure_compare(tg.generate_host(spec), spec, 5000, "empty-band")
    assert (r["status"] == O.TRACE_INSUFFICIENT).all() and (r["rounds"] == 1).all()
