"""Parity harness: the CUDA path's Alg. 1 records against the oracle, element by element.

Bars (BASELINE.json north star):
  * statuses, candidate lists, best bins, local ranges, detected periods: bit-exact;
  * Alg. 2 scores, every candidate and every local L: |Err_gpu - Err_ref| <= 1e-4 max(Err_ref, 1e-6)
    (Z30);
  * period_s exact.
Z27 (several correct results): a decision may differ only where the oracle records a margin
below what the precision difference between the two sides can move (oracle.THR_*), and then
the GPU's outcome is checked for validity against the oracle itself:
  * a different candidate list: every differing bin (and every reordered pair) must sit within
    THR_SPEC * P_max of the threshold, of a neighbour (the peak test) or of another candidate's
    power (rank / dedupe order) -- checked on the oracle's own DFT values at those bins -- and
    the rest of Alg. 1 is then compared exactly against the oracle run from line 6 on the GPU's
    list (oracle.detect(given_k=...));
  * a single Alg. 2 score off by more than the tolerance: the oracle's CEM decision margin of
    that query must be < THR_CEM (a partition flip at rounding level);
  * a query the bounded search stopped (score +inf): that candidate / L must not be the oracle's
    argmin (unless another one ties it within THR_ERR);
  * a different Tcand_opt or final L: the oracle's Err of the GPU's choice must be within THR_ERR
    (relative) of its best, or one of the two scores involved must be a flipped query; a
    different Tcand_opt is then followed by the oracle forced to the GPU's bin
    (oracle.detect(force_kb=...)) and compared exactly from line 11 on.
Every exclusion is recorded with its reason; callers print the counts.
"""
from __future__ import annotations

import numpy as np

import oracle as O

TOL = 1e-4


def _close(a: float, b: float) -> bool:
    return abs(a - b) <= TOL * max(b, 1e-6)


def _rel_gap(a: float, b: float) -> float:
    return abs(a - b) / max(min(a, b), 1e-12)


class Tally:
    def __init__(self, label: str):
        self.label = label
        self.n = 0
        self.exact = 0
        self.reasons: dict[str, int] = {}
        self.stopped = 0  # Alg. 2 queries the bounded search stopped (score +inf), each checked

    def note(self, reason: str):
        self.reasons[reason] = self.reasons.get(reason, 0) + 1

    def summary(self) -> str:
        return (f"[parity {self.label}] traces={self.n} exact={self.exact} justified-exclusions={self.reasons} "
                f"stopped-queries={self.stopped}")


def _p3(y, k: int):
    """(P[k-1], P[k], P[k+1]) by the oracle's DFT, mirrored at the edges (Z5)."""
    n2 = y.size // 2

    def m(j):
        j = abs(j)
        return y.size - j if j > n2 else j
    return [O.power_spectrum_bins(y, m(j), m(j))[0] for j in (k - 1, k, k + 1)]


def _spectral_diff_is_near_boundary(x, op: O.Params, d: O.Detection, gpu_k: list) -> bool:
    """Every bin in which the two candidate lists differ, and every pair they order
    differently, sits within THR_SPEC * P_max of a decision boundary of Alg. 1 l.3-5
    (threshold, peak test, rank/dedupe order), on the oracle's own DFT values."""
    y = O.composite(x, weights=op.weights)[0]
    pmax = d.cand_P[0]
    thr = float(np.float32(op.c_peak)) ** 2 * pmax
    eps = O.THR_SPEC * pmax
    union = sorted(set(gpu_k) | set(d.cand_k))
    P = {k: _p3(y, k) for k in union}
    diff = set(gpu_k) ^ set(d.cand_k)
    for k in diff:
        pk = P[k][1]
        near = abs(pk - thr) < eps or abs(pk - P[k][0]) < eps or abs(pk - P[k][2]) < eps
        near = near or any(j != k and abs(pk - P[j][1]) < eps for j in union)
        if not near:
            return False
    common = [k for k in gpu_k if k in d.cand_k]
    for a in range(len(common)):
        for b in range(a + 1, len(common)):
            ka, kb = common[a], common[b]
            if (d.cand_k.index(ka) < d.cand_k.index(kb)) != (gpu_k.index(ka) < gpu_k.index(kb)):
                if abs(P[ka][1] - P[kb][1]) >= eps:
                    return False
    return True


def check_trace(x, op: O.Params, r, q, gl, d: O.Detection, tally: Tally, where=""):
    """One trace: r = RESULT_DTYPE record, q = DETAIL_DTYPE record, gl = the GPU's local
    scores row (or None), d = the oracle's Detection of x under op."""
    tally.n += 1
    tag = (tally.label, where)
    assert r["status"] == d.status, (tag, "status", r["status"], d.status)
    if d.status == O.TRACE_CONSTANT:
        tally.exact += 1
        return
    if d.status != O.TRACE_OK:
        assert r["n_candidates"] == 0 and r["period"] == -1, tag
        tally.exact += 1
        return
    excluded = []
    nc = int(q["n_candidates"])
    gpu_k = [int(k) for k in q["cand_k"][:nc]]
    ref = d
    if gpu_k != d.cand_k:
        reasons = [m for m in ("d_thr", "d_peak", "d_rank", "d_order") if d.margins[m] < O.THR_SPEC]
        assert reasons, (tag, "candidate lists differ with no spectral margin", gpu_k, d.cand_k, d.margins)
        assert _spectral_diff_is_near_boundary(x, op, d, gpu_k), (tag, "differing bins not near a boundary", gpu_k,
                                                                   d.cand_k)
        excluded.append("spectral:" + "+".join(reasons))
        ref = O.detect(x, op, given_k=gpu_k)
    assert [int(v) for v in q["cand_L"][:nc]] == ref.cand_L, tag
    # Alg. 2 on every candidate
    flipped_c = set()
    ib = ref.cand_k.index(ref.best_bin)
    for c in range(nc):
        if np.isposinf(q["cand_err"][c]):
            # bounded search stopped this candidate: not the oracle's best either (up to a near-tie)
            if c == ib:
                others = [e for j, e in enumerate(ref.cand_err) if j != c]
                ok = bool(others) and _rel_gap(min(others), ref.cand_err[c]) < O.THR_ERR
                assert ok, (tag, "stopped candidate is the oracle's best", c, ref.cand_err)
                excluded.append("err-tie:stopped-candidate")
            tally.stopped += 1
            continue
        if not _close(q["cand_err"][c], ref.cand_err[c]):
            assert ref.cand_margin[c] < O.THR_CEM, (tag, "candidate score", c, q["cand_err"][c], ref.cand_err[c],
                                                    ref.cand_margin[c])
            flipped_c.add(c)
            excluded.append("cem-flip:candidate")
    # Tcand_opt (Alg. 1 l.9-10)
    if int(q["best_bin"]) != ref.best_bin:
        ig = gpu_k.index(int(q["best_bin"]))
        io = ref.cand_k.index(ref.best_bin)
        ok = _rel_gap(ref.cand_err[ig], ref.cand_err[io]) < O.THR_ERR or ig in flipped_c or io in flipped_c
        assert ok, (tag, "best candidate", q["best_bin"], ref.best_bin, ref.cand_err)
        excluded.append("err-tie:candidate" if not (flipped_c & {ig, io}) else "cem-flip:best-candidate")
        ref = O.detect(x, op, given_k=gpu_k, force_kb=int(q["best_bin"]))
    assert (int(q["local_lo"]), int(q["local_hi"])) == (ref.local_lo, ref.local_hi), tag
    assert r["best_candidate"] == ref.best_candidate, tag
    # Alg. 2 on every local L (Alg. 1 l.14-16)
    flipped_l = set()
    if gl is not None:
        n_loc = ref.local_hi - ref.local_lo + 1
        assert np.isnan(gl[n_loc:]).all(), tag
        io = ref.period - ref.local_lo
        for i in range(n_loc):
            if np.isposinf(gl[i]):
                # bounded search stopped this L: the GPU proved Err(L) > an Err another L of the
                # trace reached, so L is not the argmin -- on the oracle's scores it must not be
                # either (up to a near-tie, Z27)
                if i == io:
                    others = [e for j, e in enumerate(ref.local_err) if j != i]
                    ok = bool(others) and _rel_gap(min(others), ref.error) < O.THR_ERR
                    assert ok, (tag, "stopped L is the oracle's argmin", ref.local_lo + i, ref.local_err[i])
                    excluded.append("err-tie:stopped")
                tally.stopped += 1
                continue
            if not _close(gl[i], ref.local_err[i]):
                assert ref.local_margin[i] < O.THR_CEM, (tag, "local score", ref.local_lo + i, gl[i], ref.local_err[i],
                                                         ref.local_margin[i])
                flipped_l.add(i)
                excluded.append("cem-flip:local")
    # final argmin (Alg. 1 l.18)
    if r["period"] != ref.period:
        ig, io = int(r["period"]) - ref.local_lo, ref.period - ref.local_lo
        assert 0 <= ig < len(ref.local_err), (tag, "period outside the local range", r["period"])
        ok = _rel_gap(ref.local_err[ig], ref.local_err[io]) < O.THR_ERR or ig in flipped_l or io in flipped_l
        assert ok, (tag, "final period", r["period"], ref.period, ref.local_err[ig], ref.local_err[io])
        excluded.append("err-tie:local" if not (flipped_l & {ig, io}) else "cem-flip:period")
    else:
        i = ref.period - ref.local_lo
        if i not in flipped_l:
            assert _close(q["best_err"], ref.error), (tag, q["best_err"], ref.error)
    assert r["period_s"] == np.float32(r["period"] * op.sample_interval), tag
    if excluded:
        for e in sorted(set(excluded)):
            tally.note(e)
    else:
        tally.exact += 1


def check_batch(xs, op: O.Params, res, det, loc, ods, label: str, max_excluded_frac=0.1) -> Tally:
    tally = Tally(label)
    for i, d in enumerate(ods):
        check_trace(xs[i], op, res[i], det[i], None if loc is None else loc[i], d, tally, where=i)
    n_ex = tally.n - tally.exact
    print(tally.summary())
    assert n_ex <= max(1, int(max_excluded_frac * tally.n)), tally.summary()
    return tally
