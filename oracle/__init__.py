"""ctypes front-end to the plain-C fp64 oracle (oracle/gpoeo_oracle.c).

TEST INFRASTRUCTURE ONLY: tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package; the product path
(paper_2201_01684_b200) must not and does not. It shares no code with the CUDA path;
only the seeded input generator (tracegen/) serves both sides.

Citations: P:n = PAPER.md line n (Alg. 1, Alg. 2). Readings Z1..Z30
are listed in DESIGN.md. Pins live in tests/test_oracle_*.py. Parity unpinned (a
reading, no worked example in the paper): the CEM variant of "Gauss" (Z12) and the
composite rule (Z1).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "gpoeo_oracle.c")
_SO = os.path.join(_HERE, "liboracle.so")

TRACE_OK, TRACE_APERIODIC, TRACE_INSUFFICIENT, TRACE_CONSTANT, TRACE_UNSTABLE = 0, 1, 2, 3, 4

# Z27 thresholds (the same numbers as oracle_ambiguous() in gpoeo_oracle.c): a
# decision margin below these has several correct outcomes -- spectral decisions relative to
# P_max (fp32 FFT vs fp64 DFT), Err comparisons relative (reordered fp64 sums), CEM decisions
# relative to the score magnitude
THR_SPEC, THR_ERR, THR_CEM = 1e-5, 1e-9, 1e-10


class OrParams(ctypes.Structure):
    _fields_ = [
        ("n_samples", ctypes.c_int32),
        ("n_features", ctypes.c_int32),
        ("sample_interval", ctypes.c_double),
        ("min_period", ctypes.c_int32),
        ("max_period", ctypes.c_int32),
        ("c_peak", ctypes.c_double),
        ("max_candidates", ctypes.c_int32),
        ("num_groups", ctypes.c_int32),
        ("gmm_max_iters", ctypes.c_int32),
        ("dft_band_only", ctypes.c_int32),
    ]


class OrResult(ctypes.Structure):
    _fields_ = [
        ("status", ctypes.c_int32),
        ("period", ctypes.c_int32),
        ("period_s", ctypes.c_double),
        ("error", ctypes.c_double),
        ("best_candidate", ctypes.c_int32),
        ("best_bin", ctypes.c_int32),
        ("n_candidates", ctypes.c_int32),
        ("n_peaks", ctypes.c_int32),
        ("n_passing", ctypes.c_int32),
        ("cap_binds", ctypes.c_int32),
        ("cand_k", ctypes.c_int32 * 32),
        ("cand_L", ctypes.c_int32 * 32),
        ("cand_P", ctypes.c_double * 32),
        ("cand_err", ctypes.c_double * 32),
        ("local_lo", ctypes.c_int32),
        ("local_hi", ctypes.c_int32),
        ("p_max", ctypes.c_double),
        ("d_thr", ctypes.c_double),
        ("d_peak", ctypes.c_double),
        ("d_rank", ctypes.c_double),
        ("d_err_cand", ctypes.c_double),
        ("d_err_local", ctypes.c_double),
        ("d_cem", ctypes.c_double),
        ("n_queries", ctypes.c_int64),
        ("samples_clustered", ctypes.c_int64),
        ("cem_sample_iters", ctypes.c_int64),
        ("d_order", ctypes.c_double),
        ("cand_margin", ctypes.c_double * 32),
    ]


class OrMajor(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("period", ctypes.c_int32), ("bin", ctypes.c_int32),
                ("n_peaks", ctypes.c_int32), ("period_s", ctypes.c_double), ("power", ctypes.c_double),
                ("d_major", ctypes.c_double), ("d_peak", ctypes.c_double)]


class OrRolling(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("t_init", ctypes.c_int32), ("t_iter", ctypes.c_int32),
                ("n_sub", ctypes.c_int32), ("early", ctypes.c_int32), ("amb", ctypes.c_int32),
                ("err_init", ctypes.c_double), ("err_iter", ctypes.c_double), ("diff", ctypes.c_double),
                ("smpdur_next", ctypes.c_double), ("sub_start", ctypes.c_int32 * 64),
                ("sub_period", ctypes.c_int32 * 64), ("sub_err", ctypes.c_double * 64)]


class OrMeasure(ctypes.Structure):
    _fields_ = [("status", ctypes.c_int32), ("t_iter", ctypes.c_int32), ("rounds", ctypes.c_int32),
                ("samples", ctypes.c_int32), ("measure_start", ctypes.c_int32), ("measure_end", ctypes.c_int32),
                ("amb", ctypes.c_int32), ("pad", ctypes.c_int32), ("err_iter", ctypes.c_double)]


class OrGearWorkload(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("compute_work", "memory_work", "overhead", "p_static", "c_sm",
                                                 "c_mem", "u_c", "u_m", "noise")] + [("seed", ctypes.c_uint64)]


class OrGearResult(ctypes.Structure):
    _fields_ = [("sm_gear", ctypes.c_int32), ("mem_gear", ctypes.c_int32), ("probes_sm", ctypes.c_int32),
                ("probes_mem", ctypes.c_int32), ("objective", ctypes.c_double), ("margin_rel", ctypes.c_double),
                ("margin_round", ctypes.c_double)]


def build() -> str:
    """Compile the oracle (gcc, fp64, no FMA contraction). Building the checker is not using it."""
    if not (os.path.exists(_SO) and os.path.getmtime(_SO) >= os.path.getmtime(_SRC)):
        tmp = f"{_SO}.{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)  # atomic: a concurrent loader never sees a partial file
    return _SO


_lib = None
_lock = threading.Lock()


def _L():
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        return _load_locked()


def _load_locked():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        lib.oracle_composite.argtypes = [P, ctypes.c_int32, ctypes.c_int32, P, P, P, P]
        lib.oracle_composite.restype = ctypes.c_int
        lib.oracle_power_spectrum.argtypes = [P, ctypes.c_int32, P]
        lib.oracle_power_spectrum.restype = ctypes.c_int
        lib.oracle_power_spectrum_range.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P]
        lib.oracle_power_spectrum_range.restype = ctypes.c_int
        lib.oracle_smape.argtypes = [ctypes.c_double, ctypes.c_double]
        lib.oracle_smape.restype = ctypes.c_double
        lib.oracle_gmm_cem.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
        lib.oracle_gmm_cem.restype = ctypes.c_int
        lib.oracle_similarity_error.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, P, P]
        lib.oracle_similarity_error.restype = ctypes.c_double
        lib.oracle_candidates.argtypes = [P, ctypes.POINTER(OrParams), ctypes.POINTER(OrResult)]
        lib.oracle_candidates.restype = ctypes.c_int
        lib.oracle_local_range.argtypes = [ctypes.c_int32] * 4 + [ctypes.POINTER(ctypes.c_int32)] * 2
        lib.oracle_local_range.restype = None
        lib.oracle_detect.argtypes = [P, ctypes.POINTER(OrParams), P, ctypes.POINTER(OrResult), P]
        lib.oracle_detect.restype = ctypes.c_int
        lib.oracle_detect_ex.argtypes = [P, ctypes.POINTER(OrParams), P, ctypes.c_int32, P, ctypes.c_int32,
                                         ctypes.POINTER(OrResult), P, P]
        lib.oracle_detect_ex.restype = ctypes.c_int
        lib.oracle_ambiguous.argtypes = [ctypes.POINTER(OrResult)]
        lib.oracle_ambiguous.restype = ctypes.c_int
        lib.oracle_exhaustive.argtypes = [P, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
                                          ctypes.c_int32, P]
        lib.oracle_exhaustive.restype = ctypes.c_int32
        lib.oracle_major.argtypes = [P, ctypes.POINTER(OrParams), P, ctypes.POINTER(OrMajor)]
        lib.oracle_major.restype = ctypes.c_int
        assert lib.oracle_sizeof_major() == ctypes.sizeof(OrMajor)
        lib.oracle_rolling.argtypes = [P, ctypes.POINTER(OrParams), P, ctypes.c_double, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.POINTER(OrRolling)]
        lib.oracle_rolling.restype = ctypes.c_int
        assert lib.oracle_sizeof_rolling() == ctypes.sizeof(OrRolling)
        lib.oracle_measure.argtypes = [P, ctypes.POINTER(OrParams), P, ctypes.c_int32, ctypes.c_double,
                                       ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.POINTER(OrMeasure)]
        lib.oracle_measure.restype = ctypes.c_int
        assert lib.oracle_sizeof_measure() == ctypes.sizeof(OrMeasure)
        lib.oracle_gear_objective.argtypes = [ctypes.POINTER(OrGearWorkload), P, ctypes.c_int32, P, ctypes.c_int32,
                                              ctypes.c_double, ctypes.c_int32, ctypes.c_int32]
        lib.oracle_gear_objective.restype = ctypes.c_double
        lib.oracle_gear_search.argtypes = [ctypes.POINTER(OrGearWorkload), P, ctypes.c_int32, P, ctypes.c_int32,
                                           ctypes.c_double, ctypes.c_int32, ctypes.c_int32,
                                           ctypes.POINTER(OrGearResult)]
        lib.oracle_gear_search.restype = ctypes.c_int
        assert lib.oracle_sizeof_gear() == ctypes.sizeof(OrGearWorkload) * 1000 + ctypes.sizeof(OrGearResult)
        assert lib.oracle_sizeof_params() == ctypes.sizeof(OrParams)
        assert lib.oracle_sizeof_result() == ctypes.sizeof(OrResult)
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data)


@dataclass
class Params:
    """Alg. 1/2 parameters (defaults: c_peak 0.65 P:298/Z6, K 16 Z8, NumG 4 Z12, CEM cap 32 Z12)."""

    n_samples: int
    n_features: int = 1
    sample_interval: float = 1.0
    min_period: int = 2
    max_period: int = 0
    c_peak: float = 0.65
    max_candidates: int = 16
    num_groups: int = 4
    gmm_max_iters: int = 32
    weights: tuple | None = None
    dft_band_only: bool = False

    def c(self) -> OrParams:
        p = OrParams()
        p.n_samples = self.n_samples
        p.n_features = self.n_features
        p.sample_interval = self.sample_interval
        p.min_period = self.min_period
        p.max_period = self.max_period or self.n_samples // 2
        # the GPU ABI carries c_peak as fp32: use the same value
        p.c_peak = float(np.float32(self.c_peak))
        p.max_candidates = self.max_candidates
        p.num_groups = self.num_groups
        p.gmm_max_iters = self.gmm_max_iters
        p.dft_band_only = int(self.dft_band_only)
        return p


def params_for(spec, **kw) -> Params:
    """Params for a tracegen.TraceSpec (bounds per Z21)."""
    return Params(n_samples=spec.n_samples, n_features=spec.n_features, min_period=spec.min_period,
                  max_period=spec.max_period, **kw)


def composite(x: np.ndarray, weights=None):
    """O1: x float32 [F][N] -> (y float32 [N], mu [F], sigma [F], constant)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    F, N = x.shape
    y = np.empty(N, np.float32)
    mu = np.empty(F)
    sg = np.empty(F)
    w = None if weights is None else np.ascontiguousarray(weights, dtype=np.float64)
    c = _L().oracle_composite(_ptr(x), N, F, None if w is None else _ptr(w), _ptr(y), _ptr(mu), _ptr(sg))
    return y, mu, sg, bool(c)


def power_spectrum(y: np.ndarray) -> np.ndarray:
    """O2: naive DFT power spectrum P[0..N/2] (fp64)."""
    y = np.ascontiguousarray(y, dtype=np.float32)
    P = np.empty(y.size // 2 + 1)
    if _L().oracle_power_spectrum(_ptr(y), y.size, _ptr(P)) != 0:
        raise MemoryError
    return P


def power_spectrum_bins(y: np.ndarray, k0: int, k1: int) -> np.ndarray:
    """O2 at bins k0..k1 only (same arithmetic per bin); returns P[k0..k1]."""
    y = np.ascontiguousarray(y, dtype=np.float32)
    P = np.full(y.size // 2 + 1, np.nan)
    if _L().oracle_power_spectrum_range(_ptr(y), y.size, k0, k1, _ptr(P)) != 0:
        raise MemoryError
    return P[k0:k1 + 1].copy()


def smape(a: float, b: float) -> float:
    return _L().oracle_smape(a, b)


def gmm_cem(v: np.ndarray, num_groups: int = 4, max_iters: int = 32):
    """CEM 1-D GMM (Z12): -> (labels uint8, passes, min decision margin)."""
    v = np.ascontiguousarray(v, dtype=np.float32)
    lab = np.empty(v.size, np.uint8)
    m = ctypes.c_double(np.inf)
    it = _L().oracle_gmm_cem(_ptr(v), v.size, num_groups, max_iters, _ptr(lab), ctypes.byref(m))
    return lab, it, m.value


def similarity_error(y: np.ndarray, L: int, num_groups: int = 4, max_iters: int = 32, with_margin=False):
    """Alg. 2 Err(L) on signal y."""
    y = np.ascontiguousarray(y, dtype=np.float32)
    m = ctypes.c_double(np.inf)
    e = _L().oracle_similarity_error(_ptr(y), y.size, L, num_groups, max_iters, ctypes.byref(m), None)
    return (e, m.value) if with_margin else e


def candidates(P: np.ndarray, params: Params) -> OrResult:
    P = np.ascontiguousarray(P, dtype=np.float64)
    r = OrResult()
    _L().oracle_candidates(_ptr(P), ctypes.byref(params.c()), ctypes.byref(r))
    return r


def local_range(N: int, k_b: int, min_period: int, max_period: int):
    lo, hi = ctypes.c_int32(), ctypes.c_int32()
    _L().oracle_local_range(N, k_b, min_period, max_period, ctypes.byref(lo), ctypes.byref(hi))
    return lo.value, hi.value


@dataclass
class Detection:
    status: int
    period: int
    period_s: float
    error: float
    best_candidate: int
    best_bin: int
    n_candidates: int
    cand_k: list
    cand_L: list
    cand_err: list
    cand_P: list
    local_lo: int
    local_hi: int
    local_err: np.ndarray
    margins: dict = field(default_factory=dict)
    cand_margin: list = field(default_factory=list)
    local_margin: np.ndarray | None = None
    counters: dict = field(default_factory=dict)
    n_peaks: int = 0
    n_passing: int = 0
    cap_binds: bool = False

    def ambiguous(self, thr_spec=THR_SPEC, thr_err=THR_ERR, thr_cem=THR_CEM) -> bool:
        """Z27: several results are correct when a decision's margin is below what the
        precision difference between the two sides can move (fp32 spectrum vs fp64 DFT;
        reordered fp64 sums)."""
        return bool(self.amb_reasons(thr_spec, thr_err, thr_cem))

    def amb_reasons(self, thr_spec=THR_SPEC, thr_err=THR_ERR, thr_cem=THR_CEM) -> list:
        """The Z27 margins below their thresholds (spectral: of P_max; err: relative; cem:
        relative CEM score gap), by name."""
        m = self.margins
        th = dict(d_thr=thr_spec, d_peak=thr_spec, d_rank=thr_spec, d_order=thr_spec, d_err_cand=thr_err,
                  d_err_local=thr_err, d_cem=thr_cem)
        return [k for k, t in th.items() if m[k] < t]


def detect(x: np.ndarray, params: Params, given_k=None, force_kb: int = -1) -> Detection:
    """Alg. 1 on one trace x float32 [F][N].

    Test hooks of the parity harness (oracle_detect_ex): given_k = a candidate bin list to use
    instead of O2-O3 (Alg. 1 from line 6 on another side's candidates); force_kb = the bin to
    take as Tcand_opt instead of the argmin."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    p = params.c()
    r = OrResult()
    le = np.full(max(1, p.max_period - p.min_period + 1), np.nan)
    lm = np.full(le.size, np.nan)
    # the ABI carries w_c as fp32: use the same values
    w = None if params.weights is None else np.asarray(params.weights, np.float32).astype(np.float64)
    gk = None if given_k is None else np.ascontiguousarray(given_k, np.int32)
    rc = _L().oracle_detect_ex(_ptr(x), ctypes.byref(p), None if w is None else _ptr(w),
                               -1 if gk is None else gk.size, None if gk is None else _ptr(gk), int(force_kb),
                               ctypes.byref(r), _ptr(le), _ptr(lm))
    if rc != 0:
        raise ValueError(f"oracle_detect_ex: rc {rc}")
    nc = r.n_candidates
    nloc = (r.local_hi - r.local_lo + 1) if r.status == TRACE_OK else 0
    return Detection(
        status=r.status, period=r.period, period_s=r.period_s, error=r.error,
        best_candidate=r.best_candidate, best_bin=r.best_bin, n_candidates=nc,
        cand_k=list(r.cand_k[:nc]), cand_L=list(r.cand_L[:nc]), cand_err=list(r.cand_err[:nc]),
        cand_P=list(r.cand_P[:nc]), local_lo=r.local_lo, local_hi=r.local_hi, local_err=le[:nloc].copy(),
        margins=dict(d_thr=r.d_thr, d_peak=r.d_peak, d_rank=r.d_rank, d_order=r.d_order, d_err_cand=r.d_err_cand,
                     d_err_local=r.d_err_local, d_cem=r.d_cem),
        cand_margin=list(r.cand_margin[:nc]), local_margin=lm[:nloc].copy(),
        counters=dict(n_queries=r.n_queries, samples_clustered=r.samples_clustered,
                      cem_sample_iters=r.cem_sample_iters),
        n_peaks=r.n_peaks, n_passing=r.n_passing, cap_binds=bool(r.cap_binds))


def detect_batch(X: np.ndarray, params: Params, threads: int | None = None) -> list[Detection]:
    """Alg. 1 over X float32 [B][F][N] with a thread pool (ctypes releases the GIL)."""
    threads = threads or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda b: detect(X[b], params), range(X.shape[0])))


def exhaustive(y: np.ndarray, min_period: int, max_period: int, num_groups: int = 4, max_iters: int = 32):
    """O9: global argmin (Err, L) over every L in [min_period, max_period]; -> (L, errs)."""
    y = np.ascontiguousarray(y, dtype=np.float32)
    errs = np.empty(max_period - min_period + 1)
    L = _L().oracle_exhaustive(_ptr(y), y.size, min_period, max_period, num_groups, max_iters, _ptr(errs))
    return L, errs


@dataclass
class Major:
    """S1 spectral-only result (T_iter = 1/f_major; reading R3)."""
    status: int
    period: int
    bin: int
    period_s: float
    power: float
    n_peaks: int
    d_major: float
    d_peak: float

    def ambiguous(self, thr_spec=THR_SPEC) -> bool:
        """Z27: the fp32 FFT may order two peaks within thr_spec of P_major either way."""
        return self.d_major < thr_spec or self.d_peak < thr_spec


def major(x: np.ndarray, params: Params) -> Major:
    """S1 on one trace x float32 [F][N]."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    p = params.c()
    m = OrMajor()
    w = None if params.weights is None else np.asarray(params.weights, np.float32).astype(np.float64)
    if _L().oracle_major(_ptr(x), ctypes.byref(p), None if w is None else _ptr(w), ctypes.byref(m)) != 0:
        raise ValueError("oracle_major: invalid parameters")
    return Major(status=m.status, period=m.period, bin=m.bin, period_s=m.period_s, power=m.power,
                 n_peaks=m.n_peaks, d_major=m.d_major, d_peak=m.d_peak)


def major_batch(X: np.ndarray, params: Params, threads: int | None = None) -> list[Major]:
    threads = threads or os.cpu_count() or 1
    with ThreadPoolExecutor(max_workers=threads) as ex:
        return list(ex.map(lambda b: major(X[b], params), range(X.shape[0])))


@dataclass
class Rolling:
    """R1: Alg. 3 on one recorded trace (reading R5). Periods in samples."""
    status: int
    t_init: int
    t_iter: int
    early: bool
    diff: float
    smpdur_next: float
    sub_start: list
    sub_period: list
    sub_err: list
    amb: bool = False  # Z27: some decision of the call had several correct outcomes


def rolling(x: np.ndarray, params: Params, c_measure: float = 2.0, step: float = 0.5, c_eval: float = 6.5,
            diff_threshold: float = 0.05) -> Rolling:
    x = np.ascontiguousarray(x, dtype=np.float32)
    p = params.c()
    r = OrRolling()
    w = None if params.weights is None else np.asarray(params.weights, np.float32).astype(np.float64)
    if _L().oracle_rolling(_ptr(x), ctypes.byref(p), None if w is None else _ptr(w), c_measure, step, c_eval,
                           diff_threshold, ctypes.byref(r)) != 0:
        raise ValueError("oracle_rolling: invalid parameters")
    n = r.n_sub
    return Rolling(status=r.status, t_init=r.t_init, t_iter=r.t_iter, early=bool(r.early), diff=r.diff,
                   smpdur_next=r.smpdur_next, sub_start=list(r.sub_start[:n]), sub_period=list(r.sub_period[:n]),
                   sub_err=list(r.sub_err[:n]), amb=bool(r.amb))


def measure(x: np.ndarray, params: Params, init: int, c_measure: float = 2.0, step: float = 0.5,
            c_eval: float = 6.5, diff_threshold: float = 0.05) -> dict:
    """M1: Alg. 4 on one recorded trace x float32 [F][N_max] (reading R6)."""
    x = np.ascontiguousarray(x, dtype=np.float32)
    p = params.c()
    m = OrMeasure()
    w = None if params.weights is None else np.asarray(params.weights, np.float32).astype(np.float64)
    if _L().oracle_measure(_ptr(x), ctypes.byref(p), None if w is None else _ptr(w), init, c_measure, step, c_eval,
                           diff_threshold, ctypes.byref(m)) != 0:
        raise ValueError("oracle_measure: invalid parameters")
    return dict(status=m.status, t_iter=m.t_iter, rounds=m.rounds, samples=m.samples,
                measure_start=m.measure_start, measure_end=m.measure_end, err_iter=m.err_iter, amb=bool(m.amb))


def gear_workload(**kw) -> OrGearWorkload:
    w = OrGearWorkload()
    for k, v in kw.items():
        setattr(w, k, v)
    return w


def gear_objective(w: OrGearWorkload, sm_mhz, mem_mhz, cap: float, gs: int, gm: int) -> float:
    sm = np.ascontiguousarray(sm_mhz, np.float64)
    mem = np.ascontiguousarray(mem_mhz, np.float64)
    return _L().oracle_gear_objective(ctypes.byref(w), _ptr(sm), sm.size, _ptr(mem), mem.size, cap, gs, gm)


def gear_search(w: OrGearWorkload, sm_mhz, mem_mhz, cap: float, pred_sm: int, pred_mem: int) -> dict:
    """G1: memory then SM local search (bracket, golden section, convex fit) on the simulator."""
    sm = np.ascontiguousarray(sm_mhz, np.float64)
    mem = np.ascontiguousarray(mem_mhz, np.float64)
    r = OrGearResult()
    if _L().oracle_gear_search(ctypes.byref(w), _ptr(sm), sm.size, _ptr(mem), mem.size, cap, pred_sm, pred_mem,
                               ctypes.byref(r)) != 0:
        raise ValueError("oracle_gear_search: invalid arguments")
    return dict(sm_gear=r.sm_gear, mem_gear=r.mem_gear, probes_sm=r.probes_sm, probes_mem=r.probes_mem,
                objective=r.objective, margin_rel=r.margin_rel, margin_round=r.margin_round)
