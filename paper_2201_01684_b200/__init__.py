"""Python binding of libgpoeo.so — the B200 GPOEO iteration-period detector.

Argument marshalling only: every step of Alg. 1 / Alg. 2 runs in
the CUDA kernels behind the C ABI declared in include/gpoeo.h. PyTorch supplies device
memory and streams. There is no CPU fallback: if the library cannot be built or loaded,
or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _build

MAX_FEATURES = 8
MAX_CANDIDATES = 32

TRACE_OK, TRACE_APERIODIC, TRACE_INSUFFICIENT, TRACE_CONSTANT = 0, 1, 2, 3
STATUS_NAMES = {0: "ok", 1: "aperiodic", 2: "insufficient", 3: "constant"}


class GpoeoParams(ctypes.Structure):
    _fields_ = [
        ("n_samples", ctypes.c_int32),
        ("n_features", ctypes.c_int32),
        ("trace_stride", ctypes.c_int64),
        ("sample_interval", ctypes.c_double),
        ("min_period", ctypes.c_int32),
        ("max_period", ctypes.c_int32),
        ("c_peak", ctypes.c_float),
        ("max_candidates", ctypes.c_int32),
        ("num_groups", ctypes.c_int32),
        ("gmm_max_iters", ctypes.c_int32),
        ("feature_weights", ctypes.c_float * MAX_FEATURES),
        ("bounded_search", ctypes.c_int32),
    ]


class GpoeoCounters(ctypes.Structure):
    _fields_ = [("n_candidate_queries", ctypes.c_int64), ("n_local_queries", ctypes.c_int64),
                ("cem_sample_passes", ctypes.c_int64), ("n_pruned_queries", ctypes.c_int64)]


RESULT_DTYPE = np.dtype([("period", "<i4"), ("period_s", "<f4"), ("error", "<f4"), ("status", "<i4"),
                         ("best_candidate", "<i4"), ("n_candidates", "<i4")])
DETAIL_DTYPE = np.dtype([("n_candidates", "<i4"), ("best_bin", "<i4"), ("local_lo", "<i4"), ("local_hi", "<i4"),
                         ("cand_k", "<i4", (MAX_CANDIDATES,)), ("cand_L", "<i4", (MAX_CANDIDATES,)),
                         ("cand_P", "<f4", (MAX_CANDIDATES,)), ("cand_err", "<f8", (MAX_CANDIDATES,)),
                         ("best_err", "<f8")])
ROLLING_DTYPE = np.dtype([("status", "<i4"), ("t_init", "<i4"), ("t_iter", "<i4"), ("n_sub", "<i4"),
                          ("early", "<i4"), ("diff", "<f4"), ("smpdur_next_s", "<f4"), ("err_iter", "<f4")])
MEASURE_DTYPE = np.dtype([("status", "<i4"), ("t_iter", "<i4"), ("rounds", "<i4"), ("samples", "<i4"),
                          ("measure_start", "<i4"), ("measure_end", "<i4"), ("t_iter_s", "<f4"), ("err_iter", "<f4")])
TRACE_UNSTABLE = 4
GEAR_WORKLOAD_DTYPE = np.dtype([(n, "<f8") for n in ("compute_work", "memory_work", "overhead", "p_static", "c_sm",
                                                      "c_mem", "u_c", "u_m", "noise")] + [("seed", "<u8")])
GEAR_RESULT_DTYPE = np.dtype([("sm_gear", "<i4"), ("mem_gear", "<i4"), ("probes_sm", "<i4"), ("probes_mem", "<i4"),
                              ("objective", "<f8")])
MAJOR_DTYPE = np.dtype([("period", "<i4"), ("period_s", "<f4"), ("bin", "<i4"), ("status", "<i4")])
assert RESULT_DTYPE.itemsize == 24 and DETAIL_DTYPE.itemsize == 664 and MAJOR_DTYPE.itemsize == 16
assert ROLLING_DTYPE.itemsize == 32 and MEASURE_DTYPE.itemsize == 32
assert GEAR_WORKLOAD_DTYPE.itemsize == 80 and GEAR_RESULT_DTYPE.itemsize == 24


class GpoeoRollingParams(ctypes.Structure):
    _fields_ = [("c_measure", ctypes.c_double), ("step", ctypes.c_double), ("c_eval", ctypes.c_double),
                ("diff_threshold", ctypes.c_double)]

_lib = None


class GpoeoError(RuntimeError):
    pass


def lib_path() -> str:
    return _build.LIB


def load():
    """Build (if stale) and load libgpoeo.so. Raises if that is impossible."""
    global _lib
    if _lib is not None:
        return _lib
    path = os.environ.get("GPOEO_LIB") or _build.LIB  # GPOEO_LIB: a prebuilt variant (profiling experiments)
    if not os.environ.get("GPOEO_LIB"):
        try:
            _build.build()
        except Exception as e:  # nvcc missing on a run box: use the shipped .so if present
            if not os.path.exists(path):
                raise GpoeoError(f"libgpoeo.so is missing and cannot be built: {e}") from e
    lib = ctypes.CDLL(path)
    P = ctypes.c_void_p
    PP = ctypes.POINTER(GpoeoParams)
    lib.gpoeo_default_params.argtypes = [PP, ctypes.c_int32, ctypes.c_int32, ctypes.c_double]
    lib.gpoeo_default_params.restype = None
    lib.gpoeo_validate_params.argtypes = [PP]
    lib.gpoeo_validate_params.restype = ctypes.c_int
    lib.gpoeo_workspace_size.argtypes = [PP, ctypes.c_int64]
    lib.gpoeo_workspace_size.restype = ctypes.c_size_t
    lib.gpoeo_detect_periods.argtypes = [P, ctypes.c_int64, PP, P, P, ctypes.c_size_t, P]
    lib.gpoeo_detect_periods.restype = ctypes.c_int
    lib.gpoeo_detect_periods_ex.argtypes = [P, ctypes.c_int64, PP, P, P, P, ctypes.c_size_t, P]
    lib.gpoeo_detect_periods_ex.restype = ctypes.c_int
    lib.gpoeo_detect_periods_timed.argtypes = [P, ctypes.c_int64, PP, P, P, P, ctypes.c_size_t, P, P]
    lib.gpoeo_detect_periods_timed.restype = ctypes.c_int
    lib.gpoeo_workspace_size_host.argtypes = [PP, ctypes.c_int64]
    lib.gpoeo_workspace_size_host.restype = ctypes.c_size_t
    lib.gpoeo_detect_periods_host.argtypes = [P, ctypes.c_int64, PP, P, ctypes.c_int64, P, ctypes.c_size_t, P]
    lib.gpoeo_detect_periods_host.restype = ctypes.c_int
    lib.gpoeo_power_spectrum.argtypes = [P, ctypes.c_int64, PP, P, P, P, ctypes.c_size_t, P]
    lib.gpoeo_power_spectrum.restype = ctypes.c_int
    lib.gpoeo_similarity_workspace_size.argtypes = [ctypes.c_int64]
    lib.gpoeo_similarity_workspace_size.restype = ctypes.c_size_t
    lib.gpoeo_similarity_error.argtypes = [P, ctypes.c_int64, ctypes.c_int32, P, P, ctypes.c_int64, ctypes.c_int32,
                                           ctypes.c_int32, P, P, ctypes.c_size_t, P]
    lib.gpoeo_similarity_error.restype = ctypes.c_int
    lib.gpoeo_major_workspace_size.argtypes = [PP, ctypes.c_int64]
    lib.gpoeo_major_workspace_size.restype = ctypes.c_size_t
    lib.gpoeo_detect_major_periods.argtypes = [P, ctypes.c_int64, PP, P, P, ctypes.c_size_t, P]
    lib.gpoeo_detect_major_periods.restype = ctypes.c_int
    RP = ctypes.POINTER(GpoeoRollingParams)
    lib.gpoeo_default_rolling_params.argtypes = [RP]
    lib.gpoeo_default_rolling_params.restype = None
    lib.gpoeo_workspace_size_rolling.argtypes = [PP, RP, ctypes.c_int64]
    lib.gpoeo_workspace_size_rolling.restype = ctypes.c_size_t
    lib.gpoeo_detect_rolling.argtypes = [P, ctypes.c_int64, PP, RP, P, P, ctypes.c_size_t, P]
    lib.gpoeo_detect_rolling.restype = ctypes.c_int
    lib.gpoeo_workspace_size_measure.argtypes = [PP, RP, ctypes.c_int64]
    lib.gpoeo_workspace_size_measure.restype = ctypes.c_size_t
    lib.gpoeo_measure_adaptive.argtypes = [P, ctypes.c_int64, PP, RP, ctypes.c_int32, P, P, ctypes.c_size_t, P]
    lib.gpoeo_measure_adaptive.restype = ctypes.c_int
    lib.gpoeo_gear_search.argtypes = [P, ctypes.c_int64, P, ctypes.c_int32, P, ctypes.c_int32, ctypes.c_double, P, P,
                                      P, P]
    lib.gpoeo_gear_search.restype = ctypes.c_int
    lib.gpoeo_local_range_max.argtypes = [PP]
    lib.gpoeo_local_range_max.restype = ctypes.c_int64
    lib.gpoeo_local_scores.argtypes = [P, PP, ctypes.c_int64, P, P]
    lib.gpoeo_local_scores.restype = ctypes.c_int
    lib.gpoeo_read_counters.argtypes = [P, PP, ctypes.c_int64, ctypes.POINTER(GpoeoCounters), P]
    lib.gpoeo_read_counters.restype = ctypes.c_int
    lib.gpoeo_status_string.argtypes = [ctypes.c_int]
    lib.gpoeo_status_string.restype = ctypes.c_char_p
    lib.gpoeo_version.argtypes = []
    lib.gpoeo_version.restype = ctypes.c_int
    _lib = lib
    return lib


def _check(rc: int, what: str) -> None:
    if rc != 0:
        raise GpoeoError(f"{what}: {load().gpoeo_status_string(rc).decode()} ({rc})")


def default_params(n_samples: int, n_features: int = 1, sample_interval: float = 1.0, **kw) -> GpoeoParams:
    """gpoeo_default_params, then override any field by keyword (weights=... for w_c)."""
    p = GpoeoParams()
    load().gpoeo_default_params(ctypes.byref(p), n_samples, n_features, sample_interval)
    weights = kw.pop("weights", None)
    for k, v in kw.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, v)
    if weights is not None:
        for i, w in enumerate(weights):
            p.feature_weights[i] = w
    return p


def params_for(spec, **kw) -> GpoeoParams:
    """Params for a workload-spec object (n_samples, n_features, min/max_period)."""
    return default_params(spec.n_samples, spec.n_features, kw.pop("sample_interval", 1.0),
                          min_period=spec.min_period, max_period=spec.max_period, **kw)


def validate(p: GpoeoParams) -> int:
    return load().gpoeo_validate_params(ctypes.byref(p))


def workspace_size(p: GpoeoParams, batch: int) -> int:
    return int(load().gpoeo_workspace_size(ctypes.byref(p), batch))


def _stream_handle(stream):
    import torch
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, int):
        return ctypes.c_void_p(stream)
    return ctypes.c_void_p(stream.cuda_stream)


def alloc_workspace(nbytes: int, device=None):
    import torch
    return torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device=device or "cuda")


def detect_periods(traces, p: GpoeoParams, workspace=None, results=None, detail=False, stream=None):
    """Alg. 1 on a CUDA float32 tensor of traces [B][trace_stride] (or [B][F][N]).

    Returns (results uint8 tensor viewed as RESULT_DTYPE records, detail tensor or None,
    workspace). Asynchronous on `stream` (default: torch's current stream).
    """
    import torch
    assert traces.is_cuda and traces.dtype == torch.float32 and traces.is_contiguous()
    B = traces.shape[0]
    lib = load()
    need = workspace_size(p, B)
    if need == 0:
        _check(validate(p), "params")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, traces.device)
    if results is None:
        results = torch.empty(B * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=traces.device)
    det = torch.empty(B * DETAIL_DTYPE.itemsize, dtype=torch.uint8, device=traces.device) if detail else None
    rc = lib.gpoeo_detect_periods_ex(ctypes.c_void_p(traces.data_ptr()), B, ctypes.byref(p),
                                     ctypes.c_void_p(results.data_ptr()),
                                     ctypes.c_void_p(det.data_ptr()) if det is not None else None,
                                     ctypes.c_void_p(workspace.data_ptr()), workspace.numel(), _stream_handle(stream))
    _check(rc, "gpoeo_detect_periods")
    return results, det, workspace


PHASES = ("composite", "spectrum_peaks", "score_candidates", "select", "score_local", "final")


def detect_periods_timed(traces, p: GpoeoParams, workspace, results, events, stream=None):
    """gpoeo_detect_periods_timed with 7 torch.cuda.Event(enable_timing=True) objects
    (already recorded once so their handles exist); returns nothing (async)."""
    arr = (ctypes.c_void_p * 7)(*[ctypes.c_void_p(e.cuda_event) for e in events])
    rc = load().gpoeo_detect_periods_timed(ctypes.c_void_p(traces.data_ptr()), traces.shape[0], ctypes.byref(p),
                                           ctypes.c_void_p(results.data_ptr()), None,
                                           ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                           _stream_handle(stream), arr)
    _check(rc, "gpoeo_detect_periods_timed")


def results_numpy(results) -> np.ndarray:
    return results.cpu().numpy().view(RESULT_DTYPE)


def detail_numpy(det) -> np.ndarray:
    return det.cpu().numpy().view(DETAIL_DTYPE)


def detect_periods_host(host_traces: np.ndarray, p: GpoeoParams, chunk: int = 4096, workspace=None, stream=None,
                        out: np.ndarray | None = None) -> np.ndarray:
    """End-to-end over HOST memory (pinned numpy/torch buffer recommended): chunked H2D
    copies overlapped with compute inside the library; returns RESULT_DTYPE records."""
    lib = load()
    B = host_traces.shape[0]
    chunk = max(1, min(chunk, B))
    need = int(lib.gpoeo_workspace_size_host(ctypes.byref(p), chunk))
    if need == 0:
        _check(validate(p), "params")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need)
    if out is None:
        out = np.empty(B, dtype=RESULT_DTYPE)
    ptr = host_traces.data_ptr() if hasattr(host_traces, "data_ptr") else host_traces.ctypes.data
    rc = lib.gpoeo_detect_periods_host(ctypes.c_void_p(ptr), B, ctypes.byref(p), ctypes.c_void_p(out.ctypes.data),
                                       chunk, ctypes.c_void_p(workspace.data_ptr()), workspace.numel(),
                                       _stream_handle(stream))
    _check(rc, "gpoeo_detect_periods_host")
    return out


def power_spectrum(traces, p: GpoeoParams, want_signal=True, stream=None):
    """(spectra [B][N/2+1] fp32, signal [B][N] fp32) on the device."""
    import torch
    B = traces.shape[0]
    N = p.n_samples
    lib = load()
    ws = alloc_workspace(workspace_size(p, B) or 256, traces.device)
    spectra = torch.empty((B, N // 2 + 1), dtype=torch.float32, device=traces.device)
    signal = torch.empty((B, N), dtype=torch.float32, device=traces.device) if want_signal else None
    rc = lib.gpoeo_power_spectrum(ctypes.c_void_p(traces.data_ptr()), B, ctypes.byref(p),
                                  ctypes.c_void_p(spectra.data_ptr()),
                                  ctypes.c_void_p(signal.data_ptr()) if signal is not None else None,
                                  ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_handle(stream))
    _check(rc, "gpoeo_power_spectrum")
    return spectra, signal


def similarity_error(signal, trace_index, period, num_groups: int = 4, gmm_max_iters: int = 32, stream=None):
    """Alg. 2 Err(L) for queries (trace_index[q], period[q]) on signal [B][N] (CUDA fp32)."""
    import torch
    lib = load()
    B, N = signal.shape
    ti = torch.as_tensor(trace_index, dtype=torch.int32, device=signal.device).contiguous()
    pe = torch.as_tensor(period, dtype=torch.int32, device=signal.device).contiguous()
    nq = ti.numel()
    out = torch.empty(nq, dtype=torch.float64, device=signal.device)
    ws = alloc_workspace(int(lib.gpoeo_similarity_workspace_size(nq)), signal.device)
    rc = lib.gpoeo_similarity_error(ctypes.c_void_p(signal.data_ptr()), B, N, ctypes.c_void_p(ti.data_ptr()),
                                    ctypes.c_void_p(pe.data_ptr()), nq, num_groups, gmm_max_iters,
                                    ctypes.c_void_p(out.data_ptr()), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                    _stream_handle(stream))
    _check(rc, "gpoeo_similarity_error")
    return out


def major_workspace_size(p: GpoeoParams, batch: int) -> int:
    return int(load().gpoeo_major_workspace_size(ctypes.byref(p), batch))


def detect_major_periods(traces, p: GpoeoParams, workspace=None, results=None, stream=None):
    """Spectral-only detector (T_iter = 1/f_major; reading R3) on a CUDA float32
    tensor of traces [B][trace_stride]. Returns (results uint8 tensor of MAJOR_DTYPE
    records, workspace). Asynchronous on `stream`."""
    import torch
    assert traces.is_cuda and traces.dtype == torch.float32 and traces.is_contiguous()
    B = traces.shape[0]
    lib = load()
    need = major_workspace_size(p, B)
    if need == 0:
        _check(validate(p), "params")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, traces.device)
    if results is None:
        results = torch.empty(B * MAJOR_DTYPE.itemsize, dtype=torch.uint8, device=traces.device)
    rc = lib.gpoeo_detect_major_periods(ctypes.c_void_p(traces.data_ptr()), B, ctypes.byref(p),
                                        ctypes.c_void_p(results.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
                                        workspace.numel(), _stream_handle(stream))
    _check(rc, "gpoeo_detect_major_periods")
    return results, workspace


def major_numpy(results) -> np.ndarray:
    return results.cpu().numpy().view(MAJOR_DTYPE)


def default_rolling_params(**kw) -> GpoeoRollingParams:
    rp = GpoeoRollingParams()
    load().gpoeo_default_rolling_params(ctypes.byref(rp))
    for k, v in kw.items():
        setattr(rp, k, v)
    return rp


def detect_rolling_async(traces, p: GpoeoParams, rp: GpoeoRollingParams | None = None, workspace=None, results=None,
                         stream=None):
    """Alg. 3 (reading R5) on a CUDA float32 tensor of recorded traces
    [B][trace_stride]: enqueued on `stream`, no host round trip. Returns (results uint8 device
    tensor of ROLLING_DTYPE records, workspace)."""
    import torch
    assert traces.is_cuda and traces.dtype == torch.float32 and traces.is_contiguous()
    B = traces.shape[0]
    lib = load()
    rp = rp or default_rolling_params()
    need = int(lib.gpoeo_workspace_size_rolling(ctypes.byref(p), ctypes.byref(rp), B))
    if need == 0:
        _check(validate(p), "params")
        raise GpoeoError("invalid rolling parameters")
    if workspace is None or workspace.numel() < need:
        workspace = alloc_workspace(need, traces.device)
    if results is None:
        results = torch.empty(B * ROLLING_DTYPE.itemsize, dtype=torch.uint8, device=traces.device)
    rc = lib.gpoeo_detect_rolling(ctypes.c_void_p(traces.data_ptr()), B, ctypes.byref(p), ctypes.byref(rp),
                                  ctypes.c_void_p(results.data_ptr()), ctypes.c_void_p(workspace.data_ptr()),
                                  workspace.numel(), _stream_handle(stream))
    _check(rc, "gpoeo_detect_rolling")
    return results, workspace


def detect_rolling(traces, p: GpoeoParams, rp: GpoeoRollingParams | None = None, stream=None) -> np.ndarray:
    """detect_rolling_async, then the records on the host (ROLLING_DTYPE)."""
    import torch
    out, _ = detect_rolling_async(traces, p, rp, stream=stream)
    if stream is not None and not isinstance(stream, int):
        torch.cuda.current_stream().wait_stream(stream)
    return out.cpu().numpy().view(ROLLING_DTYPE)


def measure_adaptive(traces, p: GpoeoParams, init_samples: int, rp: GpoeoRollingParams | None = None,
                     stream=None) -> np.ndarray:
    """Alg. 4 (reading R6) over recordings [B][trace_stride] on the device (the
    simulated sampling backend); synchronous; returns MEASURE_DTYPE records."""
    import torch
    assert traces.is_cuda and traces.dtype == torch.float32 and traces.is_contiguous()
    B = traces.shape[0]
    lib = load()
    rp = rp or default_rolling_params()
    need = int(lib.gpoeo_workspace_size_measure(ctypes.byref(p), ctypes.byref(rp), B))
    if need == 0:
        _check(validate(p), "params")
        raise GpoeoError("invalid rolling parameters")
    ws = alloc_workspace(need, traces.device)
    out = np.empty(B, dtype=MEASURE_DTYPE)
    rc = lib.gpoeo_measure_adaptive(ctypes.c_void_p(traces.data_ptr()), B, ctypes.byref(p), ctypes.byref(rp),
                                    int(init_samples), ctypes.c_void_p(out.ctypes.data),
                                    ctypes.c_void_p(ws.data_ptr()), ws.numel(), _stream_handle(stream))
    _check(rc, "gpoeo_measure_adaptive")
    return out


def gear_search(workloads: np.ndarray, sm_mhz, mem_mhz, cap: float, pred_sm, pred_mem, device="cuda",
                stream=None) -> np.ndarray:
    """Gear local search (reading R7) for GEAR_WORKLOAD_DTYPE records on the
    simulated device, one GPU thread per workload; returns GEAR_RESULT_DTYPE records."""
    import torch
    lib = load()
    n = len(workloads)
    w = torch.from_numpy(np.ascontiguousarray(workloads).view(np.uint8).copy()).to(device)
    sm = torch.as_tensor(np.asarray(sm_mhz, np.float64), device=device)
    mem = torch.as_tensor(np.asarray(mem_mhz, np.float64), device=device)
    ps = torch.as_tensor(np.asarray(pred_sm, np.int32), device=device)
    pm = torch.as_tensor(np.asarray(pred_mem, np.int32), device=device)
    out = torch.empty(n * GEAR_RESULT_DTYPE.itemsize, dtype=torch.uint8, device=device)
    rc = lib.gpoeo_gear_search(ctypes.c_void_p(w.data_ptr()), n, ctypes.c_void_p(sm.data_ptr()), sm.numel(),
                               ctypes.c_void_p(mem.data_ptr()), mem.numel(), float(cap), ctypes.c_void_p(ps.data_ptr()),
                               ctypes.c_void_p(pm.data_ptr()), ctypes.c_void_p(out.data_ptr()), _stream_handle(stream))
    _check(rc, "gpoeo_gear_search")
    return out.cpu().numpy().view(GEAR_RESULT_DTYPE)


def local_scores(workspace, p: GpoeoParams, batch: int, stream=None):
    """gpoeo_local_scores: [batch][local_range_max] fp64 device tensor of the local-range
    Err(L) of the last detect call on `workspace` (NaN-padded)."""
    import torch
    lib = load()
    ml = int(lib.gpoeo_local_range_max(ctypes.byref(p)))
    out = torch.empty((batch, max(ml, 1)), dtype=torch.float64, device=workspace.device)
    _check(lib.gpoeo_local_scores(ctypes.c_void_p(workspace.data_ptr()), ctypes.byref(p), batch,
                                  ctypes.c_void_p(out.data_ptr()), _stream_handle(stream)), "gpoeo_local_scores")
    return out


def read_counters(workspace, p: GpoeoParams, batch: int, stream=None) -> dict:
    c = GpoeoCounters()
    _check(load().gpoeo_read_counters(ctypes.c_void_p(workspace.data_ptr()), ctypes.byref(p), batch,
                                      ctypes.byref(c), _stream_handle(stream)), "gpoeo_read_counters")
    return dict(n_candidate_queries=c.n_candidate_queries, n_local_queries=c.n_local_queries,
                cem_sample_passes=c.cem_sample_passes, n_pruned_queries=c.n_pruned_queries)


def version() -> int:
    return load().gpoeo_version()
