"""Seeded synthetic telemetry traces (power, SM util, mem util) for tests and bench.

TEST/BENCH INPUT INFRASTRUCTURE, shared by both sides of every parity check: the
CUDA path and the oracle consume the same bytes. Holds none of the method's
arithmetic. The recipe is documented in tracegen.h and DESIGN.md ("Input recipe").

Host build (gcc) and device build (nvcc --fmad=false) of the same header produce
bit-identical floats, so the oracle may be fed host-generated traces while the GPU
generates the full batch in HBM.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_HOST_SO = os.path.join(_HERE, "libtracegen_host.so")
_CUDA_SO = os.path.join(_HERE, "libtracegen_cuda.so")

KIND_AIBENCH = 0
KIND_HARD = 1


class TgConfig(ctypes.Structure):
    _fields_ = [
        ("kind", ctypes.c_int32),
        ("n_samples", ctypes.c_int32),
        ("n_features", ctypes.c_int32),
        ("quantize", ctypes.c_int32),
        ("seed", ctypes.c_uint64),
        ("period_lo", ctypes.c_double),
        ("period_hi", ctypes.c_double),
        ("log2_ratio", ctypes.c_double),
        ("noise", ctypes.c_double),
        ("hf_prob", ctypes.c_double),
        ("hf_amp", ctypes.c_double),
        ("aperiodic_mod", ctypes.c_int32),
        ("pad_", ctypes.c_int32),
    ]


class TgParams(ctypes.Structure):
    _fields_ = [
        ("L1", ctypes.c_double),
        ("L2", ctypes.c_double),
        ("phi0", ctypes.c_double),
        ("phi1", ctypes.c_double),
        ("cum", ctypes.c_double * 5),
        ("lev", ctypes.c_double * 4),
        ("ca", ctypes.c_double * 3),
        ("cb", ctypes.c_double * 3),
        ("hf_period", ctypes.c_double),
        ("hf_phase", ctypes.c_double),
        ("nph", ctypes.c_int32),
        ("aperiodic", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class TraceSpec:
    """One synthetic workload (BASELINE.json configs 1-5)."""

    name: str
    batch: int
    n_samples: int
    n_features: int
    period_lo: float
    period_hi: float
    min_period: int
    max_period: int
    seed: int
    noise: float = 0.05
    hf_prob: float = 0.0
    hf_amp: float = 0.08
    aperiodic_mod: int = 0
    kind: int = KIND_AIBENCH
    quantize: int = 1

    def config(self) -> TgConfig:
        c = TgConfig()
        c.kind = self.kind
        c.n_samples = self.n_samples
        c.n_features = self.n_features
        c.quantize = self.quantize
        c.seed = self.seed
        c.period_lo = self.period_lo
        c.period_hi = self.period_hi
        c.log2_ratio = math.log2(self.period_hi / self.period_lo) if self.period_hi > self.period_lo else 0.0
        c.noise = self.noise
        c.hf_prob = self.hf_prob
        c.hf_amp = self.hf_amp
        c.aperiodic_mod = self.aperiodic_mod
        return c

    def with_(self, **kw) -> "TraceSpec":
        d = dict(self.__dict__)
        d.update(kw)
        return TraceSpec(**d)


# BASELINE.json "configs", in order.
CFG1 = TraceSpec("cfg1_single_1x1x1024_L37", 1, 1024, 1, 37.0, 37.0, 4, 512, seed=1)
CFG2 = TraceSpec("cfg2_aibench71_3x8192", 71, 8192, 3, 20.0, 2000.0, 10, 4096, seed=2,
                 hf_prob=1.0 / 3.0, aperiodic_mod=18)
CFG3 = TraceSpec("cfg3_1e5x3x65536", 100_000, 65536, 3, 20.0, 2000.0, 10, 4096, seed=3,
                 hf_prob=1.0 / 3.0, aperiodic_mod=18)
CFG4 = TraceSpec("cfg4_1e6x3x65536_sharded", 1_000_000, 65536, 3, 20.0, 2000.0, 10, 4096, seed=4,
                 hf_prob=1.0 / 3.0, aperiodic_mod=18)
CFG5 = TraceSpec("cfg5_hard_1e4x3x262144", 10_000, 262144, 3, 20.0, 2000.0, 10, 8192, seed=5,
                 kind=KIND_HARD)
CONFIGS = [CFG1, CFG2, CFG3, CFG4, CFG5]


def _build_host() -> None:
    src = os.path.join(_HERE, "tracegen_host.c")
    if os.path.exists(_HOST_SO) and os.path.getmtime(_HOST_SO) >= max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "tracegen.h"))):
        return
    subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fPIC", "-shared", "-o", _HOST_SO, src, "-lm"])


def build_device() -> None:
    src = os.path.join(_HERE, "tracegen_cuda.cu")
    if os.path.exists(_CUDA_SO) and os.path.getmtime(_CUDA_SO) >= max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "tracegen.h"))):
        return
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "--fmad=false",
                           "-lineinfo", "-Xcompiler", "-fPIC", "-shared", "-o", _CUDA_SO, src])


_host_lib = None
_cuda_lib = None


def _host():
    global _host_lib
    if _host_lib is None:
        _build_host()
        lib = ctypes.CDLL(_HOST_SO)
        lib.tg_generate_host.argtypes = [ctypes.POINTER(TgConfig), ctypes.c_int64, ctypes.c_int64,
                                         ctypes.c_void_p, ctypes.c_int64]
        lib.tg_generate_host.restype = ctypes.c_int
        lib.tg_trace_params_host.argtypes = [ctypes.POINTER(TgConfig), ctypes.c_int64, ctypes.POINTER(TgParams)]
        lib.tg_trace_params_host.restype = ctypes.c_int
        assert lib.tg_sizeof_config() == ctypes.sizeof(TgConfig)
        assert lib.tg_sizeof_params() == ctypes.sizeof(TgParams)
        _host_lib = lib
    return _host_lib


def _cuda():
    global _cuda_lib
    if _cuda_lib is None:
        build_device()
        lib = ctypes.CDLL(_CUDA_SO)
        lib.tg_generate_device.argtypes = [ctypes.POINTER(TgConfig), ctypes.c_int64, ctypes.c_int64,
                                           ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p]
        lib.tg_generate_device.restype = ctypes.c_int
        _cuda_lib = lib
    return _cuda_lib


def generate_host(spec: TraceSpec, first: int = 0, count: int | None = None, threads: int | None = None) -> np.ndarray:
    """float32 array [count][F][N] of traces first..first+count-1 (host build)."""
    if count is None:
        count = spec.batch - first
    out = np.empty((count, spec.n_features, spec.n_samples), dtype=np.float32)
    cfg = spec.config()
    lib = _host()
    stride = spec.n_features * spec.n_samples
    threads = threads or min(os.cpu_count() or 1, max(1, count))
    per = (count + threads - 1) // max(1, threads)

    def work(i0):
        n = min(per, count - i0)
        if n <= 0:
            return 0
        ptr = out.ctypes.data + i0 * stride * 4
        return lib.tg_generate_host(ctypes.byref(cfg), first + i0, n, ctypes.c_void_p(ptr), stride)

    with ThreadPoolExecutor(max_workers=threads) as ex:
        rcs = list(ex.map(work, range(0, count, per)))
    if any(rcs):
        raise RuntimeError("tracegen host generation failed")
    return out


def generate_device(spec: TraceSpec, out, first: int = 0, count: int | None = None, stream: int = 0) -> None:
    """Fill a CUDA float32 tensor/pointer [count][>=F*N] with traces (device build)."""
    if count is None:
        count = spec.batch - first
    cfg = spec.config()
    ptr = out.data_ptr() if hasattr(out, "data_ptr") else int(out)
    stride = out.stride(0) if hasattr(out, "stride") and out.dim() == 2 else spec.n_features * spec.n_samples
    rc = _cuda().tg_generate_device(ctypes.byref(cfg), first, count, ctypes.c_void_p(ptr), stride,
                                    ctypes.c_void_p(stream))
    if rc != 0:
        raise RuntimeError(f"tracegen device generation failed rc={rc}")


def trace_params(spec: TraceSpec, trace: int) -> TgParams:
    p = TgParams()
    _host().tg_trace_params_host(ctypes.byref(spec.config()), trace, ctypes.byref(p))
    return p


def planted_period(spec: TraceSpec, trace: int) -> float:
    """Planted (true) iteration period in samples; nan for aperiodic traces."""
    p = trace_params(spec, trace)
    return float("nan") if p.aperiodic else p.L1
