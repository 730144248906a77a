"""CPU-side checks of the C ABI (no GPU compute): libgpoeo.so builds for sm_100a, loads,
exports every function include/gpoeo.h declares, and validates arguments synchronously.
"""
import ctypes
import os
import re
import subprocess

import pytest

import paper_2201_01684_b200 as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "gpoeo.h")


def _declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(gpoeo_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = g.load()
    names = _declared_functions()
    assert len(names) >= 12
    out = subprocess.check_output(["nm", "-D", "--defined-only", g.lib_path()], text=True)
    exported = set(l.split()[-1] for l in out.splitlines() if " T " in l)
    for n in names:
        assert n in exported, n
        assert hasattr(lib, n)


def test_built_for_sm100a():
    out = subprocess.check_output(["cuobjdump", "--list-elf", g.lib_path()], text=True)
    assert "sm_100a" in out


def test_version_and_status_strings():
    lib = g.load()
    assert g.version() == 1
    for code in (0, -1, -2, -3, -4, -5):
        assert lib.gpoeo_status_string(code)
    assert b"unknown" in lib.gpoeo_status_string(42)


def test_default_params_and_struct_layout():
    p = g.default_params(1024, 3, 0.1)
    assert (p.n_samples, p.n_features, p.trace_stride) == (1024, 3, 3072)
    assert p.min_period == 2 and p.max_period == 512
    assert abs(p.c_peak - 0.65) < 1e-7 and p.max_candidates == 16 and p.num_groups == 4
    assert p.gmm_max_iters == 32 and list(p.feature_weights) == [1.0] * 8
    assert p.bounded_search == 1
    assert ctypes.sizeof(g.GpoeoParams) == 88  # 80 + bounded_search, padded to 8
    assert g.validate(p) == 0


@pytest.mark.parametrize("field,value,code", [
    ("n_samples", 4, -2), ("n_samples", 1 << 19, -2),
    ("n_features", 0, -1), ("n_features", 9, -1),
    ("min_period", 1, -1), ("max_period", 513, -1), ("c_peak", 0.0, -1), ("c_peak", 1.5, -1),
    ("max_candidates", 0, -1), ("max_candidates", 33, -1), ("num_groups", 0, -1), ("num_groups", 9, -1),
    ("gmm_max_iters", 0, -1), ("sample_interval", 0.0, -1), ("trace_stride", 3074, -4),
    ("bounded_search", 2, -1), ("bounded_search", -1, -1),
])
def test_validation_codes(field, value, code):
    p = g.default_params(1024, 3)
    setattr(p, field, value)
    assert g.validate(p) == code
    assert g.workspace_size(p, 10) == 0


def test_non_power_of_two_lengths():
    # any N in [8, 2^18] (band-limited DFT when N is not a power of two) ...
    for N in (8, 9, 1000, 4095, 10_001):
        p = g.default_params(N, 3)
        assert g.validate(p) == 0 and g.workspace_size(p, 4) > 0
    # ... unless its band does not fit in shared memory (N/2 bins here)
    assert g.validate(g.default_params(200_000, 1)) == -2
    p = g.default_params(200_000, 1)
    p.min_period = 100  # band k <= 2000: fine
    assert g.validate(p) == 0


def test_workspace_size_monotone():
    p = g.default_params(65536, 3, min_period=10, max_period=4096)
    a, b = g.workspace_size(p, 10), g.workspace_size(p, 1000)
    assert 0 < a < b
    # dominated by the composite signal y[B][N] and the local-search list
    assert b >= 1000 * 65536 * 4


def test_errors_are_synchronous_without_a_device():
    lib = g.load()
    p = g.default_params(1024, 1)
    res = ctypes.create_string_buffer(64)
    # invalid argument -> reported before any device work
    bad = g.default_params(1 << 19, 1)  # N above 2^18
    assert lib.gpoeo_detect_periods(ctypes.c_void_p(16), 1, ctypes.byref(bad), res, ctypes.c_void_p(256), 1 << 20,
                                    None) == -2
    assert lib.gpoeo_detect_periods(ctypes.c_void_p(16), 1, ctypes.byref(p), res, None, 0, None) == -3
    need = g.workspace_size(p, 1)
    assert lib.gpoeo_detect_periods(ctypes.c_void_p(17), 1, ctypes.byref(p), res, ctypes.c_void_p(256), need,
                                    None) == -4


def test_no_cpu_fallback_without_device():
    import torch
    if torch.cuda.is_available():
        pytest.skip("device present")
    lib = g.load()
    p = g.default_params(1024, 1)
    need = g.workspace_size(p, 1)
    res = ctypes.create_string_buffer(64)
    # valid arguments but no CUDA device: the library refuses (GPOEO_ERR_CUDA), never computes on the host
    assert lib.gpoeo_detect_periods(ctypes.c_void_p(256), 1, ctypes.byref(p), res, ctypes.c_void_p(256), need,
                                    None) == -5


def test_product_path_never_touches_oracle():
    # the product (package + header) and the oracle share no code and never import each other
    banned_in_product = ("import oracle", "from oracle", "liboracle", "gpoeo_oracle", "tracegen")
    for base in (os.path.join(ROOT, "paper_2201_01684_b200"), os.path.join(ROOT, "include")):
        for dirpath, _, files in os.walk(base):
            for f in files:
                if f.endswith((".py", ".cu", ".cuh", ".h", ".c")):
                    txt = open(os.path.join(dirpath, f)).read()
                    for b in banned_in_product:
                        assert b not in txt, (f, b)
    for f in os.listdir(os.path.join(ROOT, "oracle")):
        if f.endswith((".py", ".c")):
            txt = open(os.path.join(ROOT, "oracle", f)).read()
            for b in ("import paper_2201_01684_b200", "from paper_2201_01684_b200", '#include "gpoeo', "libgpoeo",
                      "csrc/"):
                assert b not in txt, (f, b)
