"""The drop-in boundary: every symbol declared in include/*.h is exported by
the B200 library; the shared C-ABI (quantc_capi.h) is exported by the
reference oracle build too (same binding source compiled against the
reference); device entry points fail loudly without a GPU."""
import ctypes
import os
import re

import numpy as np
import pytest
import torch

from paper_2103_14949_b200 import quantc as Q

INC = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "include")


def _declared(header):
    text = open(os.path.join(INC, header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(qcu?_[a-z0-9_]+)\s*\(", text)))


def test_b200_exports_every_declared_symbol(b200):
    for header in ("quantc_capi.h", "quantc_cuda.h", "quantc_files.h"):
        names = _declared(header)
        assert len(names) >= 6
        for n in names:
            assert hasattr(b200.lib, n), f"{n} ({header}) not exported"


def test_reference_exports_the_shared_capi(ref):
    for n in _declared("quantc_capi.h"):
        assert hasattr(ref.lib, n), n
    assert ref.name == "quantc-reference"


def test_public_headers_mirror_reference_api():
    hdrs = sorted(os.listdir(os.path.join(INC, "quantc")))
    for h in ["calibration.hpp", "dtype.hpp", "graph.hpp", "hwspec.hpp", "interpreter.hpp",
              "parallel.hpp", "realize.hpp", "search.hpp", "simulate.hpp", "tensor.hpp",
              "topology.hpp"]:
        assert h in hdrs


@pytest.mark.skipif(torch.cuda.is_available(), reason="CPU-only behaviour")
def test_device_paths_fail_loudly_without_gpu(b200):
    p = Q.QParams.symmetric(1.0, 8)
    with pytest.raises(Q.DeviceError):
        b200.simulated_quantize(np.ones(4, np.float32), p)
    with pytest.raises(Q.DeviceError):
        b200.simulated_quantize_value(0.5, p)
    assert b200.lib.qcu_tcgen05_available() == 0


def test_host_scalar_helpers_match_reference(b200, ref):
    for t, b, s in [(1.0, 8, 1), (6.0, 6, 1), (1.0, 8, 0)]:
        assert b200.compute_scale(t, b, s) == ref.compute_scale(t, b, s)
    for b, s in [(8, 1), (2, 0), (16, 1), (31, 0)]:
        assert b200.quant_bounds(b, s) == ref.quant_bounds(b, s)
    for v in (3.2, 2.0, 1.5, 0.3, 1e-8):
        assert b200.round_pow2(v) == ref.round_pow2(v)
    for args in [(-1.0, 4.0, 8), (0.5, 2.0, 4)]:
        assert b200.asymmetric_zero_point(*args) == ref.asymmetric_zero_point(*args)
    counts = np.random.default_rng(0).integers(0, 9, 2048)
    for q in (0.5, 0.99, 0.999, 1.0):
        assert b200.threshold_quantile(counts, 3.0, q) == ref.threshold_quantile(counts, 3.0, q)
    assert b200.threshold_max(0.0) == ref.threshold_max(0.0) == 1e-8
    for bad in (0.0, -1.0):
        with pytest.raises(Q.InvalidArgument):
            b200.compute_scale(bad, 8, 1)
        with pytest.raises(Q.InvalidArgument):
            ref.compute_scale(bad, 8, 1)
    with pytest.raises(Q.CalibrationError):
        b200.threshold_quantile(counts, 3.0, 1.5)


def test_host_worker_pool_selftest_and_clean_exit(tmp_path):
    """quantc::parallel_for runs on persistent workers: sums are exact for any
    worker count, the lowest failing index's exception is reported, and a
    process that used the pool exits promptly (the workers never block exit)."""
    import pathlib
    import subprocess
    import sys
    repo = str(pathlib.Path(__file__).resolve().parents[1])
    code = r'''
import ctypes as C, sys
sys.path.insert(0, %r)
from paper_2103_14949_b200 import quantc as Q
L = Q.load_b200().lib
f = L.qcu_parallel_selftest
f.argtypes = [C.c_size_t, C.c_int, C.c_int64, C.POINTER(C.c_int64)]
s = C.c_int64()
for n in (0, 1, 7, 1000, 100003):
    for w in (1, 2, 8, 33):
        assert f(n, w, -1, C.byref(s)) == 0
        assert s.value == n * (n - 1) // 2, (n, w, s.value)
rc = f(1000, 8, 500, C.byref(s))
assert rc != 0
L.qcu_last_error.restype = C.c_char_p
assert b"selftest index 500" in L.qcu_last_error(), L.qcu_last_error()
print("ok")
''' % (repo,)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("ok")
