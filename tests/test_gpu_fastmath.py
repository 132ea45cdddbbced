"""The branch-free fast paths (csrc/fastdiv.cuh) against IEEE division and
the deterministic log, bitwise, over operands spanning the whole exponent
range (including zeros, subnormals, infinities and NaN, which the fast paths
must reject)."""

import ctypes

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_fast_division_and_log_are_exact_whenever_accepted():
    import torch

    from paper_2205_04148_b200 import _lib

    rng = np.random.default_rng(17)
    n = 1 << 22
    # random bit patterns (every exponent) mixed with realistic magnitudes
    bits = rng.integers(0, 2**63, n, dtype=np.int64) * rng.choice([1, -1], n)
    x = bits.view(np.float64).copy()
    y = rng.integers(0, 2**63, n, dtype=np.int64).view(np.float64).copy()
    m = n // 2
    x[:m] = rng.uniform(-1e3, 1e3, m) * 10.0 ** rng.integers(-30, 30, m)
    y[:m] = rng.uniform(-1e3, 1e3, m) * 10.0 ** rng.integers(-30, 30, m)
    x[:16] = [0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1e-310, 1e308, 1.0, 2.0, 3.0, 0.5, 1e-300, 1e300, 7.0, 9.0]
    y[:16] = [1.0, 2.0, 3.0, np.inf, 1.0, 1e-310, 5e-324, 1e-308, 0.0, -0.0, np.nan, 3.0, 1e300, 1e-300, 7.0, 3.0]
    tx, ty = torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()
    counts = torch.zeros(4, dtype=torch.int64, device="cuda")
    fn = _lib.lib().fv3b_selftest_fastmath
    fn.restype = ctypes.c_int
    fn.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    rc = fn(tx.data_ptr(), ty.data_ptr(), n, counts.data_ptr(), torch.cuda.current_stream().cuda_stream)
    assert rc == 0, _lib.lib().fv3b_last_error()
    c = counts.cpu().tolist()
    assert c[0] == 0, f"{c[0]} fast-path quotients differ from IEEE division"
    assert c[2] == 0, f"{c[2]} fast-path logs differ from det_log"
    # the realistic half is (almost) always on the fast path
    assert c[1] < n // 2 and c[3] < n // 2, c
