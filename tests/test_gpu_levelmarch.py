"""GPU parity of the benchmarked kernel shapes.

The level-marching tile kernels (d_sw transport / momentum, c_sw, tracer_2d,
fv_tp_2d) give each CTA a chunk of consecutive levels; at C2 the automatic
chunk is 40-80 levels, so the TMA refill of the next level (``issue(k + 1)``),
the mbarrier parity flip and tracer_2d's level-boundary restaging all run.
Small test domains get a chunk of 1, so these tests force the chunk with the
``fv3b_tune_set`` knob (kchunk 2, 3, 5 and nk: ragged last chunks included)
and also run the programs and the full timestep at the C2 size itself.
Semantics matched: statement-major level loop, ``reference.py:284-304``.
Everything is bitwise against the oracle (no ``**``; -fmad=false).
"""

from __future__ import annotations

import numpy as np
import pytest

from helpers import assert_outputs_equal
from oracle import interp

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def engine():
    import torch

    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2205_04148_b200 import executor

    return executor


def _tuning(**k):
    from paper_2205_04148_b200 import _lib

    return _lib.tuning(**k)


MARCH = [
    ("d_sw", (48, 48, 16), "kchunk_dsw_transport"),
    ("d_sw", (48, 48, 16), "kchunk_dsw_momentum"),
    ("d_sw", (48, 48, 16), "kchunk"),
    ("c_sw", (48, 48, 16), "kchunk_csw"),
    ("c_grid", (48, 48, 17), "kchunk_csw"),
    ("tracer_2d", (48, 48, 16), "kchunk_tracer"),
    ("fv_tp_2d", (48, 48, 16), "kchunk_fv_tp_2d"),
]


@pytest.mark.parametrize("kchunk", [2, 3, 5, 16])
@pytest.mark.parametrize("name,domain,knob", MARCH)
def test_level_march_chunks_bitwise(engine, name, domain, knob, kchunk):
    from paper_2205_04148_b200.inputs import synthetic_inputs

    inputs = synthetic_inputs(name, domain, 100 + kchunk)
    ref = interp.run_program(name, inputs, domain, interp.PERIODIC)
    with _tuning(**{knob: kchunk}):
        got = engine.run_b200(name, inputs, domain, placement=(False,) * 4)
    assert_outputs_equal(got, ref)


@pytest.mark.parametrize("name,domain", [("d_sw", (37, 21, 7)), ("c_grid", (33, 19, 9)), ("tracer_2d", (35, 29, 7))])
def test_level_march_full_tile_ragged(engine, name, domain):
    """Partial tiles, full-tile placement (edge regions fire) and a ragged
    level chunk (3 into 7 or 8 layers) at once."""
    from paper_2205_04148_b200.inputs import synthetic_inputs

    inputs = synthetic_inputs(name, domain, 31)
    ref = interp.run_program(name, inputs, domain, interp.Placement(True, True, True, True))
    with _tuning(kchunk=3):
        got = engine.run_b200(name, inputs, domain, placement=(True,) * 4)
    assert_outputs_equal(got, ref)


C2 = [
    ("d_sw", (192, 192, 80)),
    ("c_grid", (192, 192, 81)),
    ("c_sw", (192, 192, 80)),
    ("nh_d", (192, 192, 81)),
    ("p_grad_d", (192, 192, 81)),
    ("tracer_2d", (192, 192, 80)),
]


@pytest.mark.parametrize("name,domain", C2)
def test_program_at_c2_size_bitwise(engine, name, domain):
    """The programs of the C2 step at 192 x 192 x 80 (interface programs
    81), with the automatic (benchmarked) launch shapes."""
    from paper_2205_04148_b200.inputs import synthetic_inputs

    inputs = synthetic_inputs(name, domain, 2205)
    got = engine.run_b200(name, inputs, domain, placement=(False,) * 4)
    ref = interp.run_program(name, inputs, domain, interp.PERIODIC)
    assert_outputs_equal(got, ref)


INTERFACE = ("gz", "pef", "pe", "peln", "pk")


def _compare(cfg, gpu: dict, st: dict, names):
    h = cfg.halo
    for n in names:
        top = cfg.nk + 1 if n in INTERFACE else cfg.nk
        a = gpu[n][h:-h, h:-h, :top]
        b = st[n][h:-h, h:-h, :top]
        assert np.isfinite(b).all(), n
        if not np.array_equal(a, b):
            err = np.max(np.abs(a - b) / np.maximum(np.abs(b), 1e-300))
            raise AssertionError(f"{n}: {int((a != b).sum())} cells differ, max rel err {err:.3e}")


SUBSTEP_FIELDS = ["u", "v", "w", "delp", "pt", "gz", "pef", "uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy", "dp1"]


@pytest.mark.parametrize("kchunk", [0, 4])
def test_c1_acoustic_substep_bitwise(kchunk):
    """BASELINE config C1: one acoustic substep (halo, c_sw + riem_solver_c +
    p_grad_c, halo, d_sw, nh_d, halo, p_grad_d) at 48 x 48 x 16, doubly
    periodic, bitwise against the oracle step driver."""
    import torch

    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig(ni=48, nj=48, nk=16, n_split=6, dt_atmos=90.0)
    d = Dycore(cfg, initial_state(cfg))
    with _tuning(kchunk=kchunk):
        d.substep(first=True)
        torch.cuda.synchronize()
    gpu = d.download(SUBSTEP_FIELDS)
    st = initial_state(cfg)
    OracleDycore(cfg, st).substep(first=True)
    _compare(cfg, gpu, st, SUBSTEP_FIELDS)


STEP_FIELDS = ["u", "v", "w", "delp", "pt", "gz", "pef", "q0", "q3", "q7", "q5_a4", "mfx", "cy", "pe", "peln", "pk",
               "pkz", "cvm"]


def test_dycore_kchunk_forced_3_steps_bitwise():
    """Three full timesteps with every level-marching kernel on 3-level
    chunks (ragged into 10 layers), graph replay, against the oracle."""
    import torch

    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig(ni=32, nj=24, nk=10, n_split=3, dt_atmos=45.0)
    d = Dycore(cfg, initial_state(cfg))
    with _tuning(kchunk=3):
        d.capture()
        for _ in range(3):
            d.replay()
        torch.cuda.synchronize()
    gpu = d.download(STEP_FIELDS)
    st = initial_state(cfg)
    ref = OracleDycore(cfg, st)
    for _ in range(3):
        ref.step()
    _compare(cfg, gpu, st, STEP_FIELDS)


def test_c2_full_timestep_bitwise():
    """BASELINE config C2, the benchmarked workload: one full 192 x 192 x 80
    timestep (n_split = 6, nq = 8, remapping and diagnostics) as a CUDA
    graph, bitwise against the oracle step driver (about 2-3 CPU minutes)."""
    import torch

    from oracle.dycore import OracleDycore
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig()
    d = Dycore(cfg, initial_state(cfg))
    d.capture()
    d.replay()
    torch.cuda.synchronize()
    gpu = d.download(STEP_FIELDS)
    st = initial_state(cfg)
    OracleDycore(cfg, st).step()
    _compare(cfg, gpu, st, STEP_FIELDS)
