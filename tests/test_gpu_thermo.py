"""fv3b_moist_pk (csrc/thermo.cu) bitwise against the oracle restatement
(oracle/thermo.py): pe, peln, pk at the interfaces, pkz and the moist cv at
the layers, for 0..6 water species, ragged domains, and exponents spread
over most of the normal range of exp (det_exp's every branch)."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import thermo

pytestmark = pytest.mark.gpu


def _run(delp, qs, nk, sc):
    import torch

    from paper_2205_04148_b200 import _lib
    from paper_2205_04148_b200.device import Grid

    ni, nj = delp.shape[:2]
    g = Grid(ni, nj, nk, halo=3)

    def up(a):
        t = g.new3("cuda")
        g.interior(t, nk)[...] = torch.from_numpy(np.ascontiguousarray(a.transpose(2, 1, 0)))
        return t

    outs = [g.new3("cuda") for _ in range(5)]
    ins = [up(delp)] + [up(q) for q in qs]  # (kept alive until the launch has run)
    fields = [g.abi(t) for t in ins] + [g.abi(o) for o in outs]
    _lib.call("fv3b_moist_pk", fields, sc, g.domain(nk=nk + 1), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    res = {}
    for n, o in zip(("pe", "peln", "pk", "pkz", "cvm"), outs):
        lv = nk + 1 if n in ("pe", "peln", "pk") else nk
        res[n] = g.interior(o, lv).cpu().numpy().transpose(2, 1, 0)
    return res


@pytest.mark.parametrize("ni,nj,nk,nw,akap,ptop,seed", [
    (32, 8, 80, 6, 287.05 / 1004.6, 300.0, 1),
    (37, 5, 24, 3, 287.05 / 1004.6, 300.0, 2),   # ragged, 3 species
    (17, 3, 7, 0, 0.5, 1.0, 3),                   # dry
    (48, 48, 60, 6, 25.0, 1e-6, 4),               # akap * peln from -345 to +290
    (20, 6, 30, 1, -3.0, 0.5, 5),                 # negative exponents, |x| < 0.5 ln2 .. 35
    (192, 192, 80, 6, 287.05 / 1004.6, 300.0, 6),  # the C2 column count
    (5, 3, 1, 2, 287.05 / 1004.6, 300.0, 7),      # a single layer (program domain nk = 2)
    (1, 1, 2, 6, 287.05 / 1004.6, 300.0, 8),      # a single column
])
def test_moist_pk_bitwise_vs_oracle(ni, nj, nk, nw, akap, ptop, seed):
    from paper_2205_04148_b200.config import RunConfig

    rng = np.random.default_rng(seed)
    delp = (1e5 - ptop) / nk * (1 + 0.6 * rng.uniform(-1, 1, (ni, nj, nk)))
    qs = [1e-3 * rng.uniform(0, 2, (ni, nj, nk)) for _ in range(nw)]
    sc = RunConfig().moist_scalars()
    sc[0], sc[1] = ptop, akap
    got = _run(delp, qs, nk, sc)
    want = thermo.moist_pk(delp, qs, nk, sc)
    for n in want:
        assert np.array_equal(got[n], want[n]), f"{n}: max diff {np.abs(got[n] - want[n]).max()}"
