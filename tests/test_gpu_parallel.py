"""Decomposed dycore on one B200: the CUDA pack / unpack kernels
(fv3b_halo_pack_rects / unpack_rects) reproduce the single-rank periodic halo
kernel, and a 2 x 2 (and 1 x 2) decomposition advanced in lockstep with
device-copy transport (parallel.LoopbackCluster) is bitwise the single-domain
dycore on every block."""

from __future__ import annotations

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _block(a, ri, rj, ni, nj, h):
    NI, NJ = a.shape[0] - 2 * h, a.shape[1] - 2 * h
    ii = (np.arange(ri * ni - h, (ri + 1) * ni + h) % NI) + h
    jj = (np.arange(rj * nj - h, (rj + 1) * nj + h) % NJ) + h
    return a[np.ix_(ii, jj)]


class _SelfTransport:
    def exchange(self, send, recv):
        rb = dict(recv)
        for p, t in send:
            assert p == 0
            rb[p].copy_(t)


def test_device_packer_single_rank_equals_periodic_kernel():
    import torch

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import DecomposedHalo

    cfg = RunConfig(ni=40, nj=24, nk=6, nq=2)
    a = Dycore(cfg)
    b = Dycore(cfg)
    g = torch.Generator(device="cuda").manual_seed(3)
    names = ["u", "v", "w", "q0", "q1"]
    for n in names:
        a.cur[n].copy_(torch.rand(a.cur[n].shape, generator=g, device="cuda", dtype=torch.float64))
        b.cur[n].copy_(a.cur[n])
    a.halo.update(names)
    DecomposedHalo(b, 1, 1, 0, transport=_SelfTransport()).update(names)
    torch.cuda.synchronize()
    for n in names:
        assert torch.equal(a.cur[n], b.cur[n]), n


@pytest.mark.parametrize("px,py", [(2, 2), (1, 2)])
def test_loopback_decomposed_dycore_bitwise(px, py):
    import torch

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.parallel import LoopbackCluster
    from paper_2205_04148_b200.state import initial_state

    ni, nj, nk = 32, 24, 8
    glob_cfg = RunConfig(ni=px * ni, nj=py * nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
    blk_cfg = RunConfig(ni=ni, nj=nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
    st = initial_state(glob_cfg)
    h = glob_cfg.halo
    ref = Dycore(glob_cfg, st)
    blocks = []
    for r in range(px * py):
        ri, rj = r % px, r // px
        blocks.append(Dycore(blk_cfg, {n: _block(a, ri, rj, ni, nj, h) for n, a in st.items()}))
    cluster = LoopbackCluster(blocks, px, py)
    for _ in range(2):
        ref.step()
        cluster.step()
    torch.cuda.synchronize()
    names = ["u", "v", "w", "delp", "pt", "gz", "pef", "q0", "q1", "q1_a4", "mfx", "cy"]
    full = ref.download(names)
    for r, d in enumerate(blocks):
        ri, rj = r % px, r // px
        got = d.download(names)
        for n in names:
            want = _block(full[n], ri, rj, ni, nj, h)[h:-h, h:-h]
            assert np.array_equal(got[n][h:-h, h:-h], want), (r, n)
