"""GPU parity of the remap mapping (fv3b_remap_map, FV3 map1_ppm) against the
oracle restatement (oracle/remap_map.py): bitwise on seeded columns whose
Lagrangian layers are strongly perturbed (target layers spanning several
source layers and several target layers inside one source layer), plus
ragged domains, 1..16 tracers and the C2 column count."""

from __future__ import annotations

import numpy as np
import pytest

from oracle import remap_map as rm

pytestmark = pytest.mark.gpu


def _case(ni, nj, nk, nq, seed, spread):
    rng = np.random.default_rng(seed)
    delp = (1.0e5 - 300.0) / nk * (1.0 + spread * rng.uniform(-1, 1, (ni, nj, nk)))
    qs = []
    for _ in range(nq):
        q = rng.uniform(0.5, 2.0, (ni, nj, nk))
        a2 = q + 0.1 * rng.uniform(-1, 1, q.shape)
        a3 = q + 0.1 * rng.uniform(-1, 1, q.shape)
        a4 = 3.0 * (2.0 * q - (a2 + a3))
        qs.append((q, a2, a3, a4))
    return delp, qs


def _run_device(delp, qs, nk, ptop=300.0):
    import torch

    from paper_2205_04148_b200 import _lib
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.device import Grid

    ni, nj = delp.shape[:2]
    g = Grid(ni, nj, nk, halo=3)
    cfg = RunConfig(ni=ni, nj=nj, nk=nk)
    ak, bk = cfg.target_coordinate()

    def up(a):
        t = g.new3("cuda")
        g.interior(t, nk)[...] = torch.from_numpy(np.ascontiguousarray(a.transpose(2, 1, 0)))
        return t

    td = up(delp)
    tak, tbk = torch.from_numpy(ak).cuda(), torch.from_numpy(bk).cuda()
    tq = [[up(x) for x in qq] for qq in qs]
    tout = [g.new3("cuda") for _ in qs]
    fields = [g.abi(td), g.abi(tak, rank=1), g.abi(tbk, rank=1)]
    for qq, o in zip(tq, tout):
        fields += [g.abi(x) for x in qq] + [g.abi(o)]
    _lib.call("fv3b_remap_map", fields, [], g.domain(nk=nk + 1), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    down = lambda t: g.interior(t, nk).cpu().numpy().transpose(2, 1, 0)
    return down(td), [down(o) for o in tout], ak, bk


@pytest.mark.parametrize("ni,nj,nk,nq,spread,seed", [
    (32, 8, 16, 1, 0.3, 1),
    (37, 5, 24, 3, 0.9, 2),     # ragged, thick/thin layers (multi-layer spans)
    (48, 48, 80, 8, 0.5, 3),
    (17, 3, 7, 16, 0.95, 4),
    (192, 192, 80, 2, 0.3, 5),  # the C2 column count
    (5, 3, 1, 2, 0.5, 6),       # a single layer: the whole column into one target layer
    (1, 1, 2, 1, 0.9, 7),       # a single column
])
def test_remap_map_bitwise_vs_oracle(ni, nj, nk, nq, spread, seed):
    delp, qs = _case(ni, nj, nk, nq, seed, spread)
    d_delp, d_q, ak, bk = _run_device(delp, qs, nk)
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    for t, (q, a2, a3, a4) in enumerate(qs):
        want = rm.map_columns(pe1, pe2, q, a2, a3, a4, nk)
        assert np.array_equal(d_q[t], want), f"tracer {t}: max diff {np.abs(d_q[t] - want).max()}"
    assert np.array_equal(d_delp, pe2[..., 1:] - pe2[..., :-1])
    # conservation of the column integral (a property of the method)
    before = (qs[0][0] * delp).sum(axis=-1)
    after = (d_q[0] * d_delp).sum(axis=-1)
    assert np.allclose(after, before, rtol=1e-11)


def test_remap_map_rejects_aliased_output():
    import torch

    from paper_2205_04148_b200 import _lib
    from paper_2205_04148_b200.device import Grid

    g = Grid(8, 8, 4, halo=3)
    t = [g.new3("cuda") for _ in range(5)]
    ak = torch.zeros(5, dtype=torch.float64, device="cuda")
    fields = [g.abi(t[0]), g.abi(ak, rank=1), g.abi(ak, rank=1)] + [g.abi(x) for x in t[1:]] + [g.abi(t[1])]
    with pytest.raises(_lib.Fv3bError):
        _lib.call("fv3b_remap_map", fields, [], g.domain(nk=5), torch.cuda.current_stream().cuda_stream)


def test_transpose_round_trip_bitwise():
    """fv3b_transpose: reference (I, J, K) order <-> Layout window, both ways,
    on a ragged shape (tile edges in I, J and K)."""
    import torch

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore

    cfg = RunConfig(ni=37, nj=21, nk=45, nq=1, n_split=1)
    d = Dycore(cfg)
    h = cfg.halo
    shape = (cfg.ni + 2 * h, cfg.nj + 2 * h, cfg.nk + 1)
    src = torch.from_numpy(np.random.default_rng(9).standard_normal(shape)).cuda()
    d._transpose(src, d._window(d.cur["pt"]))
    assert torch.equal(d._window(d.cur["pt"]), src)
    back = torch.empty_like(src)
    d._transpose(d._window(d.cur["pt"]), back)
    torch.cuda.synchronize()
    assert torch.equal(back, src)


def _grid_fields(ni, nj, nk):
    from paper_2205_04148_b200.device import Grid

    return Grid(ni, nj, nk, halo=3)


def _log_coordinate(g, td, ak, bk, nk):
    """fv3b_log_thickness on device delp ``td``: (dlnp, lnpe1, lnpe2) tensors."""
    import torch

    from paper_2205_04148_b200 import _lib

    out = [g.new3("cuda") for _ in range(3)]
    coord = [torch.from_numpy(x).cuda() for x in (ak, bk)]
    _lib.call("fv3b_log_thickness", [g.abi(td)] + [g.abi(c, rank=1) for c in coord] + [g.abi(t) for t in out], [],
              g.domain(nk=nk), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("ni,nj,nk,seed", [(32, 8, 16, 1), (37, 5, 80, 2), (1, 1, 3, 3)])
def test_log_thickness_bitwise_vs_oracle(ni, nj, nk, seed):
    """fv3b_log_thickness: log(pe1), log(pe2) of the running-sum interfaces
    and the target coordinate, and dlnp their layer differences
    (oracle/remap_map.py log_edges / log_thickness)."""
    import torch

    from paper_2205_04148_b200.config import RunConfig

    delp, _ = _case(ni, nj, nk, 0, seed, 0.6)
    ak, bk = RunConfig(ni=ni, nj=nj, nk=nk).target_coordinate()
    g = _grid_fields(ni, nj, nk)
    td = g.new3("cuda")
    g.interior(td, nk)[...] = torch.from_numpy(np.ascontiguousarray(delp.transpose(2, 1, 0)))
    tl, t1, t2 = _log_coordinate(g, td, ak, bk, nk)
    down = lambda t, n: g.interior(t, n).cpu().numpy().transpose(2, 1, 0)
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    l1, l2 = rm.log_edges(pe1, pe2)
    assert np.array_equal(down(tl, nk), rm.log_thickness(delp, ak, nk))
    assert np.array_equal(down(t1, nk + 1), l1)
    assert np.array_equal(down(t2, nk + 1), l2)


@pytest.mark.parametrize("ni,nj,nk,nq,spread,seed", [(32, 8, 16, 1, 0.3, 1), (37, 5, 24, 2, 0.9, 2),
                                                     (48, 48, 80, 1, 0.5, 3)])
def test_remap_map_log_group_bitwise_vs_oracle(ni, nj, nk, nq, spread, seed):
    """A log-pressure group (negative group size: FV3's pt with kord_tm < 0,
    its slot holding log(pe1) then log(pe2)) beside a linear group: the log
    group maps on log(pe1) -> log(pe2) and rewrites nothing; the linear
    group maps and rewrites its thickness."""
    import torch

    from paper_2205_04148_b200 import _lib
    from paper_2205_04148_b200.config import RunConfig

    delp, qs = _case(ni, nj, nk, nq, seed, spread)
    other, qo = _case(ni, nj, nk, 1, seed + 10, spread)
    ak, bk = RunConfig(ni=ni, nj=nj, nk=nk).target_coordinate()
    g = _grid_fields(ni, nj, nk)

    def up(a):
        t = g.new3("cuda")
        g.interior(t, nk)[...] = torch.from_numpy(np.ascontiguousarray(a.transpose(2, 1, 0)))
        return t

    td, tother = up(delp), up(other)
    _, t1, t2 = _log_coordinate(g, td, ak, bk, nk)
    tq = [[up(x) for x in qq] for qq in qs]
    tqo = [up(x) for x in qo[0]]
    tout = [g.new3("cuda") for _ in qs]
    tout2 = g.new3("cuda")
    coord = [torch.from_numpy(x).cuda() for x in (ak, bk)]
    fields = [g.abi(c, rank=1) for c in coord] + [g.abi(t1), g.abi(t2)]
    for qq, o in zip(tq, tout):
        fields += [g.abi(x) for x in qq] + [g.abi(o)]
    fields.append(g.abi(tother))
    fields += [g.abi(x) for x in tqo] + [g.abi(tout2)]
    _lib.call("fv3b_remap_map", fields, [-float(nq), 1.0], g.domain(nk=nk + 1), torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    down = lambda t, n=nk: g.interior(t, n).cpu().numpy().transpose(2, 1, 0)
    pe1, pe2 = rm.pe_edges(delp, ak, bk, nk)
    l1, l2 = rm.log_edges(pe1, pe2)
    for t, (q, a2, a3, a4) in enumerate(qs):
        assert np.array_equal(down(tout[t]), rm.map_columns(l1, l2, q, a2, a3, a4, nk)), t
    assert np.array_equal(down(t1, nk + 1), l1) and np.array_equal(down(td), delp)  # nothing rewritten
    p1, p2 = rm.pe_edges(other, ak, bk, nk)
    q, a2, a3, a4 = qo[0]
    assert np.array_equal(down(tout2), rm.map_columns(p1, p2, q, a2, a3, a4, nk))
    assert np.array_equal(down(tother), p2[..., 1:] - p2[..., :-1])


def test_remap_map_rejects_log_group_without_its_target_interfaces():
    import torch

    from paper_2205_04148_b200 import _lib

    g = _grid_fields(8, 8, 4)
    t = [g.new3("cuda") for _ in range(6)]
    ak = torch.zeros(5, dtype=torch.float64, device="cuda")
    fields = [g.abi(ak, rank=1), g.abi(ak, rank=1), g.abi(t[0])] + [g.abi(x) for x in t[1:6]]
    with pytest.raises(_lib.Fv3bError):
        _lib.call("fv3b_remap_map", fields, [-1.0], g.domain(nk=5), torch.cuda.current_stream().cuda_stream)
