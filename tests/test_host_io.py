"""Host-side logic of the end-to-end path (CPU): step_host's transfer runs
(Dycore._runs) merge consecutive fields that are adjacent in one storage on
both sides into a single copy and nothing else; and LoopbackCluster rejects
device barriers without peer-store halos."""

from __future__ import annotations

import pytest
import torch

from paper_2205_04148_b200.dycore import Dycore


def _block(names, shape=(3, 4, 5)):
    b = torch.arange(len(names) * 60, dtype=torch.float64).reshape((len(names),) + shape)
    return {n: b[t] for t, n in enumerate(names)}


def test_runs_merge_adjacent_fields():
    names = ["gz", "u", "v", "w"]
    a, b = _block(names), _block(names)
    runs = Dycore._runs(names, a, b)
    assert len(runs) == 1
    x, y = runs[0]
    assert x.numel() == 4 * 60 and x.data_ptr() == a["gz"].data_ptr()
    # a tail of the block still merges; a gap splits
    assert len(Dycore._runs(["u", "v"], a, b)) == 1
    assert len(Dycore._runs(["gz", "v"], a, b)) == 2


def test_runs_split_when_either_side_is_not_adjacent():
    names = ["gz", "u", "v"]
    a = _block(names)
    b = {n: torch.zeros(3, 4, 5, dtype=torch.float64) for n in names}  # separate allocations
    runs = Dycore._runs(names, a, b)
    assert len(runs) == 3
    for (x, y), n in zip(runs, names):
        assert x.data_ptr() == a[n].data_ptr() and y.data_ptr() == b[n].data_ptr()


def test_runs_copy_equals_per_field_copy():
    names = ["gz", "u", "v", "w", "delp"]
    a = _block(names)
    b = {n: t for n, t in _block(names).items()}
    for t in b.values():
        t.zero_()
    for x, y in Dycore._runs(names, b, a):
        x.copy_(y)
    for n in names:
        assert torch.equal(a[n], b[n])


def test_flag_sync_needs_peer_halos():
    from paper_2205_04148_b200.parallel import LoopbackCluster

    class _H:
        direct = False

    class _D:
        halo = None

    with pytest.raises(ValueError):
        LoopbackCluster([_D(), _D()], 1, 2, halos=[_H(), _H()], flag_sync=True)


def test_flag_sync_word_addresses():
    """FlagSync's buffer fields: rank r release-stores into column r of each
    neighbour's flag array and waits on the neighbours' columns of its own;
    phase 0 bumps the counter, phase 1 reuses it; self-neighbours are skipped."""
    from paper_2205_04148_b200.parallel import FlagSync, new_flags

    world, rank = 4, 1
    flags = [new_flags(world, "cpu") for _ in range(world)]
    fs = FlagSync(rank, [0, 2, 1, 2], flags[rank], dict(enumerate(flags)))
    for phase in (0, 1):
        farr, nf, sarr, ns = fs._args[phase]
        f = [farr[i] for i in range(nf)]
        assert all(x.rank == 1 and x.shape[0] >= 1 for x in f)
        assert f[0].data == fs.epoch.data_ptr() and f[1].data == fs.err.data_ptr()
        assert ns == 2 and sarr[0] == (1.0 if phase == 0 else 0.0) and sarr[1] == 2.0  # neighbours 0 and 2
        assert nf == 2 + 2 * 2
        for q, p in enumerate([0, 2]):
            remote, local = f[2 + 2 * q].data, f[3 + 2 * q].data
            assert remote == flags[p].data_ptr() + 8 * (phase * world + rank)
            assert local == flags[rank].data_ptr() + 8 * (phase * world + p)

@pytest.mark.parametrize("ni,nj,nk,h", [(192, 192, 80, 4), (32, 24, 10, 4), (7, 5, 3, 2)])
def test_interior_rows_cover_exactly_the_interior(ni, nj, nk, h):
    """step_host's pitched interior upload (dycore.interior_rows): the rows
    of (offset + r * pitch, width) bytes of a reference-convention array are
    exactly its interior columns over every level, in order."""
    import numpy as np

    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import interior_rows

    cfg = RunConfig(ni=ni, nj=nj, nk=nk, halo=h)
    a = np.arange((ni + 2 * h) * (nj + 2 * h) * (nk + 1), dtype=np.float64).reshape(ni + 2 * h, nj + 2 * h, nk + 1)
    flat = a.ravel()
    off, width, rows, pitch = interior_rows(cfg)
    assert rows == ni and off % 8 == 0 and width % 8 == 0 and pitch % 8 == 0
    got = np.stack([flat[(off + r * pitch) // 8:(off + r * pitch + width) // 8] for r in range(rows)])
    assert np.array_equal(got, a[h:h + ni, h:h + nj, :].reshape(ni, -1))
