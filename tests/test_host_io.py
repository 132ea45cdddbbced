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
