"""CPU oracle of the cubed-sphere halo update and of the six-tile dycore
step (config C3).

TEST INFRASTRUCTURE ONLY (tests/, bench CPU legs).  The halo maps are the
specification in ``paper_2205_04148_b200/cubesphere.py`` (host logic: tile
connectivity, edge rotation, corner fill); this module applies them with
NumPy fancy indexing to the six tiles' reference-convention arrays (axes I,
J, K, uniform halo h), and steps six :class:`oracle.dycore.OracleDycore`
tiles (placement FULL_TILE: every tile edge region fires) in lockstep.
"""

from __future__ import annotations

import numpy as np

from paper_2205_04148_b200.cubesphere import check_names, corner_entries, edge_entries

from .dycore import OracleDycore
from .interp import FULL_TILE


def cube_halo(tiles: list[dict[str, np.ndarray]], names, n: int, h: int) -> None:
    """Refresh the halos of `names` on all six tiles (in place)."""
    check_names(names)
    # edges: every value comes from a neighbour's interior (read before any write)
    vals = []
    for t in range(6):
        ent = edge_entries(t, names, n, h)
        vals.append([(e, e.sign * tiles[e.src_tile][e.src_name][e.si + h, e.sj + h]) for e in ent])
    for t in range(6):
        for e, v in vals[t]:
            tiles[t][e.name][e.i + h, e.j + h] = v
    # corners: from the tile's own (now filled) edge halos
    ent = corner_entries(names, n, h)
    for t in range(6):
        vv = [(e, e.sign * tiles[t][e.src_name][e.si + h, e.sj + h]) for e in ent]
        for e, v in vv:
            tiles[t][e.name][e.i + h, e.j + h] = v


class OracleCube:
    """Six FULL_TILE oracle dycores with the cubed-sphere halo."""

    def __init__(self, cfg, states: list[dict[str, np.ndarray]]):
        assert cfg.ni == cfg.nj
        self.cfg = cfg
        self.tiles = [OracleDycore(cfg, st, placement=FULL_TILE) for st in states]

    def step(self) -> None:
        gens = [t.phases() for t in self.tiles]
        while True:
            reqs = [next(g, None) for g in gens]
            if all(r is None for r in reqs):
                return
            cube_halo([t.state for t in self.tiles], reqs[0], self.cfg.ni, self.cfg.halo)
