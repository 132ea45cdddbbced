"""Cubed-sphere halo specification (cubesphere.py) on CPU.

* the tile connectivity and edge maps fold onto a real cube: every tile gets
  a consistent 3-D frame on a distinct face, and every edge-halo cell lands on
  the neighbour's interior cell occupying the same point of the cube surface;
* the NumPy oracle of the six-tile step runs and stays finite.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2205_04148_b200.cubesphere import _edge_cells, _point_map, edge_entries, topology


def _fold(frame, X, Y, n):
    O, a, b = frame
    c = np.cross(a, b)
    u, v = X + 0.5, Y + 0.5
    if v > n:
        return O + u * a + n * b - (v - n) * c
    if v < 0:
        return O + u * a + v * c
    if u > n:
        return O + n * a + v * b - (u - n) * c
    if u < 0:
        return O + v * b + u * c
    return O + u * a + v * b


def _local(frame, Xp, Yp):
    O, a, b = frame
    return O + (Xp + 0.5) * a + (Yp + 0.5) * b


def test_connectivity_folds_onto_a_cube():
    n, h = 8, 3
    topo = topology()
    frames = {0: (np.array([0.0, 0.0, n]), np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0]))}
    todo = [0]
    while todo:
        t = todo.pop()
        for side, sd in topo[t].items():
            if sd.nb in frames:
                continue
            pmap, _ = _point_map(side, sd.rot, n)
            rows, pts = [], []
            for (i, j) in _edge_cells(side, n, h):
                Xp, Yp = pmap(float(i), float(j))
                rows.append([1.0, Xp + 0.5, Yp + 0.5])
                pts.append(_fold(frames[t], i, j, n))
            sol, *_ = np.linalg.lstsq(np.array(rows), np.array(pts), rcond=None)
            frames[sd.nb] = (sol[0], sol[1], sol[2])
            todo.append(sd.nb)
    assert sorted(frames) == list(range(6))
    centre = np.full(3, n / 2)
    normals = set()
    for t, (O, a, b) in frames.items():
        c = np.cross(a, b)
        for v in (a, b, c):
            assert np.allclose(np.sort(np.abs(v)), [0, 0, 1]), (t, v)
        # outward: the face centre sits n/2 along the normal from the cube centre
        assert np.allclose(O + (n / 2) * (a + b) - centre, (n / 2) * c), t
        normals.add(tuple(np.round(c).astype(int)))
    assert len(normals) == 6
    # every edge-halo cell of every tile is the neighbour's interior cell at the same point
    for t in range(6):
        for side, sd in topo[t].items():
            pmap, _ = _point_map(side, sd.rot, n)
            for (i, j) in _edge_cells(side, n, h):
                Xp, Yp = pmap(float(i), float(j))
                assert 0 <= Xp < n and 0 <= Yp < n
                np.testing.assert_allclose(_fold(frames[t], i, j, n), _local(frames[sd.nb], Xp, Yp), atol=1e-9)


def test_edge_entries_scalars_cover_each_halo_strip_once():
    n, h = 6, 3
    for t in range(6):
        ent = edge_entries(t, ["delp"], n, h)
        cells = {(e.i, e.j) for e in ent}
        assert len(cells) == len(ent) == 4 * n * h
        assert all(0 <= e.si < n and 0 <= e.sj < n and e.src_tile != t for e in ent)


@pytest.mark.slow
def test_oracle_cube_step_is_finite():
    from oracle.cube import OracleCube
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.state import initial_state

    cfg = RunConfig(ni=12, nj=12, nk=4, n_split=2, dt_atmos=20.0)
    cube = OracleCube(cfg, [initial_state(RunConfig(ni=12, nj=12, nk=4, seed=2205 + t)) for t in range(6)])
    cube.step()
    h = cfg.halo
    for t in cube.tiles:
        for f in ("u", "v", "w", "delp", "pt", "q0"):
            assert np.isfinite(t.state[f][h:-h, h:-h, : cfg.nk]).all(), f
