"""Cubed-sphere halo specification (cubesphere.py) on CPU.

* the tile connectivity and edge maps fold onto a real cube: every tile gets
  a consistent 3-D frame on a distinct face, and every edge-halo cell lands on
  the neighbour's interior cell occupying the same point of the cube surface;
* the NumPy oracle of the six-tile step runs and stays finite.
"""

from __future__ import annotations

import numpy as np
import pytest

from paper_2205_04148_b200.cubesphere import _edge_cells, _point_map, _position, _stagger, edge_entries, role, topology


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


def _frames(n, h):
    """The tiles' 3-D frames on the cube (as in test_connectivity_folds_onto_a_cube)."""
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
    return frames


def _unfolded_axes(frame, X, Y, n, beyond):
    """The tile's local x / y axes continued across its edge (the fold's
    derivatives); on the edge line itself (u or v == 0 or n) the one-sided
    derivative of the neighbour's side (`beyond`)."""
    O, a, b = frame
    c = np.cross(a, b)
    u, v = X + 0.5, Y + 0.5
    if v > n or (beyond == "N" and v >= n):
        return a, -c
    if v < 0 or (beyond == "S" and v <= 0):
        return a, c
    if u > n or (beyond == "E" and u >= n):
        return -c, b
    if u < 0 or (beyond == "W" and u <= 0):
        return c, b
    return a, b


def test_vector_halo_matches_a_solid_body_rotation():
    """Rotated vector halos against geometry: a 3-D solid-body
    rotation V = omega x (p - centre) sampled at every staggered point.  Each
    tile stores the components of V along its own axes (D-grid u, v at
    south / west edges; C-grid uc, vc at west / south edges); every edge-halo
    entry (rotation, component swap, sign, staggered shift) must reproduce
    the component of V along the tile's axes continued across the edge, at
    the halo point.  Known approximation: the 3 halo cells per tile where a
    rotated component's staggered point lies on the edge line next to
    a cube vertex take their source from the neighbour's last interior cell
    (the true source lies on the neighbour's own boundary line, owned by a
    third tile; cubesphere.edge_entries clamps), one cell away; they are
    listed exactly (u, v, uc, vc: 3 cells each per tile)."""
    n, h = 8, 3
    F = _frames(n, h)
    om, ctr = np.array([0.3, -0.5, 0.8]), np.full(3, n / 2)

    def V(p):
        return np.cross(om, p - ctr)

    clamped = []
    for t in range(6):
        for names in (["u", "v"], ["uc", "vc"]):
            for e in edge_entries(t, names, n, h):
                r = role(e.name)[0]
                dx, dy = _stagger(_position(e.name))
                X, Y = e.i + dx, e.j + dy
                side = "W" if e.i < 0 else "E" if e.i >= n else "S" if e.j < 0 else "N"
                P = _fold(F[t], X, Y, n)
                ax, ay = _unfolded_axes(F[t], X, Y, n, side)
                want = V(P) @ (ax if r == "x" else ay)
                sx, sy = _stagger(_position(e.src_name))
                Ps = _local(F[e.src_tile], e.si + sx, e.sj + sy)
                O, a, b = F[e.src_tile]
                got = e.sign * (V(Ps) @ (a if role(e.src_name)[0] == "x" else b))
                if np.linalg.norm(P - Ps) > 1e-9:
                    clamped.append((t, e.name, e.i, e.j))
                    continue
                assert abs(got - want) < 1e-9, (t, e.name, e.i, e.j, got, want)
    # exactly the vertex-adjacent cells: 3 per tile for each of u, v, uc, vc,
    # all with the staggered point on the tile's edge line
    assert len(clamped) == 72 and {c[1] for c in clamped} == {"u", "v", "uc", "vc"}
    for t, name, i, j in clamped:
        south = name in ("u", "vc")  # staggered to the cell's south edge, else its west edge
        on_line = j in (0, n) if south else i in (0, n)
        assert on_line and (i < 0 or i >= n or j < 0 or j >= n), (t, name, i, j)
