"""CPU oracle of the full dycore timestep: the shipped programs executed by
the NumPy ``run_reference`` restatement (oracle/interp.py), glued by a NumPy
halo update — the reference's execution model with the paper's multi-program
Python step driver.

TEST INFRASTRUCTURE ONLY: used by tests/, __graft_entry__.smoke() and the
CPU-baseline / ``--impl reference`` legs of bench.py.

State arrays follow ``paper_2205_04148_b200.state`` (reference convention,
uniform halo, nk+1 levels).  For each program call the state is sliced to
the program's own allocation contract (the reference ``compute_requirements``
extents recorded in the manifest), executed, and the written fields are
copied back — exactly what a user of ``run_reference`` would do.
"""

from __future__ import annotations

import numpy as np

from . import interp, remap_map, thermo

PERIODIC = interp.PERIODIC

# program -> (vertical domain: "layers" | "interfaces", {program field: state field})
BINDINGS = {
    "c_grid": ("interfaces", {}),
    "d_sw": ("layers", {}),
    "nh_d": ("interfaces", {}),
    "p_grad_d": ("interfaces", {}),
    "tracer_2d": ("layers", {"xfx": "xfa", "yfx": "yfa"}),
    "remap_tracers": ("interfaces", {}),
    "remap_profile": ("interfaces", {}),
}


def _written(doc) -> set[str]:
    decl = {f["name"]: f for f in doc["program"]["fields"]}
    out = set()
    for s in doc["program"]["stencils"]:
        for b in s["blocks"]:
            for st in b["statements"]:
                if not decl[st["target"]]["temporary"]:
                    out.add(st["target"])
    return out


class OracleDycore:
    """NumPy step driver.  ``state`` is modified in place."""

    def __init__(self, cfg, state: dict[str, np.ndarray], placement=PERIODIC):
        self.cfg = cfg
        self.state = state
        self.placement = placement
        self.docs = {n: interp.load_manifest(n) for n in BINDINGS}
        self.written = {n: _written(d) for n, d in self.docs.items()}
        h, nk = cfg.halo, cfg.nk
        for q in cfg.remapped() + ["u", "v"]:
            for a in ("a2", "a3", "a4"):
                state.setdefault(f"{q}_{a}", np.zeros_like(state["delp"]))
        self._h = h

    def _slices(self, doc, name, nk_dom):
        h = self._h
        ni, nj = self.cfg.ni, self.cfg.nj
        ext = dict(zip("IJK", doc["requirements"]["extent"][name]))
        dims = next(f["dims"] for f in doc["program"]["fields"] if f["name"] == name)
        sl = []
        for a in dims:
            lo, hi = ext[a]
            if a == "I":
                sl.append(slice(h + lo, h + ni + hi))
            elif a == "J":
                sl.append(slice(h + lo, h + nj + hi))
            else:
                sl.append(slice(0 + lo, nk_dom + hi))
        return tuple(sl)

    def call(self, prog: str, consts: dict, bind: dict | None = None) -> None:
        doc = self.docs[prog]
        vert, bind0 = BINDINGS[prog]
        bind = {**bind0, **(bind or {})}
        nk_dom = self.cfg.nk if vert == "layers" else self.cfg.nk + 1
        inputs, slices = {}, {}
        for f in doc["program"]["fields"]:
            if f["temporary"]:
                continue
            name = f["name"]
            src = bind.get(name, name)
            sl = self._slices(doc, name, nk_dom)
            slices[name] = (src, sl)
            inputs[name] = self.state[src][sl]
        out = interp.run_program(doc, inputs, (self.cfg.ni, self.cfg.nj, nk_dom), self.placement, consts)
        for name in self.written[prog]:
            src, sl = slices[name]
            self.state[src][sl] = out[name]

    def halo(self, names) -> None:
        from paper_2205_04148_b200.state import periodic_fill

        for n in names:
            periodic_fill(self.state[n], self._h)

    def phases(self):
        """One timestep; yields the field lists to halo-update (the caller
        performs the update), mirroring ``Dycore.phases``."""
        cfg, st = self.cfg, self.state
        c = dict(cfg.consts)
        dt = cfg.dt_acoustic
        for n in ("cx", "cy", "xfa", "yfa", "mfx", "mfy"):
            st[n][...] = 0.0
        st["dp1"][...] = st["delp"]
        for _ in range(cfg.n_split):
            yield from self.acoustic_phases()
        yield cfg.tracer_names() + ["cx", "cy", "xfa", "yfa", "mfx", "mfy", "delp"]
        self.call("tracer_2d", c)
        self.call("remap_tracers", c)
        ak, bk = cfg.target_coordinate()
        # pt in log pressure (FV3 kord_tm < 0): its profile at the log-pressure thickness
        if cfg.pt_logp:
            st["dlnp"] = np.zeros_like(st["delp"])
            sl = (slice(self._h, -self._h), slice(self._h, -self._h))
            st["dlnp"][sl + (slice(0, cfg.nk),)] = remap_map.log_thickness(st["delp"][sl], ak, cfg.nk)
        for n in ("pt", "w"):  # the remap_profile program on each thermodynamic field
            bind = {"q": n, "a4_2": f"{n}_a2", "a4_3": f"{n}_a3", "a4_4": f"{n}_a4"}
            if n == "pt" and cfg.pt_logp:
                bind["delp"] = "dlnp"
            self.call("remap_profile", c, bind=bind)
        # the D-grid winds at their own thickness (remap_profile program, map1_ppm)
        st["du"], st["dv"] = remap_map.face_thickness(st["delp"], cfg.nk, self._h)
        for w, dw in (("u", "du"), ("v", "dv")):
            self.call("remap_profile", c,
                      bind={"q": w, "delp": dw, "a4_2": f"{w}_a2", "a4_3": f"{w}_a3", "a4_4": f"{w}_a4"})
        # (delp's rewrite comes last: the log-pressure mapping of pt reads it)
        if cfg.pt_logp:
            remap_map.remap_map(st, ["pt"], ak, bk, cfg.nk, self._h, log=True)
        for w, dw in (("u", "du"), ("v", "dv")):
            remap_map.remap_map(st, [w], ak, bk, cfg.nk, self._h, delp_key=dw)
        remap_map.remap_map(st, cfg.remap_linear(), ak, bk, cfg.nk, self._h)
        thermo.apply(st, cfg.tracer_names()[:thermo.SPECIES], cfg.nk, self._h, thermo.constants(c))

    def acoustic_phases(self):
        """One acoustic substep (config C1), mirroring ``Dycore.acoustic_phases``
        (the caller zeroes the accumulators and sets dp1 at the step start)."""
        c, dt = dict(self.cfg.consts), self.cfg.dt_acoustic
        yield ["u", "v", "w", "delp", "pt", "gz"]
        self.call("c_grid", {**c, "dt2": 0.5 * dt})
        yield ["uc", "vc"]
        self.call("d_sw", {**c, "dt": dt})
        self.call("nh_d", {**c, "dt": dt})
        yield ["pef", "gz"]
        self.call("p_grad_d", {**c, "dt": dt})

    def substep(self, first: bool = True) -> None:
        """One acoustic substep; ``first`` starts a timestep (accumulators
        zeroed, dp1 = delp), as the device's first substep does."""
        if first:
            for n in ("cx", "cy", "xfa", "yfa", "mfx", "mfy"):
                self.state[n][...] = 0.0
            self.state["dp1"][...] = self.state["delp"]
        for names in self.acoustic_phases():
            self.halo(names)

    def step(self) -> None:
        for names in self.phases():
            self.halo(names)


PROGNOSTIC = ["u", "v", "w", "delp", "pt", "gz"]
