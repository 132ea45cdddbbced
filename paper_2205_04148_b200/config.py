"""Frozen run configuration shared by the CPU oracle step and the B200 step
("Freeze n_split, k_split, nq and dt in one run-config").

One dycore timestep (k_split = 1):

    for it in range(n_split):                         acoustic substeps
        halo_update(u, v, w, delp, pt, gz)
        c_grid    (c_sw + riem_solver_c + p_grad_c)   -> uc, vc
        halo_update(uc, vc)
        d_sw                                          -> u, v, w, delp, pt, cx, cy, xfa, yfa, mfx, mfy
        nh_d      (riem_solver3 role)                 -> w, gz, pef
        halo_update(pef, gz)
        p_grad_d                                      -> u, v
    halo_update(q*, cx, cy, xfa, yfa, mfx, mfy)
    tracer_2d (nq tracers)                            -> q*
    log_thickness (pt_logp)                           -> dlnp
    remap_tracers (remap_profile of q*, w at delp,
                   pt at dlnp, u / v at their faces)  -> *_a2, *_a3, *_a4
    remap_map (Lagrangian -> Eulerian, map1_ppm;
               pt in log pressure)                    -> q*, pt, w, u, v, delp
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .programs.templates import DAMP4, DAMPV


@dataclass(frozen=True)
class RunConfig:
    ni: int = 192
    nj: int = 192
    nk: int = 80
    n_split: int = 6
    nq: int = 8
    dt_atmos: float = 90.0
    halo: int = 4
    seed: int = 2205
    # remap pt in log pressure (FV3 fv_mapz with kord_tm < 0): its profile at
    # the log-pressure thickness, its mapping on log(pe1) -> log(pe2)
    pt_logp: bool = True
    # physical constants of the programs (templates.RIEM_CONSTS / D_CONSTS)
    consts: dict = field(default_factory=lambda: {
        "ptop": 300.0, "rdgas": 287.05, "grav": 9.80665, "gama": 1.4, "p_fac": 0.05,
        "dddmp": 0.2, "d2_bg": 0.0, "da_min": 1.0e8,
        # del6 flux-damping coefficients of d_sw (templates.D_CONSTS: (c * da_min) ** 3)
        "damp4": DAMP4, "damp4h": 0.5 * DAMP4, "dampv": DAMPV,
        "ppm_p1": 7.0 / 12.0, "ppm_p2": -1.0 / 12.0,
        # heat capacities of the post-remap diagnostics (FV3 constants; oracle/thermo.py)
        "cp_air": 1004.6, "rvgas": 461.50, "c_liq": 4185.5, "c_ice": 1972.0,
    })

    @property
    def dt_acoustic(self) -> float:
        return self.dt_atmos / self.n_split

    @property
    def cells(self) -> int:
        return self.ni * self.nj * self.nk

    def tracer_names(self) -> list[str]:
        return [f"q{n}" for n in range(self.nq)]

    def remap_linear(self) -> list[str]:
        """The remapped fields mapped in pressure at delp (pt is mapped in log
        pressure when ``pt_logp``)."""
        return self.tracer_names() + (["w"] if self.pt_logp else ["pt", "w"])

    def remapped(self) -> list[str]:
        """Fields the vertical remapping maps onto the target layers: the
        tracers, then pt and w (u and v, at staggered pressures, are not
        remapped)."""
        return self.tracer_names() + ["pt", "w"]

    def moist_names(self) -> list[str]:
        """FV3's six water species (vapour, liquid, rain, ice, snow, graupel)
        among the tracers: q0..q5 (fewer when nq < 6; absent species are 0)."""
        return self.tracer_names()[:6]

    def moist_scalars(self) -> list[float]:
        """fv3b_moist_pk scalars: ptop, akap = rdgas / cp_air, cv_air =
        cp_air - rdgas, cv_vap = 3 rvgas, c_liq, c_ice."""
        c = self.consts
        return [c["ptop"], c["rdgas"] / c["cp_air"], c["cp_air"] - c["rdgas"], 3.0 * c["rvgas"], c["c_liq"], c["c_ice"]]

    def target_coordinate(self):
        """ak, bk (nk+1) of the vertical remapping's target interfaces
        pe2 = ak + bk * ps: pure sigma below ptop, bk = k / nk."""
        import numpy as np

        bk = np.arange(self.nk + 1, dtype=np.float64) / self.nk
        return self.consts["ptop"] * (1.0 - bk), bk


# Prognostic / diagnostic state fields.  3-D fields have nk+1 levels
# (interface-capable); 2-D fields are metrics and the surface w.
STATE_3D = ["u", "v", "w", "delp", "pt", "gz", "pef", "uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy", "dp1"]
# post-remap diagnostics (fv3b_moist_pk): interface pe, peln, pk; layer pkz, cvm
DIAG_3D = ["pe", "peln", "pk", "pkz", "cvm"]
METRICS_2D = ["dx", "dy", "dxc", "dyc", "rdx", "rdy", "rdxc", "rdyc", "rdxa", "rdya", "area", "rarea", "rarea_c",
              "f0", "fc", "ws", "del6_u", "del6_v"]
