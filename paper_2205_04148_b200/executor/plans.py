"""Kernel plans: how each shipped program's driver trace maps onto libfv3b
launches.

A plan is the hand-written counterpart of one ``.stn`` program: it checks
that the resolved driver trace is the one its fused kernels implement,
binds the program's fields and scalars to the entry point's fixed argument
order (``include/fv3b.h``) and enqueues the launches.  Written
non-temporaries go to separate output buffers (the reference materialises
each right-hand side before storing it, ``reference.py:10-12``), which the
caller seeds with the input values so untouched halo cells are returned as
provided (``reference.py:335-339``).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable

import torch

from .. import _lib
from ..device import Grid
from ..program import Program


@dataclass
class LaunchCtx:
    grid: Grid
    fields: dict[str, torch.Tensor]        # current (input) buffers, by field name
    outputs: dict[str, torch.Tensor]       # output buffers of written fields
    placement: tuple
    stream: int
    nk: int                                # program vertical domain
    on_launch: Callable | None = None      # (node, start_event, end_event) timing hook
    launches: list = field(default_factory=list)
    workspace: dict = field(default_factory=dict)  # device scratch for fused temporaries

    def scratch(self, name: str) -> _lib.Field:
        """3-D device buffer for a temporary that crosses kernels of one
        fused plan (allocated once per state, reused across calls)."""
        if name not in self.workspace:
            self.workspace[name] = self.grid.new3(device=self.fields[next(iter(self.fields))].device)
        return self.grid.abi(self.workspace[name])

    def f(self, name: str, rank: int | None = None) -> _lib.Field:
        return self.grid.abi(self.fields[name], rank)

    def o(self, name: str) -> _lib.Field:
        return self.grid.abi(self.outputs[name])

    def call(self, node: str, entry: str, fields: list, scalars: list[float], nk: int | None = None) -> None:
        dom = self.grid.domain(self.placement, nk=self.nk if nk is None else nk)
        if self.on_launch is not None:
            s = torch.cuda.Event(enable_timing=True)
            e = torch.cuda.Event(enable_timing=True)
            s.record()
            _lib.call(entry, fields, scalars, dom, self.stream)
            e.record()
            self.on_launch(node, s, e)
        else:
            _lib.call(entry, fields, scalars, dom, self.stream)
        self.launches.append(node)


class Plan:
    name: str = ""
    stencils: tuple[str, ...] = ()   # expected resolved trace (stencil names)

    def written(self, prog: Program) -> list[str]:
        out = []
        for s in prog.canon["stencils"]:
            for b in s["blocks"]:
                for st in b["statements"]:
                    t = st["target"]
                    if not prog.fields[t].temporary and t not in out:
                        out.append(t)
        return out

    def check_trace(self, trace) -> None:
        names = tuple(s for s, _ in trace)
        if names != self.stencils:
            raise NotImplementedError(
                f"{self.name}: the B200 plan implements the trace {self.stencils}, got {names}")

    def run(self, prog: Program, ctx: LaunchCtx) -> None:
        raise NotImplementedError


class CopyPlan(Plan):
    name = "copy"
    stencils = ("copy_field",)

    def run(self, prog, ctx):
        ctx.call("copy_field_0", "fv3b_copy", [ctx.f("inp"), ctx.o("out")], [])


class FvTp2dPlan(Plan):
    name = "fv_tp_2d"
    stencils = ("fv_tp_2d",)

    def run(self, prog, ctx):
        (stencil, kw), = prog.trace
        s = prog.scalars(kw)
        ctx.call("fv_tp_2d_0", "fv3b_fv_tp_2d",
                 [ctx.f("q"), ctx.f("crx"), ctx.f("cry"), ctx.f("xfx"), ctx.f("yfx"),
                  ctx.f("area", 2), ctx.f("rarea", 2), ctx.o("q")],
                 [s["ppm_p1"], s["ppm_p2"]])


class Tracer2dPlan(Plan):
    name = "tracer_2d"

    def check_trace(self, trace):
        names = [s for s, _ in trace]
        nq = len(names) - 1
        if names != ["tracer_dp"] + [f"tracer_q{n}" for n in range(nq)] or not 1 <= nq <= 16:
            raise NotImplementedError(f"tracer_2d: unsupported trace {names}")

    def run(self, prog, ctx):
        trace = prog.trace
        nq = len(trace) - 1
        s = prog.scalars(trace[1][1])
        fields = [ctx.f(n) for n in ("cx", "cy", "xfx", "yfx", "mfx", "mfy", "dp1")]
        fields += [ctx.f("area", 2), ctx.f("rarea", 2)]
        fields += [ctx.f(f"q{n}") for n in range(nq)] + [ctx.o(f"q{n}") for n in range(nq)]
        ctx.call("tracer_2d_0", "fv3b_tracer_2d", fields, [s["ppm_p1"], s["ppm_p2"]])


class RiemSolverCPlan(Plan):
    name = "riem_solver_c"
    stencils = ("riem_pem", "riem_layer", "riem_coef", "riem_pp_fwd", "riem_pp_bwd", "riem_w_fwd",
                "riem_w_sweep", "riem_w_back", "riem_pe", "riem_out", "riem_gz")

    def run(self, prog, ctx):
        s = prog.scalars(prog.trace[0][1])
        ctx.call("riem_pem_0", "fv3b_riem_solver_c",
                 [ctx.f("dm"), ctx.f("pt"), ctx.f("w"), ctx.f("gz"), ctx.f("ws", 2), ctx.o("pef"), ctx.o("gz"),
                  ctx.scratch("riem_scr")],
                 [s["ptop"], s["rdgas"], s["grav"], s["gama"], s["p_fac"], s["dt"]])


class RemapPlan(Plan):
    """remap_profile (one field) and remap_tracers (q0..q{n-1})."""

    def __init__(self, name: str):
        self.name = name

    def _tracers(self, prog) -> list[str]:
        if self.name == "remap_profile":
            return [""]
        n = len(prog.trace) // 3
        return [str(t) for t in range(n)]

    def check_trace(self, trace):
        names = [s for s, _ in trace]
        if self.name == "remap_profile":
            want = ["remap_edge_fwd", "remap_edge_bwd", "remap_a4"]
        else:
            n = len(names) // 3
            want = [f"{b}_{t}" for t in range(n) for b in ("remap_edge_fwd", "remap_edge_bwd", "remap_a4")]
        if names != want:
            raise NotImplementedError(f"{self.name}: unsupported trace {names}")

    def run(self, prog, ctx):
        fields = [ctx.f("delp")]
        if self.name == "remap_profile":
            fields += [ctx.f("q"), ctx.o("a4_2"), ctx.o("a4_3"), ctx.o("a4_4")]
        else:
            for t in self._tracers(prog):
                fields += [ctx.f(f"q{t}"), ctx.o(f"q{t}_a2"), ctx.o(f"q{t}_a3"), ctx.o(f"q{t}_a4")]
        ctx.call(prog.trace[0][0] + "_0", "fv3b_remap_profile", fields, [])


C_METRICS = ("dx", "dy", "dxc", "dyc", "rdxc", "rdyc", "rarea", "rarea_c", "fc")
D_METRICS = ("dx", "dy", "dxc", "dyc", "rdx", "rdy", "rdxa", "rdya", "area", "rarea", "rarea_c", "f0", "del6_u",
             "del6_v")
D_STATE = ("u", "v", "w", "delp", "pt", "uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy")
D_OUT = ("u", "v", "w", "delp", "pt", "cx", "cy", "xfa", "yfa", "mfx", "mfy")


class CswPlan(Plan):
    name = "c_sw"
    stencils = ("c_sw_winds", "c_sw_transport", "c_sw_ke_vort", "c_sw_update")

    def run(self, prog, ctx):
        s = prog.scalars(prog.trace[0][1])
        fields = [ctx.f(n) for n in ("u", "v", "delp", "pt", "w")] + [ctx.f(m, 2) for m in C_METRICS]
        fields += [ctx.o(n) for n in ("uc", "vc", "delpc", "ptc", "wc")]
        ctx.call("c_sw_winds_0", "fv3b_c_sw", fields, [s["dt2"]])


class CGridPlan(Plan):
    name = "c_grid"
    stencils = ("c_sw_winds", "c_sw_transport", "c_sw_ke_vort", "c_sw_update") + tuple(
        f"{n}_c" for n in RiemSolverCPlan.stencils) + ("p_grad_c",)

    def run(self, prog, ctx):
        s = prog.scalars(prog.trace[0][1])
        fields = [ctx.f(n) for n in ("u", "v", "delp", "pt", "w", "gz")] + [ctx.f(m, 2) for m in C_METRICS]
        fields += [ctx.f("ws", 2), ctx.o("uc"), ctx.o("vc")]
        fields += [ctx.scratch(n) for n in ("delpcc", "ptcc", "wcc", "pkc", "gzc", "riem_scr")]
        ctx.call("c_sw_winds_0", "fv3b_c_grid", fields,
                 [s["dt2"], s["ptop"], s["rdgas"], s["grav"], s["gama"], s["p_fac"]])


class DswPlan(Plan):
    name = "d_sw"
    stencils = ("d_sw_courant", "d_sw_mass", "d_sw_heat", "d_sw_vert", "d_sw_ke", "d_sw_vort", "d_sw_damp",
                "d_sw_update")

    def run(self, prog, ctx):
        s = prog.scalars(prog.trace[0][1])
        fields = [ctx.f(n) for n in D_STATE] + [ctx.f(m, 2) for m in D_METRICS] + [ctx.o(n) for n in D_OUT]
        ctx.call("d_sw_courant_0", "fv3b_d_sw", fields,
                 [s["ppm_p1"], s["ppm_p2"], s["dt"], s["dddmp"], s["d2_bg"], s["da_min"], s["damp4"], s["damp4h"],
                  s["dampv"]])


class NhDPlan(Plan):
    name = "nh_d"
    stencils = tuple(f"{n}_d" for n in RiemSolverCPlan.stencils) + ("nh_d_w",)

    def run(self, prog, ctx):
        s = prog.scalars(prog.trace[0][1])
        fields = [ctx.f(n) for n in ("delp", "pt", "w", "gz")] + [ctx.f("ws", 2)]
        fields += [ctx.o("pef"), ctx.o("gz"), ctx.o("w"), ctx.scratch("riem_scr")]
        ctx.call("riem_pem_d_0", "fv3b_nh_d", fields,
                 [s["ptop"], s["rdgas"], s["grav"], s["gama"], s["p_fac"], s["dt"]])


class PGradDPlan(Plan):
    name = "p_grad_d"
    stencils = ("p_grad_d_corners", "p_grad_d")

    def run(self, prog, ctx):
        s = prog.scalars(prog.trace[0][1])
        fields = [ctx.f(n) for n in ("u", "v", "pef", "gz")] + [ctx.f("rdx", 2), ctx.f("rdy", 2)]
        fields += [ctx.o("u"), ctx.o("v")]
        ctx.call("p_grad_d_corners_0", "fv3b_p_grad_d", fields, [s["dt"]])


PLANS: dict[str, Plan] = {p.name: p for p in (CopyPlan(), FvTp2dPlan(), Tracer2dPlan(), RiemSolverCPlan(),
                                              RemapPlan("remap_profile"), RemapPlan("remap_tracers"), CswPlan(),
                                              CGridPlan(), DswPlan(), NhDPlan(), PGradDPlan())}


def plan_for(prog: Program) -> Plan:
    if prog.name not in PLANS:
        raise KeyError(f"no B200 plan for program {prog.name!r}")
    plan = PLANS[prog.name]
    plan.check_trace(prog.trace)
    return plan
