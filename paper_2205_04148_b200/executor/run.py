"""``run_b200``: the ``run_reference`` contract on the B200.

Reference: ``run_reference(program, inputs, domain, placement=FULL_TILE,
recorder=None, check_finite=False)`` (``executor/reference.py:307-339``):

* inputs are halo-inclusive arrays, axes in declared I, J, K order, shape
  ``n + h_lo + h_hi`` per axis from ``compute_requirements``; a wrong shape
  raises ``ValueError`` (``:164-167``); missing inputs are zero (``:168-169``);
* inputs are copied, outputs are fresh arrays for every non-temporary
  (``:335-339``), untouched halo cells returned as provided;
* ``placement`` decides which edge regions fire (``lower.py:91-93``).

``recorder`` (brute-force access marking) is a CPU-interpreter facility with
no device counterpart and is rejected.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from ..device import DEFAULT_HALO, Grid
from ..program import Program, as_program, is_graph
from .plans import LaunchCtx, plan_for

FULL_TILE = (True, True, True, True)


def placement_tuple(placement) -> tuple:
    if placement is None:
        return FULL_TILE
    if hasattr(placement, "own_i_start"):
        return (placement.own_i_start, placement.own_i_end, placement.own_j_start, placement.own_j_end)
    t = tuple(bool(x) for x in placement)
    if len(t) != 4:
        raise ValueError("placement must be a RankPlacement or 4 booleans")
    return t


@dataclass
class Uploaded:
    """Device-resident program state produced by :func:`upload`."""

    prog: Program
    grid: Grid
    domain: tuple[int, int, int]
    fields: dict[str, torch.Tensor]
    outputs: dict[str, torch.Tensor]
    placement: tuple
    workspace: dict = None

    def ctx(self, stream: int | None = None, on_launch=None) -> LaunchCtx:
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        if self.workspace is None:
            self.workspace = {}
        return LaunchCtx(self.grid, self.fields, self.outputs, self.placement, stream, self.domain[2], on_launch,
                         workspace=self.workspace)

    def download(self) -> dict[str, np.ndarray]:
        out = {}
        for name, info in self.prog.fields.items():
            if info.temporary:
                continue
            t = self.outputs.get(name, self.fields[name])
            out[name] = self.grid.get(t, info.dims, [info.halo(a)[0] for a in info.dims], info.shape(self.domain))
        return out


def upload(program, inputs: dict, domain, placement=None, device="cuda") -> Uploaded:
    """Validate and copy a program's inputs into the device layout.  A
    lowered reference ``DataflowGraph`` brings its own domain and
    ``RankPlacement`` (``ir/graph.py:257-268``) when none are given."""
    if is_graph(program):
        domain = program.domain if domain is None else domain
        placement = program.placement if placement is None else placement
    prog = as_program(program)
    domain = tuple(int(x) for x in domain)
    prog.check_domain(domain)
    if not torch.cuda.is_available():
        raise RuntimeError("run_b200 needs a CUDA device (no CPU fallback)")
    for name, info in prog.fields.items():
        if info.dtype != "float64":
            raise NotImplementedError(f"field {name!r}: only float64 fields are supported")
    need = 0
    for info in prog.fields.values():
        if not info.temporary:
            for a in info.dims:
                if a != "K":
                    need = max(need, *info.halo(a))
    grid = Grid(domain[0], domain[1], domain[2], halo=max(DEFAULT_HALO, need))
    fields: dict[str, torch.Tensor] = {}
    for name, info in prog.fields.items():
        if info.temporary:
            continue
        shape = info.shape(domain)
        t = {3: grid.new3, 2: grid.new2, 1: grid.new1}[len(info.dims)](device)
        if name in inputs:
            arr = np.asarray(inputs[name])
            if tuple(arr.shape) != shape:
                raise ValueError(f"input {name!r} has shape {tuple(arr.shape)}, expected {shape}")
            grid.put(t, arr, info.dims, [info.halo(a)[0] for a in info.dims])
        fields[name] = t
    plan = plan_for(prog)
    outputs = {n: fields[n].clone() for n in plan.written(prog)}
    return Uploaded(prog, grid, domain, fields, outputs, placement_tuple(placement))


def execute(up: Uploaded, stream: int | None = None, on_launch=None) -> list[str]:
    """Enqueue the program's kernels on the device state; returns the node
    names launched."""
    ctx = up.ctx(stream, on_launch)
    plan_for(up.prog).run(up.prog, ctx)
    return ctx.launches


def run_b200(program, inputs: dict, domain, placement=None, recorder=None, check_finite: bool = False):
    """Execute ``program`` on the B200; same contract as ``run_reference``."""
    if recorder is not None:
        raise NotImplementedError("access recording is a CPU-interpreter facility (use the oracle)")
    up = upload(program, inputs, domain, placement)
    execute(up)
    torch.cuda.synchronize()
    return up.download()
