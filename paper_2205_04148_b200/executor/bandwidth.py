"""``measure_bandwidth`` — the copy-stencil HBM probe (``SPEC.md:392-400``;
the paper's copy-stencil ceiling, ``PAPER.md:589``).

Runs the K0 copy kernel (``fv3b_copy``) over two device fields of
``domain_bytes`` each, median of ``reps`` >= 10 CUDA-event timings, and
returns bytes moved (read + write) per second.  The SPEC requires the
domain to exceed the last-level cache by 4x: B200 L2 is 126 MB, so the
default is 512 MiB per field.
"""

from __future__ import annotations

import statistics

import torch

from .. import _lib
from ..device import Grid

L2_BYTES = 126 * 10**6


def measure_bandwidth(domain_bytes: int = 512 * 2**20, reps: int = 10) -> float:
    if reps < 10:
        raise ValueError("reps must be >= 10")
    if domain_bytes < 4 * L2_BYTES:
        raise ValueError(f"domain_bytes must exceed 4x the {L2_BYTES / 1e6:.0f} MB L2")
    ni = nj = 1024
    nk = max(1, domain_bytes // (8 * ni * nj))
    g = Grid(ni, nj, nk, halo=0)
    try:
        a = g.new3(fill=1.0)
        b = g.new3(fill=0.0)
    except torch.OutOfMemoryError as e:  # pragma: no cover - depends on device
        raise MemoryError(f"insufficient device memory for a {domain_bytes} B probe") from e
    fa, fb, dom = g.abi(a), g.abi(b), g.domain(nk=nk)
    stream = torch.cuda.current_stream().cuda_stream
    for _ in range(2):
        _lib.call("fv3b_copy", [fa, fb], [], dom, stream)
    times = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        _lib.call("fv3b_copy", [fa, fb], [], dom, stream)
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e) * 1e-3)
    return 2.0 * 8 * ni * nj * nk / statistics.median(times)
