"""Device field storage in the reference ``Layout`` (``scheduling.py:323-407``).

Every field of one domain shares a single tile geometry so that one kernel
launch indexes all of its operands with one pair of strides:

* I is unit stride; each row holds ``pre_pad + halo + ni + halo`` elements
  rounded up to ``alignment`` (8 doubles = 64 B), with
  ``pre_pad = (alignment - halo % alignment) % alignment`` so the first
  interior element of every row is 64-B aligned (the paper's Fig. 7 scheme);
* J carries the same halo; K has ``nk + 1`` levels and no halo, so layer
  fields (nk) and interface fields (nk+1) share the geometry;
* 2-D (I, J) fields are one level of the same plane.

At C2 (192x192x80, halo 4) a 3-D field is 81 x 200 x 208 doubles = 27.0 MB;
the full dycore state (~40 fields) is ~1.1 GB of the 180 GB HBM.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import Domain, Field

DEFAULT_HALO = 4
ALIGN = 8


@dataclass(frozen=True)
class Grid:
    ni: int
    nj: int
    nk: int
    halo: int = DEFAULT_HALO
    align: int = ALIGN

    @property
    def pre_pad(self) -> int:
        return (self.align - self.halo % self.align) % self.align

    @property
    def pitch(self) -> int:
        n = self.pre_pad + self.ni + 2 * self.halo
        return -(-n // self.align) * self.align

    @property
    def rows(self) -> int:
        return self.nj + 2 * self.halo

    @property
    def levels(self) -> int:
        return self.nk + 1

    @property
    def i0(self) -> int:
        """Column of interior i = 0 inside a row."""
        return self.pre_pad + self.halo

    def new3(self, device="cuda", fill: float | None = 0.0) -> torch.Tensor:
        t = torch.empty((self.levels, self.rows, self.pitch), dtype=torch.float64, device=device)
        if fill is not None:
            t.fill_(fill)
        return t

    def new2(self, device="cuda", fill: float | None = 0.0) -> torch.Tensor:
        t = torch.empty((self.rows, self.pitch), dtype=torch.float64, device=device)
        if fill is not None:
            t.fill_(fill)
        return t

    def new1(self, device="cuda", fill: float | None = 0.0) -> torch.Tensor:
        t = torch.empty((self.levels,), dtype=torch.float64, device=device)
        if fill is not None:
            t.fill_(fill)
        return t

    def interior(self, t: torch.Tensor, nk: int | None = None) -> torch.Tensor:
        """(K, J, I) view of the interior of a 3-D or (J, I) of a 2-D field."""
        h, i0 = self.halo, self.i0
        if t.dim() == 3:
            return t[: (nk or self.nk), h : h + self.nj, i0 : i0 + self.ni]
        return t[h : h + self.nj, i0 : i0 + self.ni]

    def abi(self, t: torch.Tensor, rank: int | None = None) -> Field:
        """``fv3b_field`` descriptor of a tensor allocated by this grid."""
        rank = rank or t.dim()
        f = Field()
        f.data = t.data_ptr()
        if rank == 3:
            f.stride[:] = [1, self.pitch, self.pitch * self.rows]
            f.shape[:] = [self.pitch, self.rows, self.levels]
            f.halo_lo[:] = [self.i0, self.halo, 0]
        elif rank == 2:
            f.stride[:] = [1, self.pitch, 0]
            f.shape[:] = [self.pitch, self.rows, 1]
            f.halo_lo[:] = [self.i0, self.halo, 0]
        else:
            f.stride[:] = [1, 0, 0]
            f.shape[:] = [self.levels, 1, 1]
            f.halo_lo[:] = [0, 0, 0]
        f.rank = rank
        return f

    def domain(self, placement=(False, False, False, False), nk: int | None = None) -> Domain:
        d = Domain()
        d.ni, d.nj, d.nk = self.ni, self.nj, (self.nk if nk is None else nk)
        d.own_i_start, d.own_i_end, d.own_j_start, d.own_j_end = (int(bool(x)) for x in placement)
        return d

    # -- host <-> device (the reference array convention: axes in declared
    #    order I, J, K, halo-inclusive, C order; reference.py:160-170) -----

    def _window(self, dims, halo_lo, shape):
        """Slices of the device tensor covering a host array."""
        sl = {}
        for axis, lo, n in zip(dims, halo_lo, shape):
            if axis == "I":
                a = self.i0 - lo
                if a < 0 or a + n > self.pitch:
                    raise ValueError(f"I halo {lo} exceeds the device halo {self.halo}")
            elif axis == "J":
                a = self.halo - lo
                if a < 0 or a + n > self.rows:
                    raise ValueError(f"J halo {lo} exceeds the device halo {self.halo}")
            else:
                a = -lo
                if a < 0 or n - lo > self.levels:
                    raise ValueError("K halo is not supported by the device layout")
            sl[axis] = slice(a, a + n)
        return sl

    def put(self, t: torch.Tensor, host: np.ndarray, dims, halo_lo) -> None:
        """Copy a reference-convention host array into tensor ``t`` (on the
        device: one contiguous upload, then the layout change by
        fv3b_transpose; a host-side grid of the CPU tests copies directly)."""
        sl = self._window(dims, halo_lo, host.shape)
        src = torch.from_numpy(np.ascontiguousarray(host, dtype=np.float64))
        dev = t.is_cuda and src.numel() > 0
        if tuple(dims) == ("I", "J", "K"):
            if dev:
                transpose(src.to(t.device), t[sl["K"], sl["J"], sl["I"]].permute(2, 1, 0))
            else:
                t[sl["K"], sl["J"], sl["I"]].copy_(src.permute(2, 1, 0))
        elif tuple(dims) == ("I", "J"):  # (as an (I, J, 1) field)
            if dev:
                transpose(src.to(t.device).unsqueeze(2), t[sl["J"], sl["I"]].permute(1, 0).unsqueeze(2))
            else:
                t[sl["J"], sl["I"]].copy_(src.permute(1, 0))
        elif tuple(dims) == ("K",):
            t[sl["K"]].copy_(src)
        else:
            raise ValueError(f"unsupported field dims {dims}")

    def get(self, t: torch.Tensor, dims, halo_lo, shape) -> np.ndarray:
        """Reference-convention host copy of a window of device tensor ``t``."""
        sl = self._window(dims, halo_lo, shape)
        if tuple(dims) == ("I", "J", "K"):
            v = t[sl["K"], sl["J"], sl["I"]].permute(2, 1, 0)
            if t.is_cuda and v.numel():
                v, w = torch.empty(tuple(shape), dtype=torch.float64, device=t.device), v
                transpose(w, v)
        elif tuple(dims) == ("I", "J"):
            v = t[sl["J"], sl["I"]].permute(1, 0)
            if t.is_cuda and v.numel():
                v, w = torch.empty(tuple(shape), dtype=torch.float64, device=t.device), v
                transpose(w.unsqueeze(2), v.unsqueeze(2))
        elif tuple(dims) == ("K",):
            v = t[sl["K"]]
        else:
            raise ValueError(f"unsupported field dims {dims}")
        return np.ascontiguousarray(v.cpu().numpy())


def transpose(src: torch.Tensor, dst: torch.Tensor) -> None:
    """``dst <- src`` for two (I, J, K)-ordered device views of one shape
    with any strides (the reference array convention <-> the Layout):
    fv3b_transpose on the current stream."""
    fs = []
    for t in (src, dst):
        f = Field()
        f.data = t.data_ptr()
        f.stride[:] = list(t.stride())
        f.shape[:] = list(t.shape)
        f.halo_lo[:] = [0, 0, 0]
        f.rank = 3
        fs.append(f)
    d = Domain()
    d.ni, d.nj, d.nk = src.shape
    _lib.call("fv3b_transpose", fs, [], d, torch.cuda.current_stream().cuda_stream)


class capture_guard:
    """Around a CUDA-graph capture: collect garbage first and keep the
    collector off until the capture ends.  A collection during a capture can
    free device tensors of dead objects whose blocks carry cross-stream
    events, and the allocator's event queries then invalidate the capture
    (torch.cuda.graph does not collect by default)."""

    def __enter__(self):
        import gc

        gc.collect()
        torch.cuda.synchronize()
        self._was = gc.isenabled()
        gc.disable()
        return self

    def __exit__(self, *exc):
        import gc

        if self._was:
            gc.enable()
        return False

