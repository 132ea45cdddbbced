"""step_host transfer shapes, both PCIe directions at once (C2, 14 fields):
full halo-inclusive arrays (1-D per field), interior columns (2-D per
field), the interior I-slab (1-D per field: interior rows incl. the J-halo
gaps), and one 1-D copy of the same bytes.  ms and GB/s per direction."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2205_04148_b200 import _lib  # noqa: E402
from paper_2205_04148_b200.config import RunConfig  # noqa: E402


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def main():
    cfg = RunConfig()
    h = cfg.halo
    shape = (cfg.ni + 2 * h, cfg.nj + 2 * h, cfg.nk + 1)
    nf = 14
    hin = [torch.zeros(shape, dtype=torch.float64).pin_memory() for _ in range(nf)]
    hout = [torch.zeros(shape, dtype=torch.float64).pin_memory() for _ in range(nf)]
    din = [torch.zeros(shape, dtype=torch.float64, device="cuda") for _ in range(nf)]
    dout = [torch.zeros(shape, dtype=torch.float64, device="cuda") for _ in range(nf)]
    up, down = torch.cuda.Stream(), torch.cuda.Stream()
    comp = torch.cuda.current_stream()
    nl = shape[2]
    pitch = shape[1] * nl * 8
    off = (h * shape[1] + h) * nl * 8
    width = cfg.nj * nl * 8
    slab_off = h * pitch
    slab = cfg.ni * pitch

    def run(kind):
        def f():
            up.wait_stream(comp)
            down.wait_stream(comp)
            for t in range(nf):
                for s, src, dst in ((up, hin[t], din[t]), (down, dout[t], hout[t])):
                    if kind == "full":
                        with torch.cuda.stream(s):
                            dst.copy_(src, non_blocking=True)
                    elif kind == "interior2d":
                        _lib.memcpy2d(dst.data_ptr() + off, pitch, src.data_ptr() + off, pitch, width, cfg.ni, s.cuda_stream)
                    elif kind == "slab1d":
                        _lib.memcpy2d(dst.data_ptr() + slab_off, slab, src.data_ptr() + slab_off, slab, slab, 1, s.cuda_stream)
            comp.wait_stream(up)
            comp.wait_stream(down)
        return f

    nbytes = {"full": nf * shape[0] * pitch, "interior2d": nf * cfg.ni * width, "slab1d": nf * slab}
    for kind in ("full", "interior2d", "slab1d"):
        ms = timed(run(kind))
        print(json.dumps({"kind": kind, "MB_each_way": round(nbytes[kind] / 1e6, 1), "ms": round(ms, 3),
                          "GBps_each_way": round(nbytes[kind] / ms / 1e6, 1)}), flush=True)
    # the same with every field's host buffer a view of one pinned block
    numel = shape[0] * shape[1] * shape[2]
    bin_, bout = torch.zeros(nf * numel, dtype=torch.float64).pin_memory(), torch.zeros(nf * numel, dtype=torch.float64).pin_memory()
    hin[:] = [bin_[t * numel:(t + 1) * numel].view(shape) for t in range(nf)]
    hout[:] = [bout[t * numel:(t + 1) * numel].view(shape) for t in range(nf)]
    for kind in ("full", "interior2d"):
        ms = timed(run(kind))
        kind = kind + "_oneblock"
        nb = nbytes[kind.split("_")[0]]
        print(json.dumps({"kind": kind, "MB_each_way": round(nb / 1e6, 1), "ms": round(ms, 3),
                          "GBps_each_way": round(nb / ms / 1e6, 1)}), flush=True)
    # one copy per direction of the whole block
    dbin = torch.zeros(nf * numel, dtype=torch.float64, device="cuda")
    dbout = torch.zeros(nf * numel, dtype=torch.float64, device="cuda")

    def big():
        up.wait_stream(comp)
        down.wait_stream(comp)
        with torch.cuda.stream(up):
            dbin.copy_(bin_, non_blocking=True)
        with torch.cuda.stream(down):
            bout.copy_(dbout, non_blocking=True)
        comp.wait_stream(up)
        comp.wait_stream(down)

    ms = timed(big)
    print(json.dumps({"kind": "one_copy_each_way", "MB_each_way": round(nf * numel * 8 / 1e6, 1), "ms": round(ms, 3),
                      "GBps_each_way": round(nf * numel * 8 / ms / 1e6, 1)}), flush=True)
    return
    for kind in ():
        ms = 0
        print(json.dumps({"kind": kind, "MB_each_way": round(nbytes[kind] / 1e6, 1), "ms": round(ms, 3),
                          "GBps_each_way": round(nbytes[kind] / ms / 1e6, 1)}), flush=True)


if __name__ == "__main__":
    main()
