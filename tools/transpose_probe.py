"""Time fv3b_transpose (host convention <-> Layout window) for the 14
prognostic fields of C2, both directions (microseconds per field)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore

cfg = RunConfig()
d = Dycore(cfg)
names = d.prognostic()
st = d._io_stages(names)[0][0]


def run(to_state):
    for n in names:
        if to_state:
            d._transpose(st[n], d._window(d.cur[n]))
        else:
            d._transpose(d._window(d.cur[n]), st[n])


for direction in (True, False):
    run(direction)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(10):
        run(direction)
    b.record()
    torch.cuda.synchronize()
    us = a.elapsed_time(b) / 10 / len(names) * 1e3
    mb = 2 * st[names[0]].numel() * 8 / 1e6
    print(f"{'in ' if direction else 'out'}: {us:.1f} us per field ({mb / us * 1e-3 * 1e3:.0f} GB/s of {mb:.1f} MB moved)")
