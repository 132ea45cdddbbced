"""Scratch: stream timeline of pipelined Dycore.step_host calls (C2): when
each call's uploads / compute / downloads start and end."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.state import initial_state

cfg = RunConfig()
st = initial_state(cfg)
d = Dycore(cfg, st)
h_in, h_out = d.host_buffers(), d.host_buffers()
for n, t in h_in.items():
    t.copy_(torch.from_numpy(st[n]))
for _ in range(3):
    d.step_host(h_in, h_out)
torch.cuda.synchronize()
up, down = d._io_streams()
comp = torch.cuda.current_stream()
marks = []
ev = lambda s: (lambda e: (e.record(s), e)[1])(torch.cuda.Event(enable_timing=True))
t0 = ev(comp)
chained = "chained" in sys.argv  # each call's input is the previous call's output
for i in range(6):
    a = (ev(up), ev(comp), ev(down))
    done = d.step_host(h_in, h_out)
    b = (ev(up), ev(comp), ev(down))
    marks.append((a, b))
    if chained:
        h_in, h_out = h_out, h_in
comp.wait_event(done)
t1 = ev(comp)
torch.cuda.synchronize()
print(f"period {t0.elapsed_time(t1) / 6:.2f} ms")
for i, (a, b) in enumerate(marks):
    print(f"call {i}: enqueue-marks up {t0.elapsed_time(a[0]):7.2f}->{t0.elapsed_time(b[0]):7.2f}  "
          f"comp {t0.elapsed_time(a[1]):7.2f}->{t0.elapsed_time(b[1]):7.2f}  "
          f"down {t0.elapsed_time(a[2]):7.2f}->{t0.elapsed_time(b[2]):7.2f}")
