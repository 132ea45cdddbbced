"""Scratch: CPU enqueue time of Dycore.step_host vs the e2e period (C2)."""
import sys, time
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
for _ in range(2):
    d.step_host(h_in, h_out)
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(10):
    d.step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"step(): enqueue {(t1 - t0) / 10 * 1e3:.2f} ms/step, wall {(t2 - t0) / 10 * 1e3:.2f} ms/step")
t0 = time.perf_counter()
for _ in range(10):
    ev = d.step_host(h_in, h_out)
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"step_host(): enqueue {(t1 - t0) / 10 * 1e3:.2f} ms/step, wall {(t2 - t0) / 10 * 1e3:.2f} ms/step")
