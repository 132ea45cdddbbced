"""Scratch: time the full dycore step (graph replay) and per-kernel shares."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.state import initial_state

args = [a for a in sys.argv[1:] if not a.startswith('--')]
ni = int(args[0]) if args else 192
cfg = RunConfig(ni=ni, nj=ni, nk=80, pt_logp='--linear-pt' not in sys.argv)
t = time.time()
d = Dycore(cfg, initial_state(cfg))
print("init", time.time() - t, flush=True)
for _ in range(2):
    d.step()
torch.cuda.synchronize()
d.capture()
for _ in range(3):
    d.replay()
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
N = 10
for _ in range(N):
    d.replay()
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / N
print(f"step {ms:.3f} ms  cells/s {cfg.cells / ms * 1e3:.3e}")
# per-kernel (eager, events around each launch, GPU kept busy with a sleep)
class T:
    def __init__(self): self.ev = []
    def start(self, n):
        a = torch.cuda.Event(enable_timing=True); a.record(); self.ev.append([n, a, None])
    def stop(self, n):
        b = torch.cuda.Event(enable_timing=True); b.record(); self.ev[-1][2] = b
d.timer = T()
torch.cuda._sleep(50_000_000)
d.step()
torch.cuda.synchronize()
tot = {}
for n, a, b in d.timer.ev:
    tot[n] = tot.get(n, 0.0) + a.elapsed_time(b)
for n, v in sorted(tot.items(), key=lambda x: -x[1]):
    print(f"  {n:14s} {v:8.3f} ms")
print("sum", sum(tot.values()))
