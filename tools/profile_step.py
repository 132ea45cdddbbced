"""One eager dycore timestep at C2 size for ncu captures (n_split from argv,
default 1 so every kernel of the step appears once)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.state import initial_state

n_split = int(sys.argv[1]) if len(sys.argv) > 1 else 1
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 1
cfg = RunConfig(n_split=n_split)
d = Dycore(cfg, initial_state(cfg))
for _ in range(steps):
    d.step()
torch.cuda.synchronize()
print("done")
