"""One small eager timestep (every kernel of the step at least once) for
compute-sanitizer runs: memcheck / racecheck / synccheck (tools/sanitize.sh)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.state import initial_state

cfg = RunConfig(ni=40, nj=24, nk=6, n_split=1, dt_atmos=20.0)
d = Dycore(cfg, initial_state(cfg))
d.step()
torch.cuda.synchronize()
print("step done")
