"""One small eager timestep (every kernel of the step at least once) for
compute-sanitizer runs: memcheck / racecheck / synccheck (tools/sanitize.sh)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch

from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.state import initial_state

from paper_2205_04148_b200 import _lib

cfg = RunConfig(ni=40, nj=24, nk=6, n_split=1, dt_atmos=20.0)
d = Dycore(cfg, initial_state(cfg))
d.step()
torch.cuda.synchronize()
print("step done")
# the level-marching tile kernels with multi-level chunks, the last one
# ragged (6 = 4 + 2 levels): the TMA refill of the next level, the mbarrier
# phase flip and tracer_2d's level-boundary restaging (the C2 launch shapes)
with _lib.tuning(kchunk=4):
    d.step()
torch.cuda.synchronize()
print("kchunk=4 step done")
# the program-level kernels the step does not launch (run_b200, ragged domains,
# full-tile placement: edge regions fire)
from paper_2205_04148_b200.executor import run_b200
from paper_2205_04148_b200.inputs import synthetic_inputs

for name, dom, place in (("fv_tp_2d", (37, 21, 4), (False,) * 4), ("c_sw", (37, 21, 3), (True,) * 4),
                         ("d_sw", (37, 21, 3), (True,) * 4), ("d_sw", (35, 17, 5), (False,) * 4),
                         ("riem_solver_c", (33, 7, 9), (False,) * 4), ("remap_profile", (33, 7, 9), (False,) * 4),
                         ("copy", (33, 17, 5), (False,) * 4)):
    run_b200(name, synthetic_inputs(name, dom, 1), dom, placement=place)
torch.cuda.synchronize()
print("programs done")
# the peer-memory halo path (fv3b_halo_peer_rects): a 1 x 2 loopback
# decomposition in stream order.  The device-side neighbour barriers
# (fv3b_peer_barrier) cannot run under the sanitizer: it serialises kernels,
# so a rank's spin never sees the other stream arrive (the spin is bounded
# and reports a timeout instead of hanging).
from paper_2205_04148_b200.parallel import LoopbackCluster

blk = RunConfig(ni=20, nj=12, nk=6, n_split=1, dt_atmos=20.0)
cl = LoopbackCluster([Dycore(blk, initial_state(blk)) for _ in range(2)], 1, 2, direct=True)
cl.step()
torch.cuda.synchronize()
print("peer halos done")
# the cubed sphere by peer stores (fv3b_halo_peer_idx): six FULL_TILE tiles in stream order
from paper_2205_04148_b200.cubesphere import CubePeerHalo, LoopbackTiles

cub = RunConfig(ni=12, nj=12, nk=4, n_split=1, dt_atmos=20.0)
tiles = [Dycore(cub, initial_state(RunConfig(ni=12, nj=12, nk=4, seed=7 + t)), placement=(True,) * 4)
         for t in range(6)]
peers = LoopbackTiles(tiles)
LoopbackCluster(tiles, halos=[CubePeerHalo(d, t, peers) for t, d in enumerate(tiles)]).step()
torch.cuda.synchronize()
print("cube peer halos done")
