"""Kernel-boundary cost inside the CUDA-graph C2 step: replays a captured
timestep under torch.profiler (CUPTI kernel records) and reports, per step,
the span from the first kernel's start to the last kernel's end, the sum of
the kernel durations, and the largest gaps between consecutive kernels.

    python tools/graph_gaps.py [steps]          (on the GPU box)
"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

from paper_2205_04148_b200.config import RunConfig  # noqa: E402
from paper_2205_04148_b200.dycore import Dycore  # noqa: E402
from paper_2205_04148_b200.state import initial_state  # noqa: E402

steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
cfg = RunConfig()
d = Dycore(cfg, initial_state(cfg))
for _ in range(2):
    d.step()
torch.cuda.synchronize()
d.capture()
for _ in range(3):
    d.replay()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA], acc_events=True) as prof:
    for _ in range(steps):
        d.replay()
        torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA and "Memcpy" not in e.name
      and "Memset" not in e.name]
ev.sort(key=lambda e: e.time_range.start)
# split into steps at the host synchronisations: gaps > 50 us
groups, cur = [], [ev[0]]
for a, b in zip(ev, ev[1:]):
    if b.time_range.start - a.time_range.end > 50:
        groups.append(cur)
        cur = []
    cur.append(b)
groups.append(cur)
out = []
for g in groups:
    span = g[-1].time_range.end - g[0].time_range.start
    busy = sum(e.time_range.end - e.time_range.start for e in g)
    gaps = sorted(((b.time_range.start - a.time_range.end, a.name[:40], b.name[:40]) for a, b in zip(g, g[1:])),
                  reverse=True)
    out.append({"kernels": len(g), "span_us": round(span, 1), "kernel_sum_us": round(busy, 1),
                "gap_sum_us": round(sum(x[0] for x in gaps), 1),
                "median_gap_us": round(sorted(x[0] for x in gaps)[len(gaps) // 2], 2),
                "largest_gaps": [(round(x[0], 1), x[1], x[2]) for x in gaps[:5]]})
for o in out:
    print(json.dumps(o))
# per-kernel time inside the graph, averaged over the steps (ms per step)
per = {}
for g in groups:
    for e in g:
        k = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "").replace("fv3b::", "")
        per[k] = per.get(k, 0.0) + (e.time_range.end - e.time_range.start) / 1e3 / len(groups)
print(json.dumps({"graph_ms_per_step_by_kernel": {k: round(v, 4) for k, v in sorted(per.items(), key=lambda x: -x[1])}}))
