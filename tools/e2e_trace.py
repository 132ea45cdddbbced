"""Per-stream timeline of pipelined Dycore.step_host calls (C2): events
recorded around each phase on the upload, compute and download streams
(monkeypatched into step_host's own copy / transpose calls), printed as
start-end milliseconds relative to the first call."""

from __future__ import annotations

import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2205_04148_b200.config import RunConfig  # noqa: E402
from paper_2205_04148_b200.dycore import Dycore  # noqa: E402
from paper_2205_04148_b200.state import initial_state  # noqa: E402


def main():
    cfg = RunConfig()
    st = initial_state(cfg)
    d = Dycore(cfg, st)
    h_in, h_out = d.host_buffers(), d.host_buffers()
    for n, t in h_in.items():
        t.copy_(torch.from_numpy(st[n]))
    for _ in range(3):
        d.step_host(h_in, h_out)
    torch.cuda.synchronize()
    marks = []
    orig_runs = Dycore._runs

    def runs(names, a, b):  # every transfer run: events on the current (copy) stream around it
        out = orig_runs(names, a, b)
        s = torch.cuda.current_stream()
        res = []
        for x, y in out:
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)

            class _V:  # wraps dst.copy_ to bracket it with events
                def __init__(self, t):
                    self.t = t

                def copy_(self, src, non_blocking=False):
                    e0.record(torch.cuda.current_stream())
                    self.t.copy_(src, non_blocking=non_blocking)
                    e1.record(torch.cuda.current_stream())
                    marks.append(("up" if self.t.is_cuda else "down", len(names), e0, e1))

            res.append((_V(x), y))
        return res

    Dycore._runs = staticmethod(runs)
    comp = torch.cuda.current_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t0.record(comp)
    starts = []
    for _ in range(6):
        e = torch.cuda.Event(enable_timing=True)
        e.record(comp)
        starts.append(e)
        done = d.step_host(h_in, h_out)
    comp.wait_event(done)
    t1 = torch.cuda.Event(enable_timing=True)
    t1.record(comp)
    torch.cuda.synchronize()
    print(f"period {t0.elapsed_time(t1) / 6:.2f} ms")
    print("compute enqueue points:", [round(t0.elapsed_time(e), 2) for e in starts])
    for kind, n, a, b in marks:
        print(f"{kind:4s} {n:2d} fields  {t0.elapsed_time(a):7.2f} -> {t0.elapsed_time(b):7.2f}")


if __name__ == "__main__":
    main()
