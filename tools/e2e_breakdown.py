"""Where the end-to-end step time goes (C2, one B200): device step eager vs
CUDA-graph replay, the interior-column uploads / downloads alone and both
directions at once, and the pipelined step_host period.  Milliseconds."""

from __future__ import annotations

import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import torch  # noqa: E402

from paper_2205_04148_b200.config import RunConfig  # noqa: E402
from paper_2205_04148_b200.dycore import Dycore  # noqa: E402
from paper_2205_04148_b200.state import initial_state  # noqa: E402


def timed(fn, reps=8):
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
    st = initial_state(cfg)
    d = Dycore(cfg, st)
    h_in, h_out = d.host_buffers(), d.host_buffers()
    for n, t in h_in.items():
        t.copy_(torch.from_numpy(st[n]))
    out = {}
    out["eager_step"] = timed(d.step)
    d.capture()
    out["graph_step"] = timed(d.replay)
    stages = d._io_stages(list(h_in))
    up, down = d._io_streams()
    comp = torch.cuda.current_stream()

    def xfer(do_up, do_down):
        def run():
            up.wait_stream(comp)
            down.wait_stream(comp)
            if do_up:
                with torch.cuda.stream(up):
                    for n in h_in:
                        stages[0][0][n].copy_(h_in[n], non_blocking=True)
            if do_down:
                with torch.cuda.stream(down):
                    for n in h_out:
                        h_out[n].copy_(stages[1][0][n], non_blocking=True)
            comp.wait_stream(up)
            comp.wait_stream(down)
        return run

    out["upload_only"] = timed(xfer(True, False))
    out["download_only"] = timed(xfer(False, True))
    out["both"] = timed(xfer(True, True))
    # host enqueue cost of one eager step_host call
    import time
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(4):
        d.step_host(h_in, h_out)
    host_ms = (time.perf_counter() - t) / 4 * 1e3
    torch.cuda.synchronize()
    out["step_host_enqueue_host_ms"] = host_ms

    def e2e():
        done = d.step_host(h_in, h_out)
        comp.wait_event(done)

    out["step_host_period"] = timed(lambda: d.step_host(h_in, h_out), reps=10)
    out["step_host_serial"] = timed(e2e, reps=4)
    out["bytes_each_way_MB"] = sum(t.numel() * 8 for t in h_in.values()) / 1e6
    print(json.dumps({k: round(v, 3) for k, v in out.items()}))


if __name__ == "__main__":
    main()
