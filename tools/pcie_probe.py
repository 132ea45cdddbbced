"""Pinned host <-> device copy bandwidth on this box (the bound of bench.py's
e2e number): 25 MB transfers (one state field), H2D alone, D2H alone and both
directions at once on two streams.  Prints one JSON line."""
import json
import torch

n = 198 * 198 * 81
reps = 14
h = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(2)]
d = [torch.empty(n, dtype=torch.float64, device="cuda") for _ in range(2)]
up, down = torch.cuda.Stream(), torch.cuda.Stream()


def run(do_up, do_down, rounds=5):
    best = 0.0
    for _ in range(rounds):
        torch.cuda.synchronize()
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        up.wait_stream(torch.cuda.current_stream())
        down.wait_stream(torch.cuda.current_stream())
        for _ in range(reps):
            if do_up:
                with torch.cuda.stream(up):
                    d[0].copy_(h[0], non_blocking=True)
            if do_down:
                with torch.cuda.stream(down):
                    h[1].copy_(d[1], non_blocking=True)
        torch.cuda.current_stream().wait_stream(up)
        torch.cuda.current_stream().wait_stream(down)
        e.record()
        e.synchronize()
        best = max(best, reps * n * 8 / (s.elapsed_time(e) * 1e-3) / 1e9)
    return best


out = {"bytes_per_copy": n * 8, "h2d_GBps": run(True, False), "d2h_GBps": run(False, True),
       "bidir_GBps_per_direction": run(True, True)}
print(json.dumps(out))
