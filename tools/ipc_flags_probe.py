"""Two processes on one GPU exchanging halos through CUDA IPC with the
device-side neighbour barrier (FlagSync) instead of host barriers.  The
contexts time-slice on one device, so this checks the protocol, not speed.
Bitwise check against the single-domain dycore, as the GPU test does."""

from __future__ import annotations

import socket
import sys
import time

sys.path.insert(0, "tests")

import numpy as np  # noqa: E402
import torch  # noqa: E402

from test_gpu_parallel import _block, _ipc_worker  # noqa: E402


def main():
    from paper_2205_04148_b200.config import RunConfig
    from paper_2205_04148_b200.dycore import Dycore
    from paper_2205_04148_b200.state import initial_state

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = torch.multiprocessing.get_context("spawn")
    q = ctx.Queue()
    t0 = time.time()
    procs = [ctx.Process(target=_ipc_worker, args=(r, port, q, True)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    ni, nj, nk = 32, 24, 8
    cfg = RunConfig(ni=ni, nj=2 * nj, nk=nk, n_split=2, nq=2, dt_atmos=30.0)
    ref = Dycore(cfg, initial_state(cfg))
    for _ in range(2):
        ref.step()
    torch.cuda.synchronize()
    h = cfg.halo
    full = ref.download(list(res[0]))
    ok = all(np.array_equal(got, _block(full[n], 0, r, ni, nj, h)[h:-h, h:-h]) for r in range(2) for n, got in res[r].items())
    print({"bitwise": ok, "seconds": round(time.time() - t0, 1)})


if __name__ == "__main__":
    main()
