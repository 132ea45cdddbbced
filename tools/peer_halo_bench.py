"""Halo-update cost on one GPU: the 2 x 2 loopback decomposition of the C2
domain (4 blocks of 96 x 96 x 80) with message buffers (pack / device copy /
unpack, the NCCL path's structure) versus peer-memory stores
(fv3b_halo_peer_rects, PeerHalo), and the single-domain periodic fill.
Prints one JSON line per field group."""

from __future__ import annotations

import json

import torch

from paper_2205_04148_b200.config import RunConfig
from paper_2205_04148_b200.dycore import Dycore
from paper_2205_04148_b200.parallel import LoopbackCluster


def timed(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps * 1e3


def main():
    nk, nq = 80, 8
    blk = RunConfig(ni=96, nj=96, nk=nk, nq=nq)
    glob = RunConfig(ni=192, nj=192, nk=nk, nq=nq)
    groups = {"dsw": ["u", "v", "w", "delp", "pt", "gz"], "c": ["uc", "vc"],
              "tracers": glob.tracer_names() + ["delp"]}
    single = Dycore(glob)
    packed = LoopbackCluster([Dycore(blk) for _ in range(4)], 2, 2)
    direct = LoopbackCluster([Dycore(blk) for _ in range(4)], 2, 2, direct=True)
    flags = LoopbackCluster([Dycore(blk) for _ in range(4)], 2, 2, direct=True, flag_sync=True)
    for g, names in groups.items():
        out = {"group": g, "fields": len(names)}
        out["single_us"] = timed(lambda: single.halo.update(names))
        out["packed_us"] = timed(lambda: packed.exchange_all([names] * 4))
        out["direct_us"] = timed(lambda: direct.exchange_all([names] * 4))

        def flagged():
            for s in flags.streams:
                s.wait_stream(torch.cuda.current_stream())
            flags.exchange_all([names] * 4)
            for s in flags.streams:
                torch.cuda.current_stream().wait_stream(s)

        out["flags_us"] = timed(flagged)
        # the same as captured graphs (launch overhead removed)
        for key, fn in (("packed_graph_us", lambda: packed.exchange_all([names] * 4)),
                        ("direct_graph_us", lambda: direct.exchange_all([names] * 4)),
                        ("flags_graph_us", flagged)):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            out[key] = timed(gr.replay)
        print(json.dumps({k: (round(v, 1) if isinstance(v, float) else v) for k, v in out.items()}), flush=True)


if __name__ == "__main__":
    main()
