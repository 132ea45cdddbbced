"""measure_bandwidth (the copy-stencil probe) against the
measured HBM peak: python tools/bw_probe.py"""
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2205_04148_b200.executor import measure_bandwidth  # noqa: E402

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] * 1e9
for mib in (512, 1024, 2048):
    bw = measure_bandwidth(mib * 2**20, reps=20)
    print(json.dumps({"domain_MiB": mib, "copy_GBps": round(bw / 1e9, 1), "peak_GBps": peak / 1e9,
                      "frac": round(bw / peak, 3)}))
