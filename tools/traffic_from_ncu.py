"""Per-program DRAM traffic per launch from one ncu --set full capture of a
single eager C2 step with n_split = 1 (tools/profile_step.py 1 1), written to
profiles/traffic.json for bench.py's roofline ``traffic`` field.

    python tools/traffic_from_ncu.py gpurun_out/prof_X.ncu-rep
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hdr, units = r[0], r[1]
rows = [dict(zip(hdr, x)) for x in r[2:]]
u = dict(zip(hdr, units))


def nbytes(d, key):
    return float(d[key]) * SCALE.get(u[key], 1.0)


seq = []
for d in rows:
    name = d["Kernel Name"]
    b = nbytes(d, "dram__bytes_read.sum") + nbytes(d, "dram__bytes_write.sum")
    seq.append((name, b))
# kernel order of one n_split = 1 step (halo launches interleaved)
prog = {}
riem_seen = 0
for name, b in seq:
    if "csw_kernel" in name or "p_grad_c" in name:
        key = "c_grid"
    elif "riem_kernel" in name:
        key = "c_grid" if riem_seen == 0 else "nh_d"
        riem_seen += 1
    elif "dsw_" in name:
        key = "d_sw"
    elif "p_grad_d" in name:
        key = "p_grad_d"
    elif "tp_kernel" in name:
        key = "tracer_2d"
    elif "remap_kernel" in name:
        key = "remap_tracers"
    elif "halo" in name:
        key = "halo"
    else:
        continue
    prog[key] = prog.get(key, 0.0) + b
prog["_source"] = f"ncu --set full, {Path(rep).name}: dram__bytes_read.sum + dram__bytes_write.sum per launch"
Path("profiles/traffic.json").write_text(json.dumps(prog, indent=1, sort_keys=True) + "\n")
print(json.dumps(prog, indent=1))
