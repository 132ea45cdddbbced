"""Per-program DRAM traffic per launch from one ncu --set full capture of a
single eager C2 step with n_split = 1 (tools/profile_step.py 1 1), written to
profiles/traffic.json for bench.py's roofline ``traffic`` field.

    python tools/traffic_from_ncu.py gpurun_out/prof_X.ncu-rep [more.ncu-rep ...]

Several reports (e.g. a full capture plus a re-capture of one kernel) are
read in order; a program's bytes come from the last report that has it.
"""
import csv
import io
import json
import subprocess
import sys
from pathlib import Path

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    u = dict(zip(hdr, units))
    nb = lambda d, key: float(d[key]) * SCALE.get(u[key], 1.0)
    return [(d["Kernel Name"], nb(d, "dram__bytes_read.sum") + nb(d, "dram__bytes_write.sum"))
            for d in (dict(zip(hdr, x)) for x in r[2:])]


def programs(seq):
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
        elif "tp_kernel" in name or "tracer2_kernel" in name:
            key = "tracer_2d"
        elif "remap_kernel" in name:
            key = "remap_tracers"
        elif "halo" in name:
            key = "halo"
        else:
            continue
        prog[key] = prog.get(key, 0.0) + b
    return prog


prog = {}
for rep in sys.argv[1:]:
    prog.update(programs(launches(rep)))
prog["_source"] = "ncu --set full, " + ", ".join(Path(r).name for r in sys.argv[1:]) + ": dram__bytes_read.sum + dram__bytes_write.sum per launch"
Path("profiles/traffic.json").write_text(json.dumps(prog, indent=1, sort_keys=True) + "\n")
print(json.dumps(prog, indent=1))
