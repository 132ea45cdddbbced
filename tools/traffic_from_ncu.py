"""Per-program DRAM traffic and fp64 thread operations per launch from one
ncu --set full capture of a single eager C2 step with n_split = 1
(tools/profile_step.py 1 1), written to profiles/traffic.json (bench.py's
roofline ``traffic`` field) and profiles/fp64.json (its ``fp64`` roofline:
DADD + DMUL + DFMA thread instructions, each one fp64 operation issue).

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
FP64 = [f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum.per_cycle_elapsed" for o in ("dadd", "dmul", "dfma")]


def launches(rep, what="bytes"):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    u = dict(zip(hdr, units))
    nb = lambda d, key: float(d[key]) * SCALE.get(u[key], 1.0)

    def ops(d):  # (summed over sub-partitions) per-cycle rates x elapsed cycles
        cyc = float(d["smsp__cycles_elapsed.avg"])
        return sum(float(d[k]) for k in FP64 if d.get(k) not in (None, "", "n/a")) * cyc

    rows = [dict(zip(hdr, x)) for x in r[2:]]
    if what == "fp64":
        return [(d["Kernel Name"], ops(d)) for d in rows]
    return [(d["Kernel Name"], nb(d, "dram__bytes_read.sum") + nb(d, "dram__bytes_write.sum")) for d in rows]


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
        elif "remap_map" in name:  # (the scalars' launch, then the winds' and pt's)
            key = "remap_map_winds" if "remap_map" in prog else "remap_map"
        elif "face_thickness" in name:
            key = "remap_faces"
        elif "log_thickness" in name:
            key = "remap_logp"
        elif "halo" in name:
            key = "halo"
        else:
            continue
        prog[key] = prog.get(key, 0.0) + b
    return prog


names = ", ".join(Path(r).name for r in sys.argv[1:])
for what, path, src in (("bytes", "profiles/traffic.json", "dram__bytes_read.sum + dram__bytes_write.sum per launch"),
                        ("fp64", "profiles/fp64.json", "fp64 thread operations (DADD + DMUL + DFMA) per launch")):
    prog = {}
    for rep in sys.argv[1:]:
        prog.update({k: v for k, v in programs(launches(rep, what)).items() if v > 0 or what == "bytes"})
    prog["_source"] = f"ncu --set full, {names}: {src}"
    Path(path).write_text(json.dumps(prog, indent=1, sort_keys=True) + "\n")
    print(json.dumps(prog, indent=1))
