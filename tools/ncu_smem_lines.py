"""Top CUDA source lines of one kernel by shared-memory wavefronts (and the
excess over ideal, i.e. bank conflicts):  python tools/ncu_smem_lines.py REP KERNEL_REGEX [N] [launch-skip]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
f = lambda v: float(v) if v not in ("", "-") else 0.0
acc = defaultdict(lambda: [0.0, 0.0, 0.0, ""])
fname, hdr = "?", None
for x in rows:
    if not x:
        continue
    if x[0] in ("File Name", "File Path"):
        fname = x[1].split("/")[-1]
    elif x[0] == "Line No":
        hdr = x
    elif hdr and x[0].isdigit() and len(x) == len(hdr):
        d = dict(zip(hdr[3:], x[3:]))
        a = acc[(fname, x[0])]
        a[0] += f(d.get("L1 Wavefronts Shared", ""))
        a[1] += f(d.get("L1 Wavefronts Shared Ideal", ""))
        a[2] += f(d.get("Warp Stall Sampling (All Samples)", ""))
        a[3] = x[1].strip()[:80]
tw = sum(v[0] for v in acc.values()) or 1
ti = sum(v[1] for v in acc.values()) or 1
print(f"shared wavefronts {tw:.0f} ideal {ti:.0f} excess {tw - ti:.0f}")
for (fn, ln), v in sorted(acc.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{fn[:14]:>14}:{ln:<4} wf {100 * v[0] / tw:5.1f}%  excess {100 * (v[0] - v[1]) / tw:5.1f}%  {v[3]}")
