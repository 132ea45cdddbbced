"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples
and executed instructions:  python tools/ncu_lines.py REP KERNEL_REGEX [N] [launch]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(out)))
hi = next(i for i, x in enumerate(r) if x and x[0] == "Line No")
hdr = r[hi]
rows = [x for x in r[hi + 1:] if len(x) > 8 and x[0].isdigit()]
s_i = hdr.index("Warp Stall Sampling (All Samples)")
i_i = hdr.index("Instructions Executed")
f = lambda v: float(v) if v not in ("", "-") else 0.0
ts = sum(f(x[s_i]) for x in rows) or 1
ti = sum(f(x[i_i]) for x in rows) or 1
print(f"samples {ts:.0f} instructions {ti:.0f}")
for x in sorted(rows, key=lambda x: -f(x[s_i]))[:n]:
    print(f"{x[0]:>5} stall {100 * f(x[s_i]) / ts:5.1f}%  inst {100 * f(x[i_i]) / ti:5.1f}%  {x[1].strip()[:100]}")
