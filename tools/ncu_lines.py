"""Top CUDA source lines of one kernel in an ncu report by warp-stall samples
and executed instructions:  python tools/ncu_lines.py REP KERNEL_REGEX [N] [launch]"""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = sys.argv[4] if len(sys.argv) > 4 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--launch-skip", skip,
                      "--launch-count", "1", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for x in csv.reader(io.StringIO(out)):
    if not x:
        continue
    if x[0] in ("File Name", "File Path"):
        fname = x[1].split("/")[-1]
    elif x[0] == "Line No":
        hdr = x
    elif hdr and x[0].isdigit() and len(x) == len(hdr):
        rows.append((fname, x))
s_i = hdr.index("Warp Stall Sampling (All Samples)")
i_i = hdr.index("Instructions Executed")
f = lambda v: float(v) if v not in ("", "-") else 0.0
ts = sum(f(x[s_i]) for _, x in rows) or 1
ti = sum(f(x[i_i]) for _, x in rows) or 1
print(f"samples {ts:.0f} instructions {ti:.0f}")
for fn, x in sorted(rows, key=lambda r: -f(r[1][s_i]))[:n]:
    print(f"{fn[:14]:>14}:{x[0]:<4} stall {100 * f(x[s_i]) / ts:5.1f}%  inst {100 * f(x[i_i]) / ti:5.1f}%  {x[1].strip()[:90]}")
