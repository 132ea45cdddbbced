"""Algorithmic fp64 operations per launch of every dycore program (the
compute-side counterpart of the first-touch bytes): the shipped .stn program
evaluated once per point, as the reference interpreter does -- every
statement's arithmetic over its iteration plane (non-temporaries the
interior, temporaries their extension, region statements their resolved
cells; reference.py:261-281) and its levels -- with no tile-halo
recomputation, no fast-path reciprocal refinement and no range tests.

Counts per launch: add (+, -), mul, div, sqrt, transcendental calls (log,
exp), and the non-arithmetic compare / min / max / select separately.
``fp64_ops`` = add + mul + div + sqrt + transcendental, each counted once
(a division costs about 14 DFMA-pipe operations on the B200, log ~25, so
the executed count the ncu DADD + DMUL + DFMA figure measures is larger even
without redundancy).  Written into paper_2205_04148_b200/traffic_table.json
(key ``algorithmic_ops``), which bench.py reports beside the executed count.

    python tools/opcount.py [ni]
"""
import json
import sys
from collections import Counter
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from oracle import interp  # noqa: E402

nk = 80
PROGS = [("c_grid", nk + 1), ("d_sw", nk), ("nh_d", nk + 1), ("p_grad_d", nk + 1), ("tracer_2d", nk),
         ("remap_tracers", nk + 1)]


def expr_ops(e, c: Counter) -> Counter:
    tag = e[0]
    if tag in ("c", "s", "f"):
        return c
    if tag == "neg":
        return expr_ops(e[1], c)  # a sign flip (an operand modifier in SASS)
    if tag == "bin":
        c[{"+": "add", "-": "add", "*": "mul", "/": "div"}.get(e[1], "pow")] += 1
        expr_ops(e[2], c)
        return expr_ops(e[3], c)
    if tag == "cmp":
        c["cmp"] += 1
        expr_ops(e[2], c)
        return expr_ops(e[3], c)
    if tag == "call":
        c[{"sqrt": "sqrt", "log": "transcendental", "exp": "transcendental", "abs": "cmp", "min": "cmp",
           "max": "cmp", "select": "cmp"}[e[1]]] += 1
        for a in e[2]:
            expr_ops(a, c)
        return c
    raise TypeError(e)


class _Shape:
    """The parts of the interpreter context _ranges reads (no arrays)."""

    def __init__(self, doc, domain):
        self.decl = {f["name"]: f for f in doc["program"]["fields"]}
        self.ext = doc["requirements"]["extension"]
        self.sizes = dict(zip("IJK", domain))


def program_ops(name: str, domain, placement=interp.PERIODIC) -> dict:
    doc = interp.load_manifest(name)
    ctx = _Shape(doc, domain)
    stencils = {s["name"]: s for s in doc["program"]["stencils"]}
    total = Counter()
    for stencil, _ in doc["trace"]:
        for block in stencils[stencil]["blocks"]:
            k0, k1 = interp._resolve_interval(block["interval"], domain[2])
            levels = max(0, k1 - k0)
            for s in block["statements"]:
                r = interp._ranges(ctx, s, placement)
                if r is None:
                    continue
                pts = (r["I"][1] - r["I"][0]) * (r["J"][1] - r["J"][0]) * levels
                for op, n in expr_ops(s["expr"], Counter()).items():
                    total[op] += n * pts
    out = dict(sorted(total.items()))
    out["fp64_ops"] = sum(total[o] for o in ("add", "mul", "div", "sqrt", "transcendental", "pow"))
    out["cells"] = domain[0] * domain[1] * domain[2]
    return out


if __name__ == "__main__":
    ni = int(sys.argv[1]) if len(sys.argv) > 1 else 192
    path = ROOT / "paper_2205_04148_b200" / "traffic_table.json"
    table = json.loads(path.read_text()) if path.exists() else {}
    for name, k in PROGS:
        dom = (ni, ni, k)
        row = table.setdefault(f"{name}@{ni}x{ni}x{k}", {})
        row["algorithmic_ops"] = program_ops(name, dom)
        print(name, dom, row["algorithmic_ops"], f"{row['algorithmic_ops']['fp64_ops'] / row['algorithmic_ops']['cells']:.1f} per cell")
    path.write_text(json.dumps(table, indent=1, sort_keys=True) + "\n")
