"""Algorithmic (compulsory) HBM bytes of a program execution.

``bytes(K) = 8 * sum over non-temporary f of (|cells whose first access is a
read| + |cells written|)``; temporaries cost nothing (they live in shared
memory / registers).  Computed analytically from the reference's own extent
contract (``compute_requirements``, recorded in the manifest): a field whose
first access in the trace is a read contributes its whole touched box, a
written field its written cells (interior, plus region cells).  The tests
check this against a brute-force first-touch recorder run through the CPU
oracle (the ``AccessRecorder`` hook, ``reference.py:56-124``).
"""

from __future__ import annotations

from .program import Program, as_program


def _reads(e, out):
    tag = e[0]
    if tag == "f":
        out.add(e[1])
    elif tag == "neg":
        _reads(e[1], out)
    elif tag in ("bin", "cmp"):
        _reads(e[2], out)
        _reads(e[3], out)
    elif tag == "call":
        for a in e[2]:
            _reads(a, out)
    return out


def first_access(prog: Program) -> dict[str, str]:
    """'read' or 'write' per non-temporary field, in trace order."""
    stencils = {s["name"]: s for s in prog.canon["stencils"]}
    first: dict[str, str] = {}
    for stencil, _ in prog.trace:
        for block in stencils[stencil]["blocks"]:
            for st in block["statements"]:
                for f in sorted(_reads(st["expr"], set())):
                    if not prog.fields[f].temporary:
                        first.setdefault(f, "read")
                t = st["target"]
                if not prog.fields[t].temporary:
                    first.setdefault(t, "write")
    return first


def written_fields(prog: Program) -> set[str]:
    out = set()
    for s in prog.canon["stencils"]:
        for b in s["blocks"]:
            for st in b["statements"]:
                if not prog.fields[st["target"]].temporary:
                    out.add(st["target"])
    return out


def _interval_levels(prog: Program, name: str, nk: int) -> int:
    """Levels a field is written on (union of the intervals writing it)."""
    lv = set()
    for s in prog.canon["stencils"]:
        for b in s["blocks"]:
            if any(st["target"] == name for st in b["statements"]):
                a = [x[1] if x[0] == "start" else nk + x[1] for x in b["interval"]]
                lv.update(range(a[0], a[1]))
    return len(lv)


def compulsory_bytes(program, domain, itemsize: int = 8) -> int:
    prog = as_program(program)
    ni, nj, nk = domain
    first = first_access(prog)
    written = written_fields(prog)
    total = 0
    for name, kind in first.items():
        info = prog.fields[name]
        if kind == "read":
            cells = 1
            for n in info.shape(tuple(domain)):
                cells *= n
            total += cells
        if name in written:
            cells = 1
            for a in info.dims:
                cells *= {"I": ni, "J": nj}.get(a, 0) or _interval_levels(prog, name, nk)
            total += cells
    return total * itemsize
