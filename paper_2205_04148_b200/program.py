"""Canonical, JSON-serialisable form of a stencil program, plus the pieces of
the reference front end the B200 engine needs at run time.

The engine is a drop-in for ``stencilkit.executor.reference.run_reference``
(reference ``pkg/src/stencilkit/executor/reference.py:307-339``).  A caller
hands it the program object it already has.  Two program sources are
accepted:

* a ``stencilkit.frontend.ast.StencilProgram`` (the reference AST,
  ``frontend/ast.py:333-347``).  It is walked duck-typed by class name, so
  the reference package does not have to be importable on the GPU host;
* a :class:`Program` loaded from one of this package's manifests
  (``programs/<name>.json``), written by ``tools/gen_programs.py`` from the
  ``.stn`` sources next to it.

Both become the same canonical tree.  Its structural fingerprint (fields and
stencil bodies; constants and driver excluded) selects the hand-written
kernel plan; the driver is resolved here, restating ``resolve_driver``
(``frontend/validate.py:98-146``), so constants and loop counts may differ
from the manifest's.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from pathlib import Path
from typing import Any

PROGRAM_DIR = Path(__file__).resolve().parent / "programs"

# ---------------------------------------------------------------------------
# reference AST -> canonical tree (duck-typed; frontend/ast.py:69-347)
# ---------------------------------------------------------------------------


def _edge(e):
    return None if e is None else [e.anchor, int(e.offset)]


def _axis(c):
    return [c.kind, _edge(c.lo), _edge(c.hi)]


def canon_expr(e) -> list:
    kind = type(e).__name__
    if kind == "Const":
        return ["c", float(e.value)]
    if kind == "ScalarRef":
        return ["s", e.name]
    if kind == "FieldRead":
        o = e.offset
        return ["f", e.field, int(o.di), int(o.dj), int(o.dk)]
    if kind == "UnaryOp":
        return ["neg", canon_expr(e.operand)]
    if kind == "BinOp":
        return ["bin", e.op, canon_expr(e.lhs), canon_expr(e.rhs)]
    if kind == "Compare":
        return ["cmp", e.op, canon_expr(e.lhs), canon_expr(e.rhs)]
    if kind == "Call":
        return ["call", e.func, [canon_expr(a) for a in e.args]]
    raise TypeError(f"cannot canonicalise expression node {kind}")


def _canon_driver(stmts) -> list:
    out = []
    for s in stmts:
        kind = type(s).__name__
        if kind == "DriverAssign":
            out.append(["assign", s.name, canon_expr(s.expr)])
        elif kind == "DriverIf":
            out.append(["if", canon_expr(s.cond), _canon_driver(s.then), _canon_driver(s.orelse)])
        elif kind == "DriverLoop":
            out.append(["for", s.var, canon_expr(s.count), _canon_driver(s.body), bool(s.unroll)])
        elif kind == "DriverInvoke":
            out.append(["invoke", s.stencil, {k: canon_expr(v) for k, v in s.kwargs.items()}])
        else:
            raise TypeError(f"unknown driver statement {kind}")
    return out


def canonicalize(program) -> dict:
    """Canonical tree of a reference ``StencilProgram``."""
    stencils = []
    for s in program.stencils:
        blocks = []
        for b in s.blocks:
            iv = b.interval
            stmts = []
            for st in b.statements:
                region = None
                if st.region is not None:
                    region = {"i": _axis(st.region.i), "j": _axis(st.region.j)}
                stmts.append({"target": st.target, "expr": canon_expr(st.expr), "region": region})
            blocks.append(
                {
                    "policy": b.policy,
                    "interval": [[iv.start.anchor, int(iv.start.offset)], [iv.end.anchor, int(iv.end.offset)]],
                    "statements": stmts,
                }
            )
        stencils.append({"name": s.name, "params": list(s.params), "blocks": blocks})
    return {
        "consts": [[c.name, float(c.value)] for c in program.consts],
        "fields": [
            {"name": f.name, "dims": list(f.dims), "dtype": f.dtype, "temporary": bool(f.temporary)}
            for f in program.fields
        ],
        "stencils": stencils,
        "driver": _canon_driver(program.driver),
    }


def fingerprint(canon: dict) -> str:
    """Structural hash: field declarations and stencil bodies only."""
    doc = json.dumps({"fields": canon["fields"], "stencils": canon["stencils"]}, sort_keys=True)
    return hashlib.sha256(doc.encode()).hexdigest()[:16]


# ---------------------------------------------------------------------------
# driver resolution (restates frontend/validate.py:57-146)
# ---------------------------------------------------------------------------


class DriverResolutionError(Exception):
    pass


def _eval_driver(e, env: dict[str, float]) -> float:
    tag = e[0]
    if tag == "c":
        return e[1]
    if tag == "s":
        if e[1] not in env:
            raise DriverResolutionError(f"undefined name {e[1]!r}")
        return env[e[1]]
    if tag == "neg":
        return -_eval_driver(e[1], env)
    if tag == "bin":
        a, b = _eval_driver(e[2], env), _eval_driver(e[3], env)
        op = e[1]
        if op == "+":
            return a + b
        if op == "-":
            return a - b
        if op == "*":
            return a * b
        if op == "/":
            return a / b
        return a**b
    if tag == "cmp":
        a, b = _eval_driver(e[2], env), _eval_driver(e[3], env)
        return float({"<": a < b, "<=": a <= b, ">": a > b, ">=": a >= b, "==": a == b, "!=": a != b}[e[1]])
    raise DriverResolutionError("field reads and calls are not allowed in the driver")


def resolve_trace(canon: dict) -> list[tuple[str, dict[str, float]]]:
    """Straight-line invocation list ``[(stencil, kwargs)]``."""
    env = {n: v for n, v in canon["consts"]}
    trace: list[tuple[str, dict[str, float]]] = []

    def run(stmts):
        for s in stmts:
            tag = s[0]
            if tag == "assign":
                env[s[1]] = _eval_driver(s[2], env)
            elif tag == "if":
                run(s[2] if _eval_driver(s[1], env) != 0.0 else s[3])
            elif tag == "for":
                count = _eval_driver(s[2], env)
                if count != int(count) or count < 0:
                    raise DriverResolutionError(f"loop trip count must be a non-negative integer, got {count!r}")
                for it in range(int(count)):
                    env[s[1]] = float(it)
                    run(s[3])
                env.pop(s[1], None)
            elif tag == "invoke":
                trace.append((s[1], {k: float(_eval_driver(v, env)) for k, v in sorted(s[2].items())}))

    run(canon["driver"])
    return trace


# ---------------------------------------------------------------------------
# Program: canonical tree + manifest requirements
# ---------------------------------------------------------------------------


@dataclass(frozen=True)
class FieldInfo:
    name: str
    dims: tuple[str, ...]
    dtype: str
    temporary: bool
    extent: tuple[tuple[int, int], tuple[int, int], tuple[int, int]]  # (lo<=0, hi>=0) per I,J,K

    def halo(self, axis: str) -> tuple[int, int]:
        lo, hi = self.extent["IJK".index(axis)]
        return -lo, hi

    def shape(self, domain: tuple[int, int, int]) -> tuple[int, ...]:
        out = []
        for axis in self.dims:
            lo, hi = self.halo(axis)
            out.append(lo + domain["IJK".index(axis)] + hi)
        return tuple(out)


@dataclass
class Program:
    """A program the engine knows: canonical tree + requirement contract.

    ``requirements`` is the output of the reference's own
    ``compute_requirements`` (``frontend/extents.py:108-188``) recorded in the
    manifest, so the allocation/shape contract is the reference's.
    """

    name: str
    canon: dict
    fields: dict[str, FieldInfo]
    extension: dict[str, dict[str, tuple[int, int]]]
    min_domain: tuple[int, int, int]
    consts: dict[str, float] = field(default_factory=dict)
    fp: str = ""

    @property
    def trace(self) -> list[tuple[str, dict[str, float]]]:
        if "trace" in self.canon:  # a lowered graph's resolved execution trace
            return [(n, dict(kw)) for n, kw in self.canon["trace"]]
        return resolve_trace(self.canon)

    def scalars(self, invoke_kwargs: dict[str, float]) -> dict[str, float]:
        s = dict(self.consts)
        s.update(invoke_kwargs)
        return s

    def non_temporaries(self) -> list[str]:
        return [n for n, f in self.fields.items() if not f.temporary]

    def check_domain(self, domain: tuple[int, int, int]) -> None:
        ni, nj, nk = domain
        mi, mj, mk = self.min_domain
        if ni < mi or nj < mj or nk < mk:
            raise ValueError(f"domain {domain} is below the program minimum {self.min_domain}")


def program_from_manifest(doc: dict) -> Program:
    req = doc["requirements"]
    fields = {}
    for f in doc["program"]["fields"]:
        ext = req["extent"][f["name"]]
        fields[f["name"]] = FieldInfo(
            name=f["name"],
            dims=tuple(f["dims"]),
            dtype=f["dtype"],
            temporary=f["temporary"],
            extent=tuple(tuple(x) for x in ext),
        )
    ext = {n: {a: tuple(v) for a, v in d.items()} for n, d in req["extension"].items()}
    canon = doc["program"]
    return Program(
        name=doc["name"],
        canon=canon,
        fields=fields,
        extension=ext,
        min_domain=tuple(req["min_domain"]),
        consts={n: v for n, v in canon["consts"]},
        fp=doc["fingerprint"],
    )


_CACHE: dict[str, Program] = {}


def load_program(name: str) -> Program:
    """Load ``programs/<name>.json`` (generated from ``programs/<name>.stn``)."""
    if name not in _CACHE:
        path = PROGRAM_DIR / f"{name}.json"
        if not path.exists():
            raise KeyError(f"no program manifest {path}")
        _CACHE[name] = program_from_manifest(json.loads(path.read_text()))
    return _CACHE[name]


def known_programs() -> dict[str, Program]:
    """All shipped manifests keyed by structural fingerprint."""
    out = {}
    for path in sorted(PROGRAM_DIR.glob("*.json")):
        p = load_program(path.stem)
        out[p.fp] = p
    return out


def known_programs_names() -> list[str]:
    return sorted(p.stem for p in PROGRAM_DIR.glob("*.json"))


def _structure_fp(canon: dict) -> str:
    """Fingerprint of fields + stencil blocks, without stencil parameter
    lists (a lowered graph does not carry them)."""
    st = [{"name": s["name"], "blocks": s["blocks"]} for s in canon["stencils"]]
    # (field catalogue by name: graph documents list arrays sorted, serialize.py:171-186)
    fields = sorted(canon["fields"], key=lambda f: f["name"])
    doc = json.dumps({"fields": fields, "stencils": st}, sort_keys=True)
    return hashlib.sha256(doc.encode()).hexdigest()[:16]


def is_graph(obj: Any) -> bool:
    return all(hasattr(obj, a) for a in ("arrays", "states", "execution_trace"))


def canonicalize_graph(graph) -> dict:
    """Canonical tree of a reference ``DataflowGraph`` (``ir/graph.py:257-355``,
    as produced by ``lower``): fields from its array catalog, stencils from
    its StencilNodes (node name ``<stencil>_<block>``, ``graph.py:138-143``)
    and the resolved invocation trace from ``execution_trace``
    (``graph.py:299-329``), the order ``run_reference_graph`` executes
    (``reference.py:342-365``).  Fused nodes (``a+b``) are not accepted."""
    fields = [{"name": n, "dims": list(a.dims), "dtype": a.dtype, "temporary": bool(a.transient)}
              for n, a in graph.arrays.items()]
    blocks: dict[str, dict[int, dict]] = {}
    order: list[str] = []
    by_state = {s.name: s for s in graph.states}
    trace = []
    for sname, env in graph.execution_trace():
        cur = None
        for node in by_state[sname].sequence:
            if "+" in node.name or len(node.blocks) != 1:
                raise KeyError(f"fused graph node {node.name!r} has no B200 kernel plan")
            stencil, bi = node.name.rsplit("_", 1)
            b = node.blocks[0]
            iv = b.interval
            stmts = []
            for st in b.statements:
                region = None
                if st.region is not None:
                    region = {"i": _axis(st.region.i), "j": _axis(st.region.j)}
                stmts.append({"target": st.target, "expr": canon_expr(st.expr), "region": region})
            if stencil not in blocks:
                blocks[stencil] = {}
                order.append(stencil)
            blocks[stencil][int(bi)] = {
                "policy": b.policy,
                "interval": [[iv.start.anchor, int(iv.start.offset)], [iv.end.anchor, int(iv.end.offset)]],
                "statements": stmts,
            }
            kw = {k: float(_eval_driver(canon_expr(v), dict(env))) for k, v in sorted(node.kwargs.items())}
            if cur is None or cur[0] != stencil:
                cur = (stencil, kw)
                trace.append(cur)
    stencils = [{"name": n, "params": [], "blocks": [blocks[n][i] for i in sorted(blocks[n])]} for n in order]
    consts = [[k, float(v)] for k, v in getattr(graph, "symbols", {}).items()]
    return {"consts": consts, "fields": fields, "stencils": stencils, "driver": [], "trace": trace}


def as_program(program: Any) -> Program:
    """Accept a :class:`Program`, a manifest name, a reference AST or a
    lowered reference ``DataflowGraph``.

    A reference ``StencilProgram`` is matched to a shipped manifest by
    structural fingerprint; its own constants and driver are kept.
    Raises ``KeyError`` when no hand-written plan exists for the program.
    """
    if isinstance(program, Program):
        return program
    if isinstance(program, str):
        return load_program(program)
    if is_graph(program):
        canon = canonicalize_graph(program)
        fp = _structure_fp(canon)
        known = {_structure_fp(p.canon): p for p in known_programs().values()}
        if fp not in known:
            raise KeyError(f"no B200 kernel plan for graph structure {fp}")
        base = known[fp]
        return Program(name=base.name, canon=canon, fields=base.fields, extension=base.extension,
                       min_domain=base.min_domain, consts={n: v for n, v in canon["consts"]}, fp=base.fp)
    canon = canonicalize(program)
    fp = fingerprint(canon)
    known = known_programs()
    if fp not in known:
        raise KeyError(
            f"no B200 kernel plan for program fingerprint {fp}; shipped programs: "
            + ", ".join(sorted(p.name for p in known.values()))
        )
    base = known[fp]
    return Program(
        name=base.name,
        canon=canon,
        fields=base.fields,
        extension=base.extension,
        min_domain=base.min_domain,
        consts={n: v for n, v in canon["consts"]},
        fp=fp,
    )
