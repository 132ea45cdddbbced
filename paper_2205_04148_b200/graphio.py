"""Graph persistence in the reference's document format.

The reference persists lowered dataflow graphs with ``graph_to_json`` /
``graph_from_json`` (``ir/serialize.py:154-306``): a versioned,
deterministic JSON document (``"format": "stencilkit-graph"``, version 1)
with the array catalogue (dims, dtype, transient, extent, extension,
``Layout``), the states and their StencilNodes (blocks, kwargs, schedule),
the transitions, loops and symbols.  This module reads and writes that
format without the reference package:

* :func:`graph_from_json` parses a document into a :class:`Graph` whose
  node, block and expression objects carry the reference class names, so the
  engine takes it wherever it takes a reference ``DataflowGraph``
  (``run_b200``, ``run_scheduled``; ``program.canonicalize_graph``), with
  ``execution_trace`` restating ``graph.py:299-329``;
* :func:`graph_to_json` writes a :class:`Graph` (or a reference
  ``DataflowGraph``) back, byte-identical to the reference writer for the
  same graph (sorted keys, indent 1);
* :func:`program_graph` builds the straight-line graph of a shipped program
  on a domain: one state per resolved driver invocation, one node per
  stencil block (``<stencil>_<block>``, ``graph.py:138-143``), arrays with
  the reference ``allocate_layout`` rule (``scheduling.py:377-407``) and the
  reference's extents.  The reference ``graph_from_json`` loads it and its
  ``run_reference_graph`` executes it (tests/test_graphio.py).

Memlets and expansions are derived data in the reference and are not part
of the document (``serialize.py:1-5``).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from typing import Any

from .program import Program, _eval_driver, as_program, canon_expr

FORMAT_NAME = "stencilkit-graph"
FORMAT_VERSION = 1
DEFAULT_ALIGNMENT = 8


class SerializationError(Exception):
    pass


# -- AST node types with the reference class names (frontend/ast.py) -------------


@dataclass(frozen=True)
class Offset:
    di: int
    dj: int
    dk: int


@dataclass(frozen=True)
class Const:
    value: float


@dataclass(frozen=True)
class ScalarRef:
    name: str


@dataclass(frozen=True)
class FieldRead:
    field: str
    offset: Offset


@dataclass(frozen=True)
class UnaryOp:
    op: str
    operand: Any


@dataclass(frozen=True)
class BinOp:
    op: str
    lhs: Any
    rhs: Any


@dataclass(frozen=True)
class Compare:
    op: str
    lhs: Any
    rhs: Any


@dataclass(frozen=True)
class Call:
    func: str
    args: tuple


@dataclass(frozen=True)
class VBound:
    anchor: str
    offset: int


@dataclass(frozen=True)
class Interval:
    start: VBound
    end: VBound


@dataclass(frozen=True)
class EdgeIndex:
    anchor: str
    offset: int


@dataclass(frozen=True)
class AxisConstraint:
    kind: str
    lo: EdgeIndex | None
    hi: EdgeIndex | None


@dataclass(frozen=True)
class HorizontalRegion:
    i: AxisConstraint
    j: AxisConstraint


@dataclass(frozen=True)
class Statement:
    target: str
    expr: Any
    region: HorizontalRegion | None = None


@dataclass(frozen=True)
class ComputationBlock:
    policy: str
    interval: Interval
    statements: list


# -- graph containers (ir/graph.py:226-355) ----------------------------------------


@dataclass
class ArrayInfo:
    name: str
    dims: tuple
    dtype: str
    transient: bool
    extent: dict          # {"i": [lo, hi], "j": ..., "k": ...}
    layout: dict          # Layout.to_json
    extension: dict = field(default_factory=dict)


@dataclass
class StencilNode:
    name: str
    uid: str
    blocks: list
    kwargs: dict
    schedule: dict        # Schedule.to_json
    participants: tuple = ()


@dataclass
class DataflowState:
    name: str
    sequence: list = field(default_factory=list)


@dataclass
class Transition:
    src: str
    dst: str
    condition: tuple | None
    assignments: dict


@dataclass
class RankPlacement:
    own_i_start: bool = True
    own_i_end: bool = True
    own_j_start: bool = True
    own_j_end: bool = True


@dataclass
class Graph:
    arrays: dict
    states: list
    transitions: list
    start_state: str
    symbols: dict
    domain: tuple
    placement: RankPlacement
    alignment: int = DEFAULT_ALIGNMENT
    loops: list = field(default_factory=list)
    version: int = 0

    def out_transitions(self, state: str) -> list:
        return [t for t in self.transitions if t.src == state]

    def execution_trace(self, max_steps: int = 1_000_000) -> list:
        """The executed state sequence with the symbol environment at each
        state entry (restates graph.py:299-329)."""
        env = dict(self.symbols)
        out = [(self.start_state, dict(env))]
        current, steps = self.start_state, 0
        while True:
            outs = self.out_transitions(current)
            if not outs:
                return out
            taken = None
            for t in outs:
                if t.condition is None:
                    taken = t
                    break
                expr, flag = t.condition
                if (_eval_driver(canon_expr(expr), env) != 0.0) == flag:
                    taken = t
                    break
            if taken is None:
                raise RuntimeError(f"no enabled transition out of state {current!r}")
            for name, expr in taken.assignments.items():
                env[name] = _eval_driver(canon_expr(expr), env)
            current = taken.dst
            out.append((current, dict(env)))
            steps += 1
            if steps > max_steps:
                raise RuntimeError("state machine does not terminate")

    def unrolled_trace(self) -> list:
        return [name for name, _ in self.execution_trace()]


# -- expressions (serialize.py:54-94) -------------------------------------------


def expr_to_json(e) -> Any:
    kind = type(e).__name__
    if kind == "Const":
        return {"k": "c", "v": e.value}
    if kind == "ScalarRef":
        return {"k": "s", "n": e.name}
    if kind == "FieldRead":
        return {"k": "r", "f": e.field, "o": [e.offset.di, e.offset.dj, e.offset.dk]}
    if kind == "UnaryOp":
        return {"k": "u", "x": expr_to_json(e.operand)}
    if kind == "BinOp":
        return {"k": "b", "op": e.op, "l": expr_to_json(e.lhs), "r": expr_to_json(e.rhs)}
    if kind == "Compare":
        return {"k": "cmp", "op": e.op, "l": expr_to_json(e.lhs), "r": expr_to_json(e.rhs)}
    if kind == "Call":
        return {"k": "f", "fn": e.func, "a": [expr_to_json(a) for a in e.args]}
    raise SerializationError(f"cannot serialize expression {e!r}")


def expr_from_json(doc: Any):
    kind = doc["k"]
    if kind == "c":
        return Const(doc["v"])
    if kind == "s":
        return ScalarRef(doc["n"])
    if kind == "r":
        di, dj, dk = doc["o"]
        return FieldRead(doc["f"], Offset(di, dj, dk))
    if kind == "u":
        return UnaryOp("-", expr_from_json(doc["x"]))
    if kind == "b":
        return BinOp(doc["op"], expr_from_json(doc["l"]), expr_from_json(doc["r"]))
    if kind == "cmp":
        return Compare(doc["op"], expr_from_json(doc["l"]), expr_from_json(doc["r"]))
    if kind == "f":
        return Call(doc["fn"], tuple(expr_from_json(a) for a in doc["a"]))
    raise SerializationError(f"unknown expression kind {kind!r}")


# -- blocks (serialize.py:97-148) -------------------------------------------------


def _region_to_json(r) -> Any:
    if r is None:
        return None

    def conv(c):
        def enc(e):
            return None if e is None else [e.anchor, e.offset]

        return {"kind": c.kind, "lo": enc(c.lo), "hi": enc(c.hi)}

    return {"i": conv(r.i), "j": conv(r.j)}


def _region_from_json(doc) -> HorizontalRegion | None:
    if doc is None:
        return None

    def conv(c):
        def dec(e):
            return None if e is None else EdgeIndex(e[0], e[1])

        return AxisConstraint(c["kind"], dec(c["lo"]), dec(c["hi"]))

    return HorizontalRegion(conv(doc["i"]), conv(doc["j"]))


def _block_to_json(b) -> Any:
    iv = b.interval
    return {
        "policy": b.policy,
        "interval": [iv.start.anchor, iv.start.offset, iv.end.anchor, iv.end.offset],
        "statements": [{"target": s.target, "expr": expr_to_json(s.expr), "region": _region_to_json(s.region)}
                       for s in b.statements],
    }


def _block_from_json(doc) -> ComputationBlock:
    iv = doc["interval"]
    return ComputationBlock(doc["policy"], Interval(VBound(iv[0], iv[1]), VBound(iv[2], iv[3])),
                            [Statement(s["target"], expr_from_json(s["expr"]), _region_from_json(s["region"]))
                             for s in doc["statements"]])


# -- documents ---------------------------------------------------------------------


def _extent_doc(e) -> dict:
    if isinstance(e, dict):
        return {a: list(e[a]) for a in ("i", "j", "k")}
    return {"i": list(e.i), "j": list(e.j), "k": list(e.k)}


def _layout_doc(lay) -> dict:
    return dict(lay) if isinstance(lay, dict) else lay.to_json()


def _schedule_doc(s) -> dict:
    return dict(s) if isinstance(s, dict) else s.to_json()


def graph_to_json(graph) -> str:
    """The reference document of ``graph`` (a :class:`Graph` or a reference
    ``DataflowGraph``): serialize.py:154-228, same keys and ordering."""
    p = graph.placement
    doc = {
        "format": FORMAT_NAME,
        "version": FORMAT_VERSION,
        "domain": list(graph.domain),
        "alignment": graph.alignment,
        "start_state": graph.start_state,
        "symbols": dict(sorted(graph.symbols.items())),
        "placement": {"own_i_start": p.own_i_start, "own_i_end": p.own_i_end, "own_j_start": p.own_j_start,
                      "own_j_end": p.own_j_end},
        "graph_version": graph.version,
        "arrays": {
            name: {
                "dims": list(info.dims),
                "dtype": info.dtype,
                "transient": info.transient,
                "extent": _extent_doc(info.extent),
                "extension": {a: list(r) for a, r in sorted(info.extension.items())},
                "layout": _layout_doc(info.layout),
            }
            for name, info in sorted(graph.arrays.items())
        },
        "states": [
            {
                "name": state.name,
                "nodes": [
                    {
                        "name": node.name,
                        "uid": node.uid,
                        "participants": list(node.participants),
                        "kwargs": {k: expr_to_json(v) for k, v in sorted(node.kwargs.items())},
                        "schedule": _schedule_doc(node.schedule),
                        "blocks": [_block_to_json(b) for b in node.blocks],
                    }
                    for node in state.sequence
                ],
            }
            for state in graph.states
        ],
        "transitions": [
            {
                "src": t.src,
                "dst": t.dst,
                "condition": None if t.condition is None else {"expr": expr_to_json(t.condition[0]),
                                                               "flag": t.condition[1]},
                "assignments": {k: expr_to_json(v) for k, v in sorted(t.assignments.items())},
            }
            for t in graph.transitions
        ],
        "loops": [
            {"var": lp.var, "count": expr_to_json(lp.count), "guard": lp.guard, "body": list(lp.body),
             "exit": lp.exit, "unrollable": lp.unrollable}
            for lp in graph.loops
        ],
    }
    return json.dumps(doc, indent=1, sort_keys=True)


@dataclass
class LoopInfo:
    var: str
    count: Any
    guard: str
    body: list
    exit: str
    unrollable: bool


def graph_from_json(text: str) -> Graph:
    """Parse a reference graph document (serialize.py:231-306)."""
    doc = json.loads(text)
    if doc.get("format") != FORMAT_NAME:
        raise SerializationError("not a stencilkit graph document")
    if doc.get("version") != FORMAT_VERSION:
        raise SerializationError(f"unsupported graph format version {doc.get('version')!r}")
    arrays = {
        name: ArrayInfo(name=name, dims=tuple(a["dims"]), dtype=a["dtype"], transient=a["transient"],
                        extent={k: tuple(v) for k, v in a["extent"].items()}, layout=dict(a["layout"]),
                        extension={k: tuple(v) for k, v in a["extension"].items()})
        for name, a in doc["arrays"].items()
    }
    states = []
    for sdoc in doc["states"]:
        st = DataflowState(name=sdoc["name"])
        for n in sdoc["nodes"]:
            st.sequence.append(StencilNode(name=n["name"], uid=n["uid"],
                                           blocks=[_block_from_json(b) for b in n["blocks"]],
                                           kwargs={k: expr_from_json(v) for k, v in n["kwargs"].items()},
                                           schedule=dict(n["schedule"]), participants=tuple(n["participants"])))
        states.append(st)
    transitions = [Transition(t["src"], t["dst"],
                              None if t["condition"] is None else (expr_from_json(t["condition"]["expr"]),
                                                                   t["condition"]["flag"]),
                              {k: expr_from_json(v) for k, v in t["assignments"].items()})
                   for t in doc["transitions"]]
    loops = [LoopInfo(lp["var"], expr_from_json(lp["count"]), lp["guard"], list(lp["body"]), lp["exit"],
                      lp["unrollable"]) for lp in doc["loops"]]
    return Graph(arrays=arrays, states=states, transitions=transitions, start_state=doc["start_state"],
                 symbols=dict(doc["symbols"]), domain=tuple(doc["domain"]),
                 placement=RankPlacement(**doc["placement"]), alignment=doc["alignment"], loops=loops,
                 version=doc["graph_version"])


# -- the straight-line graph of a shipped program -------------------------------------


def _expr_from_canon(c):
    tag = c[0]
    if tag == "c":
        return Const(c[1])
    if tag == "s":
        return ScalarRef(c[1])
    if tag == "f":
        return FieldRead(c[1], Offset(c[2], c[3], c[4]))
    if tag == "neg":
        return UnaryOp("-", _expr_from_canon(c[1]))
    if tag == "bin":
        return BinOp(c[1], _expr_from_canon(c[2]), _expr_from_canon(c[3]))
    if tag == "cmp":
        return Compare(c[1], _expr_from_canon(c[2]), _expr_from_canon(c[3]))
    if tag == "call":
        return Call(c[1], tuple(_expr_from_canon(a) for a in c[2]))
    raise SerializationError(f"unknown canonical expression {tag!r}")


def _block_from_canon(b) -> ComputationBlock:
    (sa, so), (ea, eo) = b["interval"]
    stmts = []
    for s in b["statements"]:
        region = None
        if s["region"] is not None:
            def ax(c):
                return AxisConstraint(c[0], None if c[1] is None else EdgeIndex(*c[1]),
                                      None if c[2] is None else EdgeIndex(*c[2]))

            region = HorizontalRegion(ax(s["region"]["i"]), ax(s["region"]["j"]))
        stmts.append(Statement(s["target"], _expr_from_canon(s["expr"]), region))
    return ComputationBlock(b["policy"], Interval(VBound(sa, so), VBound(ea, eo)), stmts)


def allocate_layout(dims, extent: dict, domain, alignment: int = DEFAULT_ALIGNMENT) -> dict:
    """The reference Layout rule (scheduling.py:377-407) as its JSON document."""
    sizes = dict(zip(("I", "J", "K"), domain))
    shape, halo_lo = [], []
    for axis in dims:
        lo, hi = extent[axis.lower()]
        shape.append(-lo + sizes[axis] + hi)
        halo_lo.append(-lo)
    padded = list(shape)
    if dims:
        padded[0] = -(-shape[0] // alignment) * alignment
    strides, acc = [0] * len(dims), 1
    for d in range(len(dims)):
        strides[d] = acc
        acc *= padded[d]
    pre_pad = (alignment - (halo_lo[0] % alignment)) % alignment if dims else 0
    return {"dims": list(dims), "shape": shape, "halo_lo": halo_lo, "strides": strides, "pre_pad": pre_pad,
            "alignment": alignment}


DEFAULT_SCHEDULE = {"dim_order": ["Interval", "Operation", "K", "J", "I"], "tile_i": None, "tile_j": None,
                    "loop_dims": [], "caches": [], "region_strategy": "predicated"}
VERTICAL_SCHEDULE = {**DEFAULT_SCHEDULE, "dim_order": ["J", "I", "Interval", "Operation", "K"], "loop_dims": ["K"]}


def program_graph(program, domain, placement=(True, True, True, True)) -> Graph:
    """Straight-line graph of a shipped program (a :class:`Program` or name):
    state ``s<n>`` per resolved invocation with its kwargs as constants,
    node ``<stencil>_<block>`` per block, the reference's array catalogue
    (extents and extensions from the manifest, Layouts by allocate_layout),
    the paper's default schedules (scheduling.py:247-263: a sequential K
    loop for FORWARD / BACKWARD blocks, caches left empty)."""
    prog = as_program(program)
    canon = prog.canon
    arrays = {}
    for f in canon["fields"]:
        name = f["name"]
        ext = prog.fields[name].extent  # ((lo, hi) per I, J, K) from compute_requirements
        e = {"i": tuple(ext[0]), "j": tuple(ext[1]), "k": tuple(ext[2])}
        arrays[name] = ArrayInfo(name=name, dims=tuple(f["dims"]), dtype=f["dtype"], transient=f["temporary"],
                                 extent=e, layout=allocate_layout(tuple(f["dims"]), e, domain),
                                 extension={a: tuple(v) for a, v in prog.extension.get(name, {}).items()})
    by_name = {s["name"]: s for s in canon["stencils"]}
    states, transitions = [], []
    for n, (stencil, kwargs) in enumerate(prog.trace):
        st = DataflowState(name=f"s{n}")
        for b, block in enumerate(by_name[stencil]["blocks"]):
            sched = VERTICAL_SCHEDULE if block["policy"] in ("FORWARD", "BACKWARD") else DEFAULT_SCHEDULE
            st.sequence.append(StencilNode(name=f"{stencil}_{b}", uid=f"{stencil}_{b}@s{n}",
                                           blocks=[_block_from_canon(block)],
                                           kwargs={k: Const(float(v)) for k, v in kwargs.items()},
                                           schedule=dict(sched), participants=(f"{stencil}_{b}",)))
        states.append(st)
        if n:
            transitions.append(Transition(f"s{n - 1}", f"s{n}", None, {}))
    return Graph(arrays=arrays, states=states, transitions=transitions, start_state="s0",
                 symbols={k: float(v) for k, v in canon["consts"]}, domain=tuple(domain),
                 placement=RankPlacement(*(bool(x) for x in placement)))
