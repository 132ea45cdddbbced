"""Bandwidth-bound performance model and the model-augmented kernel report
(the paper's Fig. 10; reference SPEC ``perf_model``, ``SPEC.md:436-503``),
on B200 measurements.

* :func:`model_kernel` — ``KernelBound`` of one program launch: unique
  (first-touch compulsory) bytes / machine bandwidth;
* :func:`build_report` — per kernel: measured time (max over invocation
  configurations, median over reps), modeled bound, utilization, flags;
  ranked by summed runtime grouped by kernel type;
* :func:`hotspot_list` — top kernels by grouped runtime x (1 - utilization);
* :func:`report_to_csv` — ``kernel,invocations,measured_s,bound_s,utilization,flags``
  (``SPEC.md:634``).

The bytes are the first-touch compulsory bytes of SURVEY 8d (the reference
AccessRecorder rule): brute-force values from ``traffic_table.json``
(tools/traffic_table.py) when the configuration is tabulated, else the
box model of :mod:`.traffic` (an upper bound: whole halo boxes).
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field
from pathlib import Path

from .traffic import compulsory_bytes

_TABLE = Path(__file__).resolve().parent / "traffic_table.json"


def unique_bytes(program: str, domain) -> tuple[int, str]:
    """(bytes, source) of one launch of `program` on `domain`.  The remap
    mapping (not a .stn program: its source-layer search is data dependent)
    takes ``domain = (ni, nj, nk + 1, nq)``."""
    if program == "remap_faces":  # fv3b_face_thickness: delp read, du / dv written
        ni, nj, nk = domain[:3]
        return 8 * 3 * ni * nj * nk, "analytic (each operand level once)"
    if program == "remap_logp":  # fv3b_log_thickness: delp read; dlnp, lnpe1, lnpe2 written
        ni, nj, nk = domain[:3]
        return 8 * ni * nj * (2 * nk + 2 * (nk + 1)), "analytic (each operand level once)"
    if program == "moist_pk":  # delp + moist tracers read; pe, peln, pk (interfaces), pkz, cvm written
        ni, nj, nki, nw = domain
        return 8 * ni * nj * ((1 + nw) * (nki - 1) + 3 * nki + 2 * (nki - 1)), "analytic (each operand level once)"
    if program in ("remap_map", "remap_map_winds"):
        ni, nj, nki, nq = domain
        cells = ni * nj * (nki - 1)
        # delp read and rewritten; per tracer q, a4_2, a4_3, a4_4 read, q_out written; ak, bk
        return 8 * (cells * (2 + 5 * nq) + 2 * nki), "analytic (each operand level once: upper bound)"
    if program == "remap_tracers" and len(domain) == 4:
        # the program profiles 8 tracers; the timestep's launch profiles `nfields`
        # fields of the same shape (bytes scale per field, delp aside)
        b8, src = unique_bytes(program, domain[:3])
        cells = domain[0] * domain[1] * domain[2]
        per = (b8 - 8 * cells) / 8
        return int(8 * cells + per * domain[3]), src + f", scaled to {domain[3]} fields"
    key = f"{program}@{domain[0]}x{domain[1]}x{domain[2]}"
    if _TABLE.exists():
        tab = json.loads(_TABLE.read_text())
        if key in tab:
            return int(tab[key]["first_touch_bytes"]), "first-touch (brute force)"
    return int(compulsory_bytes(program, tuple(domain))), "box model (upper bound)"


def movement_bytes(program: str, domain) -> dict | None:
    """The reference's per-node movement model of one launch (the paper's
    method: ``trace_movement(lower(program))``, reference
    ir/movement.py:64-74), committed in ``traffic_table.json`` by
    tools/traffic_table.py: all containers (every stencil node an unfused
    kernel) and the non-transient ones.  None when not tabulated."""
    if not _TABLE.exists() or len(domain) != 3:
        return None
    row = json.loads(_TABLE.read_text()).get(f"{program}@{domain[0]}x{domain[1]}x{domain[2]}", {})
    if "movement_model_bytes" not in row:
        return None
    return {"all_containers": int(row["movement_model_bytes"]),
            "non_transient": int(row["movement_model_nontransient_bytes"])}


@dataclass
class KernelBound:
    kernel: str
    unique_bytes: int
    bound_time: float
    measured_time: float | None = None
    invocations: int = 0
    total_time: float = 0.0
    source: str = ""

    @property
    def utilization(self) -> float | None:
        if not self.measured_time:
            return None
        return self.bound_time / self.measured_time

    @property
    def flags(self) -> list[str]:
        out = []
        if self.measured_time is None:
            out.append("unmeasured")
        elif self.utilization > 1.05:
            out.append("model-violation(cache-resident?)")
        return out


@dataclass
class PerfReport:
    entries: list[KernelBound]
    ranking: list[str] = field(default_factory=list)
    machine_bandwidth: float = 0.0


def model_kernel(program: str, domain, bandwidth: float) -> KernelBound:
    """Bound of one launch: unique bytes / bandwidth (bytes/s)."""
    if bandwidth <= 0:
        raise ValueError("bandwidth must be positive")
    b, src = unique_bytes(program, domain)
    return KernelBound(program, b, b / bandwidth, source=src)


def build_report(timings: dict[str, list[float]], domains: dict[str, tuple], bandwidth: float) -> PerfReport:
    """``timings``: kernel -> per-invocation seconds (all reps); ``domains``:
    kernel -> program domain of the launch (kernel = program name)."""
    import statistics

    entries = []
    for kern, dom in domains.items():
        kb = model_kernel(kern, dom, bandwidth)
        ts = timings.get(kern)
        if ts:
            kb.measured_time = statistics.median(ts)
            kb.invocations = len(ts)
            kb.total_time = sum(ts)
        entries.append(kb)
    ranking = [e.kernel for e in sorted(entries, key=lambda e: -e.total_time)]
    return PerfReport(entries, ranking, bandwidth)


def hotspot_list(report: PerfReport, top_n: int = 5) -> list[str]:
    def score(e):
        u = e.utilization
        return e.total_time * (1.0 - min(u, 1.0)) if u is not None else float("inf")

    return [e.kernel for e in sorted(report.entries, key=score, reverse=True)][:top_n]


def report_to_csv(report: PerfReport, reps: int = 1) -> str:
    lines = ["kernel,invocations,measured_s,bound_s,utilization,flags"]
    by = {e.kernel: e for e in report.entries}
    for k in report.ranking:
        e = by[k]
        m = f"{e.measured_time:.9e}" if e.measured_time else ""
        u = f"{e.utilization:.4f}" if e.utilization is not None else ""
        lines.append(f"{k},{e.invocations // max(reps, 1)},{m},{e.bound_time:.9e},{u},{'|'.join(e.flags)}")
    return "\n".join(lines) + "\n"
