"""Regenerate ``programs/*.stn`` from the templates and write the manifests.

Runs in the build container only (it imports the reference front end through
``tests/_ref.py``).  For every program it:

1. parses the ``.stn`` with the reference ``parse_program`` (``parser.py:696``)
   and requires ``validate(program) == []`` (``validate.py:221``);
2. records the reference's own allocation contract from
   ``compute_requirements`` (``extents.py:108-188``): per-field extents,
   temporary extensions and the minimum domain;
3. stores the canonical AST (``program.canonicalize``) and its structural
   fingerprint, which the B200 engine uses to select the kernel plan.

Usage: ``python tools/gen_programs.py``
"""

from __future__ import annotations

import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import _ref  # noqa: E402

from paper_2205_04148_b200.program import canonicalize, fingerprint, resolve_trace  # noqa: E402
from paper_2205_04148_b200.programs import templates  # noqa: E402


def manifest(name: str, text: str, ref) -> dict:
    prog = ref.parse_program(text)
    diags = ref.validate(prog)
    if diags:
        raise SystemExit(f"{name}: validation failed:\n" + "\n".join(d.format(name) for d in diags))
    req = ref.compute_requirements(prog)
    canon = canonicalize(prog)
    trace_ref = [(inv.stencil, dict(inv.kwargs)) for inv in ref.resolve_driver(prog)]
    assert resolve_trace(canon) == trace_ref, "driver restatement disagrees with resolve_driver"
    nk_min = req.min_nk
    return {
        "name": name,
        "fingerprint": fingerprint(canon),
        "program": canon,
        "requirements": {
            "extent": {n: [list(e.i), list(e.j), list(e.k)] for n, e in req.extent.items()},
            "extension": {n: {a: list(v) for a, v in d.items()} for n, d in req.extension.items()},
            "min_domain": [req.min_ni, req.min_nj, nk_min],
        },
        "trace": trace_ref,
    }


def main() -> None:
    ref = _ref.load()
    paths = templates.write_all()
    for p in paths:
        doc = manifest(p.stem, p.read_text(), ref)
        out = p.with_suffix(".json")
        out.write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
        n_stmt = sum(len(b["statements"]) for s in doc["program"]["stencils"] for b in s["blocks"])
        print(f"{p.stem:16s} fp={doc['fingerprint']} statements={n_stmt} min_domain={doc['requirements']['min_domain']}")


if __name__ == "__main__":
    main()
