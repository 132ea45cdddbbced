"""Import shim for the reference package (this container only).

``stencilkit.executor.__init__`` imports two modules that do not exist in the
reference tree (``executor/__init__.py:6-13``), so the package cannot be
imported as-is.  Pre-registering an empty ``stencilkit.executor`` package
whose ``__path__`` points at the real directory lets ``.reference`` load.

One documented oracle extension is installed: ``log`` and ``exp`` builtins
(FV3's ``riem_solver_c`` needs a logarithm; the reference DSL has only
``sqrt abs min max select``, ``frontend/ast.py:28``).  The parser shares the
``BUILTINS`` dict (``parser.py:31,261``) and ``_eval`` recurses through its
module-global name (``reference.py:202-258``), so wrapping the global is
enough.  ``log`` is the deterministic fdlibm-algorithm ``oracle.detmath.det_log``
(so host and device agree bitwise); ``exp`` is ``numpy.exp``.

The reference is located through ``$STENCILKIT_REF`` (default
``/root/reference/pkg/src``).  It is never present on the GPU host; callers
must treat :func:`available` as False there.
"""

from __future__ import annotations

import os
import pathlib
import sys
import types

REF = pathlib.Path(os.environ.get("STENCILKIT_REF", "/root/reference/pkg/src"))

_loaded = None


def available() -> bool:
    return (REF / "stencilkit" / "executor" / "reference.py").exists()


def load():
    """Return a namespace with the reference entry points (shimmed)."""
    global _loaded
    if _loaded is not None:
        return _loaded
    if not available():
        raise ImportError(f"reference package not found under {REF}")
    import numpy as np

    from oracle.detmath import det_log

    if str(REF) not in sys.path:
        sys.path.insert(0, str(REF))
    import stencilkit  # noqa: F401

    if "stencilkit.executor" not in sys.modules:
        m = types.ModuleType("stencilkit.executor")
        m.__path__ = [str(REF / "stencilkit" / "executor")]
        sys.modules["stencilkit.executor"] = m
    from stencilkit.frontend import ast as sk_ast
    from stencilkit.frontend import parse_program, validate
    from stencilkit.frontend.extents import compute_requirements
    from stencilkit.frontend.validate import resolve_driver
    from stencilkit.ir.graph import FULL_TILE, RankPlacement
    import stencilkit.executor.reference as sk_ref

    sk_ast.BUILTINS.setdefault("log", 1)
    sk_ast.BUILTINS.setdefault("exp", 1)
    if not getattr(sk_ref, "_fv3b_ext", False):
        base_eval = sk_ref._eval

        def _eval_ext(expr, ctx, ranges, k, scalars, record):
            if isinstance(expr, sk_ast.Call) and expr.func in ("log", "exp"):
                arg = _eval_ext(expr.args[0], ctx, ranges, k, scalars, record)
                if expr.func == "log":
                    return det_log(arg)
                with np.errstate(all="ignore"):
                    return np.exp(arg)
            return base_eval(expr, ctx, ranges, k, scalars, record)

        sk_ref._eval = _eval_ext
        sk_ref._fv3b_ext = True

    _loaded = types.SimpleNamespace(
        parse_program=parse_program,
        validate=validate,
        compute_requirements=compute_requirements,
        resolve_driver=resolve_driver,
        run_reference=sk_ref.run_reference,
        AccessRecorder=sk_ref.AccessRecorder,
        RankPlacement=RankPlacement,
        FULL_TILE=FULL_TILE,
        ast=sk_ast,
    )
    return _loaded
