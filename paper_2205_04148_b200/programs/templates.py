"""Python templates that emit the FV3 programs in the reference ``.stn`` DSL.

The reference language has no functions, field parameters or loops over
fields (``parser.py:1-23``), and FV3 repeats the same
finite-volume motifs in x and y and for many fields.  These
helpers emit the repeated statement groups; ``write_all()`` regenerates every
``programs/*.stn`` file.  The ``.stn`` text is the specification: the CPU
oracle executes it and the CUDA kernels in ``csrc/`` restate it statement by
statement.

Grid staggering (FV3 naming, cell (i, j) centred at (i, j)):
  u, vc, dx, dyc, rdx, rdyc  at south edges   (i,     j-1/2)
  v, uc, dy, dxc, rdy, rdxc  at west edges    (i-1/2, j    )
  area, rarea, f0, rdxa, rdya at centres      (i,     j    )
  area_c, rarea_c, fc, divg  at corners       (i-1/2, j-1/2)

Arithmetic rules for kernel authors (Appendix A): every statement is left
associative ``+ - * /``; no ``**`` (glibc ``pow`` is not correctly rounded);
``log``/``exp`` only in the vertical solver (oracle extension, tests/_ref.py).
"""

from __future__ import annotations

from pathlib import Path

HERE = Path(__file__).resolve().parent

# PPM edge interpolation weights 7/12 and -1/12 (Colella & Woodward 1984)
PPM_P1 = repr(7.0 / 12.0)
PPM_P2 = repr(-1.0 / 12.0)
# 4th-order D->A / A->C interpolation weights 9/16 and -1/16 (d2a2c_vect)
A1 = repr(9.0 / 16.0)
A2 = repr(-1.0 / 16.0)

COMMON_CONSTS = [
    ("ppm_p1", PPM_P1),
    ("ppm_p2", PPM_P2),
]


def _off(axis: str, d: int) -> str:
    return f"[{d}, 0, 0]" if axis == "x" else f"[0, {d}, 0]"


def ppm_flux(axis: str, q: str, c: str, out: str, tag: str, q2d: bool = False) -> list[str]:
    """Upwind PPM face value of ``q`` at the low face of each cell along
    ``axis`` (FV3 xppm/yppm with the hord=5 smoothness switch).

    ``out`` at index i (x) is the value on the face between cells i-1 and i,
    taken from the upwind cell chosen by the sign of Courant number ``c``.
    Temporaries are suffixed with ``tag`` so each instance has its own
    extension.
    """
    o = lambda d: _off(axis, d)  # noqa: E731
    al, bl, br, b0, sm = (f"al_{tag}", f"bl_{tag}", f"br_{tag}", f"b0_{tag}", f"sm_{tag}")
    return [
        f"{al} = ppm_p1 * ({q}{o(-1)} + {q}) + ppm_p2 * ({q}{o(-2)} + {q}{o(1)})",
        f"{bl} = {al} - {q}",
        f"{br} = {al}{o(1)} - {q}",
        f"{b0} = {bl} + {br}",
        f"{sm} = select(abs(3.0 * {b0}) < abs({bl} - {br}), 1.0, 0.0)",
        f"{out} = select({c} > 0.0, "
        f"{q}{o(-1)} + select({sm}{o(-1)} + {sm} > 0.0, (1.0 - {c}) * ({br}{o(-1)} - {c} * {b0}{o(-1)}), 0.0), "
        f"{q} + select({sm}{o(-1)} + {sm} > 0.0, (1.0 + {c}) * ({bl} + {c} * {b0}), 0.0))",
    ]


def fv_tp_2d(q: str, crx: str, cry: str, xfx: str, yfx: str, fx: str, fy: str, tag: str,
             mfx: str | None = None, mfy: str | None = None) -> list[str]:
    """FV3 ``fv_tp_2d``: 2-D transport fluxes of ``q`` with the inner
    (advective) updates in both directions (Lin & Rood 1996).

    Produces ``fx`` (west faces) and ``fy`` (south faces); they are area
    (``xfx``/``yfx``) or mass (``mfx``/``mfy``) weighted.
    """
    qi, qj = f"qi_{tag}", f"qj_{tag}"
    fx1, fx2, fy1, fy2 = f"fx1_{tag}", f"fx2_{tag}", f"fy1_{tag}", f"fy2_{tag}"
    wx = mfx or xfx
    wy = mfy or yfx
    lines = []
    lines += ppm_flux("y", q, cry, fy2, f"{tag}y0")
    lines.append(f"{qi} = ({q} * area + {fy2} * {yfx} - {fy2}[0, 1, 0] * {yfx}[0, 1, 0]) / "
                 f"(area + {yfx} - {yfx}[0, 1, 0])")
    lines += ppm_flux("x", qi, crx, fx1, f"{tag}x1")
    lines += ppm_flux("x", q, crx, fx2, f"{tag}x0")
    lines.append(f"{qj} = ({q} * area + {fx2} * {xfx} - {fx2}[1, 0, 0] * {xfx}[1, 0, 0]) / "
                 f"(area + {xfx} - {xfx}[1, 0, 0])")
    lines += ppm_flux("y", qj, cry, fy1, f"{tag}y1")
    lines.append(f"{fx} = 0.5 * ({fx1} + {fx2}) * {wx}")
    lines.append(f"{fy} = 0.5 * ({fy1} + {fy2}) * {wy}")
    return lines


def _block(policy: str, interval: str, lines: list[str], indent: int = 4) -> list[str]:
    pad = " " * indent
    out = [f"{pad}with computation({policy}), interval({interval}):"]
    out += [f"{pad}    {ln}" if not ln.startswith("@") else f"{pad}    {ln[1:]}" for ln in lines]
    return out


def _region(spec: str, lines: list[str]) -> list[str]:
    """Region block inside a computation body (lines get one more indent)."""
    return [f"@with horizontal(region[{spec}]):"] + [f"@    {ln}" for ln in lines]


def _fields(decls: list[tuple[str, str, bool]]) -> list[str]:
    out = []
    for name, dims, temp in decls:
        out.append(f"field {name} : float64 [{dims}]" + (" temporary" if temp else ""))
    return out


def _consts(pairs) -> list[str]:
    return [f"const {n} = {v}" for n, v in pairs]


def _collect_temps(lines: list[str], known: set[str]) -> list[str]:
    temps = []
    for ln in lines:
        body = ln.lstrip("@").strip()
        if body.startswith("with ") or "=" not in body:
            continue
        tgt = body.split("=", 1)[0].strip()
        if tgt not in known and tgt not in temps:
            temps.append(tgt)
    return temps


IJK, IJ, K = "I, J, K", "I, J", "K"


def program_text(consts, fields, stencils, driver) -> str:
    """Assemble a program; temporaries not declared in ``fields`` are
    declared automatically as 3-D temporaries."""
    known = {f[0] for f in fields}
    all_lines = [ln for _, _, blocks in stencils for _, _, body in blocks for ln in body]
    temps = _collect_temps(all_lines, known)
    out = _consts(consts) + [""] + _fields(fields + [(t, IJK, True) for t in temps]) + [""]
    for name, params, blocks in stencils:
        head = f"stencil {name}" + (f" uses ({', '.join(params)})" if params else "") + ":"
        out.append(head)
        for policy, interval, body in blocks:
            out += _block(policy, interval, body)
        out.append("")
    out.append("driver:")
    out += [f"    {d}" for d in driver]
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------------------
# K0: copy stencil (bandwidth ceiling)
# ---------------------------------------------------------------------------


def copy_program() -> str:
    return program_text(
        [],
        [("inp", IJK, False), ("out", IJK, False)],
        [("copy_field", [], [("PARALLEL", "...", ["out = inp"])])],
        ["copy_field()"],
    )


# ---------------------------------------------------------------------------
# K1: fv_tp_2d + flux-form update of one scalar (Table II "fv_tp_2d")
# ---------------------------------------------------------------------------


def fv_tp_2d_program() -> str:
    body = fv_tp_2d("q", "crx", "cry", "xfx", "yfx", "fx", "fy", "a")
    body.append("q = q + (fx - fx[1, 0, 0] + fy - fy[0, 1, 0]) * rarea")
    return program_text(
        COMMON_CONSTS,
        [("q", IJK, False), ("crx", IJK, False), ("cry", IJK, False), ("xfx", IJK, False),
         ("yfx", IJK, False), ("area", IJ, False), ("rarea", IJ, False)],
        [("fv_tp_2d", [], [("PARALLEL", "...", body)])],
        ["fv_tp_2d()"],
    )


# ---------------------------------------------------------------------------
# K7: tracer advection with accumulated Courant numbers and mass fluxes
# ---------------------------------------------------------------------------

NQ = 8


def tracer_2d_program(nq: int = NQ) -> str:
    stencils = [
        ("tracer_dp", [], [("PARALLEL", "...", [
            "dp2 = dp1 + (mfx - mfx[1, 0, 0] + mfy - mfy[0, 1, 0]) * rarea",
        ])]),
    ]
    for n in range(nq):
        body = fv_tp_2d(f"q{n}", "cx", "cy", "xfx", "yfx", "fx", "fy", "t", mfx="mfx", mfy="mfy")
        body.append(f"q{n} = (q{n} * dp1 + (fx - fx[1, 0, 0] + fy - fy[0, 1, 0]) * rarea) / dp2")
        stencils.append((f"tracer_q{n}", [], [("PARALLEL", "...", body)]))
    fields = [(f"q{n}", IJK, False) for n in range(nq)]
    fields += [("cx", IJK, False), ("cy", IJK, False), ("xfx", IJK, False), ("yfx", IJK, False),
               ("mfx", IJK, False), ("mfy", IJK, False), ("dp1", IJK, False),
               ("area", IJ, False), ("rarea", IJ, False)]
    driver = ["tracer_dp()"] + [f"tracer_q{n}()" for n in range(nq)]
    return program_text(COMMON_CONSTS, fields, stencils, driver)


def write_all() -> list[Path]:
    progs = {
        "copy": copy_program(),
        "fv_tp_2d": fv_tp_2d_program(),
        "tracer_2d": tracer_2d_program(),
    }
    paths = []
    for name, text in progs.items():
        p = HERE / f"{name}.stn"
        p.write_text(f"# generated by programs/templates.py ({name}); edit the template, not this file\n" + text)
        paths.append(p)
    return paths


if __name__ == "__main__":
    for p in write_all():
        print(p)
