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


def delnflux(q: str, tag: str, nord: int, damp: str, mass: str | None = None,
             damp2: str | None = None) -> tuple[list[str], str, str]:
    """FV3 ``deln_flux``: the del-(2 nord + 2) diffusive fluxes of ``q``
    (nord = 0: del2, 1: del4, 2: del6), to be added to a transport flux.

    ``d2`` starts as ``damp * q`` (or ``q`` when the fluxes are mass
    weighted); each order takes the flux-form divergence (``rarea``) of the
    previous face fluxes ``del6_v * (d2[-1] - d2)`` / ``del6_u * ...`` and
    flips the difference, so the operator stays diffusive.  Returns the
    statements and the (x, y) increments: ``dfx`` / ``dfy`` of the last
    order, times ``damp2 * (mass[-1] + mass)`` when mass weighted.  Each
    order has its own temporaries (minimal extensions, extents.py:128-164).
    Grid copy of corner halos at cube vertices (FV3 copy_corners) is not
    applied.
    """
    lines = []
    d2 = q if mass is not None else f"d2_{tag}0"
    if mass is None:
        lines.append(f"{d2} = {damp} * {q}")
    fx2, fy2 = f"dfx_{tag}0", f"dfy_{tag}0"
    lines.append(f"{fx2} = del6_v * ({d2}[-1, 0, 0] - {d2})")
    lines.append(f"{fy2} = del6_u * ({d2}[0, -1, 0] - {d2})")
    for n in range(1, nord + 1):
        d2 = f"d2_{tag}{n}"
        lines.append(f"{d2} = ({fx2} - {fx2}[1, 0, 0] + {fy2} - {fy2}[0, 1, 0]) * rarea")
        fx2, fy2 = f"dfx_{tag}{n}", f"dfy_{tag}{n}"
        lines.append(f"{fx2} = del6_v * ({d2} - {d2}[-1, 0, 0])")
        lines.append(f"{fy2} = del6_u * ({d2} - {d2}[0, -1, 0])")
    if mass is None:
        return lines, fx2, fy2
    return lines, f"{damp2} * ({mass}[-1, 0, 0] + {mass}) * {fx2}", f"{damp2} * ({mass}[0, -1, 0] + {mass}) * {fy2}"


def deln_coefficient(c: float, da_min: float, nord: int) -> float:
    """FV3's damping coefficient (c * da_min) ** (nord + 1), as repeated
    products (no pow; the value is a program constant and a kernel scalar)."""
    x = c * da_min
    d = x
    for _ in range(nord):
        d = d * x
    return d


def fv_tp_2d(q: str, crx: str, cry: str, xfx: str, yfx: str, fx: str, fy: str, tag: str,
             mfx: str | None = None, mfy: str | None = None,
             damp: tuple[str, str] | None = None) -> list[str]:
    """FV3 ``fv_tp_2d``: 2-D transport fluxes of ``q`` with the inner
    (advective) updates in both directions (Lin & Rood 1996).

    Produces ``fx`` (west faces) and ``fy`` (south faces); they are area
    (``xfx``/``yfx``) or mass (``mfx``/``mfy``) weighted.  ``damp``: the
    (x, y) flux increments of a ``delnflux`` chain, added in the same
    statement (fv_tp_2d's nord / damp_c arguments).
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
    dx_, dy_ = (f" + {damp[0]}", f" + {damp[1]}") if damp else ("", "")
    lines.append(f"{fx} = 0.5 * ({fx1} + {fx2}) * {wx}{dx_}")
    lines.append(f"{fy} = 0.5 * ({fy1} + {fy2}) * {wy}{dy_}")
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


# ---------------------------------------------------------------------------
# K4: riem_solver_c — semi-implicit vertical acoustic solve (SIM1 type),
# PAPER.md:595-603.  Program domain nk+1 (interfaces); layer statements use
# interval(0, -1) (the DSL cannot write level nk of an nk domain,
# validate.py:266-276).
# ---------------------------------------------------------------------------

RIEM_CONSTS = [
    ("ptop", "300.0"),
    ("rdgas", "287.05"),
    ("grav", "9.80665"),
    ("gama", "1.4"),          # 1 / (1 - kappa)
    ("p_fac", "0.05"),
]


def riem_stencils(dm: str, pt: str, w: str, gz_in: str, ws: str, pef: str, gz_out: str,
                  dt: str = "dt", sfx: str = "") -> list:
    """The riem_solver_c stencil sequence (7 stencils; the paper's version
    is 3 GT4Py stencils / 22 kernels).  ``gz_out`` may equal ``gz_in``;
    ``sfx`` suffixes temporaries and stencil names."""
    T = lambda n: f"{n}{sfx}"  # noqa: E731
    pem, dz, pm, pe, grat, bb, dd = T("pem"), T("dzc"), T("pmc"), T("pec"), T("grat"), T("bbc"), T("ddc")
    bet, gam, pp, aa, bw, gw, w2, pe2 = T("betp"), T("gamp"), T("ppc"), T("aac"), T("betw"), T("gamw"), T("w2c"), T("pe2c")
    t1g = f"gama * 2.0 * {dt} * {dt}"
    st = [
        (T("riem_pem"), [], [
            ("FORWARD", "0, 1", [f"{pem} = ptop"]),
            ("FORWARD", "1, None", [f"{pem} = {pem}[0, 0, -1] + {dm}[0, 0, -1]"]),
        ]),
        (T("riem_layer"), [], [
            ("PARALLEL", "0, -1", [
                f"{dz} = ({gz_in}[0, 0, 1] - {gz_in}) / grav",
                f"{pm} = {dm} / log({pem}[0, 0, 1] / {pem})",
                f"{pe} = {dm} * rdgas * {pt} / ({gz_in} - {gz_in}[0, 0, 1]) - {pm}",
            ]),
        ]),
        (T("riem_coef"), [], [
            ("PARALLEL", "0, -2", [
                f"{grat} = {dm} / {dm}[0, 0, 1]",
                f"{bb} = 2.0 * (1.0 + {grat})",
                f"{dd} = 3.0 * ({pe} + {grat} * {pe}[0, 0, 1])",
            ]),
            ("PARALLEL", "-2, -1", [
                f"{bb} = 2.0",
                f"{dd} = 3.0 * {pe}",
            ]),
        ]),
        (T("riem_pp_fwd"), [], [
            ("FORWARD", "0, 1", [f"{bet} = {bb}", f"{pp} = 0.0"]),
            ("FORWARD", "1, 2", [
                f"{pp} = {dd}[0, 0, -1] / {bet}[0, 0, -1]",
                f"{gam} = {grat}[0, 0, -1] / {bet}[0, 0, -1]",
                f"{bet} = {bb} - {gam}",
            ]),
            ("FORWARD", "2, -1", [
                f"{pp} = ({dd}[0, 0, -1] - {pp}[0, 0, -1]) / {bet}[0, 0, -1]",
                f"{gam} = {grat}[0, 0, -1] / {bet}[0, 0, -1]",
                f"{bet} = {bb} - {gam}",
            ]),
            ("FORWARD", "-1, None", [f"{pp} = ({dd}[0, 0, -1] - {pp}[0, 0, -1]) / {bet}[0, 0, -1]"]),
        ]),
        (T("riem_pp_bwd"), [], [
            ("BACKWARD", "1, -1", [f"{pp} = {pp} - {gam} * {pp}[0, 0, 1]"]),
        ]),
        (T("riem_w_fwd"), [], [
            ("PARALLEL", "1, -1", [f"{aa} = {t1g} / ({dz}[0, 0, -1] + {dz}) * ({pem} + {pp})"]),
            ("PARALLEL", "-1, None", [f"{aa} = {t1g} / {dz}[0, 0, -1] * ({pem} + {pp})"]),
        ]),
        (T("riem_w_sweep"), [], [
            ("FORWARD", "0, 1", [
                f"{bw} = {dm} - {aa}[0, 0, 1]",
                f"{w2} = ({dm} * {w} + {dt} * {pp}[0, 0, 1]) / {bw}",
            ]),
            ("FORWARD", "1, -2", [
                f"{gw} = {aa} / {bw}[0, 0, -1]",
                f"{bw} = {dm} - ({aa} + {aa}[0, 0, 1] + {aa} * {gw})",
                f"{w2} = ({dm} * {w} + {dt} * ({pp}[0, 0, 1] - {pp}) - {aa} * {w2}[0, 0, -1]) / {bw}",
            ]),
            ("FORWARD", "-2, -1", [
                f"{gw} = {aa} / {bw}[0, 0, -1]",
                f"{bw} = {dm} - ({aa} + {aa}[0, 0, 1] + {aa} * {gw})",
                f"{w2} = ({dm} * {w} + {dt} * ({pp}[0, 0, 1] - {pp}) - {aa}[0, 0, 1] * {ws} - {aa} * {w2}[0, 0, -1]) / {bw}",
            ]),
        ]),
        (T("riem_w_back"), [], [
            ("BACKWARD", "0, -2", [f"{w2} = {w2} - {gw}[0, 0, 1] * {w2}[0, 0, 1]"]),
        ]),
        (T("riem_pe"), [], [
            ("FORWARD", "0, 1", [f"{pe2} = 0.0"]),
            ("FORWARD", "1, None", [f"{pe2} = {pe2}[0, 0, -1] + {dm}[0, 0, -1] * ({w2}[0, 0, -1] - {w}[0, 0, -1]) / {dt}"]),
        ]),
        (T("riem_out"), [], [
            ("PARALLEL", "...", [f"{pef} = {pe2} + {pem}"]),
        ]),
    ]
    gz_lines = []
    if gz_out != gz_in:
        gz_lines.append(("BACKWARD", "-1, None", [f"{gz_out} = {gz_in}"]))
    gz_lines.append(("BACKWARD", "0, -1", [
        f"{gz_out} = {gz_out}[0, 0, 1] + {dm} * rdgas * {pt} / max(p_fac * {pm}, {pm} + 0.5 * ({pe2} + {pe2}[0, 0, 1]))",
    ]))
    st.append((T("riem_gz"), [], gz_lines))
    return st


def riem_solver_c_program() -> str:
    fields = [("dm", IJK, False), ("pt", IJK, False), ("w", IJK, False), ("gz", IJK, False),
              ("ws", IJ, False), ("pef", IJK, False)]
    stencils = riem_stencils("dm", "pt", "w", "gz", "ws", "pef", "gz")
    return program_text(RIEM_CONSTS + [("dt", "7.5")], fields, stencils, [f"{s[0]}()" for s in stencils])


# ---------------------------------------------------------------------------
# K5: remap_profile — PPM sub-grid profile for vertical remapping
# (cs_profile-type edge solve + Colella-Woodward monotonicity).
# Program domain nk+1: edge values live on interfaces.
# ---------------------------------------------------------------------------


def remap_stencils(q: str, delp: str, a2: str, a3: str, a4: str, sfx: str = "") -> list:
    T = lambda n: f"{n}{sfx}"  # noqa: E731
    grat, bet, gam, qe, d4, abot = T("grat_r"), T("bet_r"), T("gam_r"), T("qe_r"), T("d4_r"), T("abot_r")
    al, ar, ext, da1, a6, a6da, da2 = T("al_r"), T("ar_r"), T("ext_r"), T("da1_r"), T("a6_r"), T("a6da_r"), T("da2_r")
    return [
        (T("remap_edge_fwd"), [], [
            ("FORWARD", "0, 1", [
                f"{grat} = {delp}[0, 0, 1] / {delp}",
                f"{bet} = {grat} * ({grat} + 0.5)",
                f"{qe} = (({grat} + {grat}) * ({grat} + 1.0) * {q} + {q}[0, 0, 1]) / {bet}",
                f"{gam} = (1.0 + {grat} * ({grat} + 1.5)) / {bet}",
            ]),
            ("FORWARD", "1, -1", [
                f"{d4} = {delp}[0, 0, -1] / {delp}",
                f"{bet} = 2.0 + {d4} + {d4} - {gam}[0, 0, -1]",
                f"{qe} = (3.0 * ({q}[0, 0, -1] + {d4} * {q}) - {qe}[0, 0, -1]) / {bet}",
                f"{gam} = {d4} / {bet}",
            ]),
            ("FORWARD", "-1, None", [
                f"{abot} = 1.0 + {d4}[0, 0, -1] * ({d4}[0, 0, -1] + 1.5)",
                f"{qe} = (2.0 * {d4}[0, 0, -1] * ({d4}[0, 0, -1] + 1.0) * {q}[0, 0, -1] + {q}[0, 0, -2] - {abot} * {qe}[0, 0, -1]) / "
                f"({d4}[0, 0, -1] * ({d4}[0, 0, -1] + 0.5) - {abot} * {gam}[0, 0, -1])",
            ]),
        ]),
        (T("remap_edge_bwd"), [], [
            ("BACKWARD", "0, -1", [f"{qe} = {qe} - {gam} * {qe}[0, 0, 1]"]),
        ]),
        (T("remap_a4"), [], [
            ("PARALLEL", "0, -1", [
                f"{al} = {qe}",
                f"{ar} = {qe}[0, 0, 1]",
                f"{ext} = ({ar} - {q}) * ({q} - {al})",
                f"{da1} = {ar} - {al}",
                f"{a6} = 3.0 * (2.0 * {q} - ({al} + {ar}))",
                f"{a6da} = {a6} * {da1}",
                f"{da2} = {da1} * {da1}",
                f"{a2} = select({ext} <= 0.0, {q}, select({a6da} > {da2}, 3.0 * {q} - 2.0 * {ar}, {al}))",
                f"{a3} = select({ext} <= 0.0, {q}, select({a6da} < -{da2}, 3.0 * {q} - 2.0 * {al}, {ar}))",
                f"{a4} = 3.0 * (2.0 * {q} - ({a2} + {a3}))",
            ]),
        ]),
    ]


def remap_profile_program() -> str:
    fields = [("q", IJK, False), ("delp", IJK, False), ("a4_2", IJK, False), ("a4_3", IJK, False),
              ("a4_4", IJK, False)]
    st = remap_stencils("q", "delp", "a4_2", "a4_3", "a4_4")
    return program_text([], fields, st, [f"{s[0]}()" for s in st])


def remap_tracers_program(nq: int = NQ) -> str:
    fields = [("delp", IJK, False)]
    st = []
    for n in range(nq):
        fields += [(f"q{n}", IJK, False), (f"q{n}_a2", IJK, False), (f"q{n}_a3", IJK, False), (f"q{n}_a4", IJK, False)]
        st += remap_stencils(f"q{n}", "delp", f"q{n}_a2", f"q{n}_a3", f"q{n}_a4", sfx=f"_{n}")
    return program_text([], fields, st, [f"{s[0]}()" for s in st])


# ---------------------------------------------------------------------------
# K2: c_sw — C-grid half step (d2a2c winds, transportdelp, C-grid KE and
# vorticity, uc/vc update).  Orthogonal-metric form; the
# four tile-corner circulation fixes are regions that fire only on owned
# tile corners (cubed sphere).  ``layer`` is the interval of layer
# statements: "..." in an nk domain, "0, -1" in the nk+1 fused C-grid program.
# ---------------------------------------------------------------------------

C_METRICS = ["dx", "dy", "dxc", "dyc", "rdxc", "rdyc", "rarea", "rarea_c", "fc"]


def c_sw_stencils(layer: str, out_delpc: str, out_ptc: str, out_wc: str, uc: str, vc: str) -> list:
    return [
        ("c_sw_winds", [], [("PARALLEL", layer, [
            f"ua = {A2} * (u[0, -1, 0] + u[0, 2, 0]) + {A1} * (u + u[0, 1, 0])",
            f"va = {A2} * (v[-1, 0, 0] + v[2, 0, 0]) + {A1} * (v + v[1, 0, 0])",
            f"uct = {A2} * (ua[-2, 0, 0] + ua[1, 0, 0]) + {A1} * (ua[-1, 0, 0] + ua)",
            f"vct = {A2} * (va[0, -2, 0] + va[0, 1, 0]) + {A1} * (va[0, -1, 0] + va)",
        ])]),
        ("c_sw_transport", [], [("PARALLEL", layer, [
            "utc = dt2 * uct * dy",
            "vtc = dt2 * vct * dx",
            "fxc = utc * select(utc > 0.0, delp[-1, 0, 0], delp)",
            "fyc = vtc * select(vtc > 0.0, delp[0, -1, 0], delp)",
            "fxp = fxc * select(utc > 0.0, pt[-1, 0, 0], pt)",
            "fyp = fyc * select(vtc > 0.0, pt[0, -1, 0], pt)",
            "fxw = fxc * select(utc > 0.0, w[-1, 0, 0], w)",
            "fyw = fyc * select(vtc > 0.0, w[0, -1, 0], w)",
            f"{out_delpc} = delp + (fxc - fxc[1, 0, 0] + fyc - fyc[0, 1, 0]) * rarea",
            f"{out_ptc} = (pt * delp + (fxp - fxp[1, 0, 0] + fyp - fyp[0, 1, 0]) * rarea) / {out_delpc}",
            f"{out_wc} = (w * delp + (fxw - fxw[1, 0, 0] + fyw - fyw[0, 1, 0]) * rarea) / {out_delpc}",
        ])]),
        ("c_sw_ke_vort", [], [("PARALLEL", layer, [
            "keu = select(ua > 0.0, uct, uct[1, 0, 0])",
            "kev = select(va > 0.0, vct, vct[0, 1, 0])",
            "kec = 0.5 * dt2 * (ua * keu + va * kev)",
            "vortc = fc + rarea_c * (uct[0, -1, 0] * dxc[0, -1] - uct * dxc + vct * dyc - vct[-1, 0, 0] * dyc[-1, 0])",
            *_region("i_start, j_start", ["vortc = fc + rarea_c * (vct * dyc - uct * dxc - vct[-1, 0, 0] * dyc[-1, 0])"]),
            *_region("i_end, j_start", ["vortc = fc + rarea_c * (uct[0, -1, 0] * dxc[0, -1] - uct * dxc - vct[-1, 0, 0] * dyc[-1, 0])"]),
            *_region("i_end, j_end", ["vortc = fc + rarea_c * (uct[0, -1, 0] * dxc[0, -1] + vct * dyc - vct[-1, 0, 0] * dyc[-1, 0])"]),
            *_region("i_start, j_end", ["vortc = fc + rarea_c * (uct[0, -1, 0] * dxc[0, -1] - uct * dxc + vct * dyc)"]),
        ])]),
        ("c_sw_update", [], [("PARALLEL", layer, [
            "fy1c = dt2 * v",
            f"{uc} = uct + fy1c * select(fy1c > 0.0, vortc, vortc[0, 1, 0]) + rdxc * (kec[-1, 0, 0] - kec)",
            "fx1c = dt2 * u",
            f"{vc} = vct - fx1c * select(fx1c > 0.0, vortc, vortc[1, 0, 0]) + rdyc * (kec[0, -1, 0] - kec)",
        ])]),
    ]


def c_sw_program() -> str:
    fields = [(n, IJK, False) for n in ("u", "v", "delp", "pt", "w", "uc", "vc", "delpc", "ptc", "wc")]
    fields += [(m, IJ, False) for m in C_METRICS]
    st = c_sw_stencils("...", "delpc", "ptc", "wc", "uc", "vc")
    return program_text([("dt2", "7.5")], fields, st, [f"{x[0]}()" for x in st])


def c_grid_program() -> str:
    """c_sw + riem_solver_c + p_grad_c fused in one nk+1 program, so the
    C-grid thickness/temperature/w and the solver's pressure/geopotential
    are temporaries (extended one cell where p_grad_c needs them) and no
    halo exchange is needed between them (FV3 computes them on the
    extended domain for the same reason)."""
    fields = [(n, IJK, False) for n in ("u", "v", "delp", "pt", "w", "gz", "uc", "vc")]
    fields += [(m, IJ, False) for m in C_METRICS] + [("ws", IJ, False)]
    st = c_sw_stencils("0, -1", "delpcc", "ptcc", "wcc", "uc", "vc")
    st += riem_stencils("delpcc", "ptcc", "wcc", "gz", "ws", "pkc", "gzc", dt="dt2", sfx="_c")
    st.append(("p_grad_c", [], [("PARALLEL", "0, -1", [
        "wkc = pkc[0, 0, 1] - pkc",
        "uc = uc + dt2 * rdxc / (wkc[-1, 0, 0] + wkc) * ((gzc[-1, 0, 1] - gzc) * (pkc[0, 0, 1] - pkc[-1, 0, 0]) + "
        "(gzc[-1, 0, 0] - gzc[0, 0, 1]) * (pkc[-1, 0, 1] - pkc))",
        "vc = vc + dt2 * rdyc / (wkc[0, -1, 0] + wkc) * ((gzc[0, -1, 1] - gzc) * (pkc[0, 0, 1] - pkc[0, -1, 0]) + "
        "(gzc[0, -1, 0] - gzc[0, 0, 1]) * (pkc[0, -1, 1] - pkc))",
    ])]))
    return program_text(RIEM_CONSTS + [("dt2", "7.5")], fields, st, [f"{x[0]}()" for x in st])


# ---------------------------------------------------------------------------
# K3: d_sw — D-grid Lagrangian step: Courant numbers from the C-grid winds,
# fv_tp_2d of delp (mass fluxes) / pt / w (mass weighted), vorticity and
# kinetic energy, vorticity transport, Smagorinsky-scaled divergence
# damping (the paper's Smagorinsky listing with sqrt instead of **,
# PAPER.md:532-537), del6 flux damping (FV3 delnflux) of delp, pt, w and the
# vorticity, u/v update, and the tracer-flux accumulators.
# ---------------------------------------------------------------------------

D_METRICS = ["dx", "dy", "dxc", "dyc", "rdx", "rdy", "rdxa", "rdya", "area", "rarea", "rarea_c", "f0",
             "del6_u", "del6_v"]
# flux damping (FV3 d_sw / fv_tp_2d nord, damp_c): del6 (nord = 2) on the
# delp, pt and w fluxes (d4_bg) and on the vorticity flux (vtdm4)
NORD = 2
D4_BG, VTDM4, DA_MIN = 0.12, 0.05, 1.0e8
DAMP4 = deln_coefficient(D4_BG, DA_MIN, NORD)
DAMPV = deln_coefficient(VTDM4, DA_MIN, NORD)
D_CONSTS = [("dt", "15.0"), ("dddmp", "0.2"), ("d2_bg", "0.0"), ("da_min", repr(DA_MIN)),
            ("damp4", repr(DAMP4)), ("damp4h", repr(0.5 * DAMP4)), ("dampv", repr(DAMPV))]


def d_sw_stencils() -> list:
    courant = [
        "xfx = dt * uc * dy",
        "crx = select(uc > 0.0, dt * uc * rdxa[-1, 0], dt * uc * rdxa)",
        "yfx = dt * vc * dx",
        "cry = select(vc > 0.0, dt * vc * rdya[0, -1], dt * vc * rdya)",
    ]
    dmass, dmx, dmy = delnflux("delp", "d", NORD, "damp4")
    mass = dmass + fv_tp_2d("delp", "crx", "cry", "xfx", "yfx", "fxm", "fym", "d", damp=(dmx, dmy))
    mass += ["delpn = delp + (fxm - fxm[1, 0, 0] + fym - fym[0, 1, 0]) * rarea"]
    dheat, dpx, dpy = delnflux("pt", "p", NORD, "damp4", mass="delp", damp2="damp4h")
    heat = dheat + fv_tp_2d("pt", "crx", "cry", "xfx", "yfx", "gxp", "gyp", "p", mfx="fxm", mfy="fym",
                            damp=(dpx, dpy))
    dvert, dwx, dwy = delnflux("w", "w", NORD, "damp4", mass="delp", damp2="damp4h")
    vert = dvert + fv_tp_2d("w", "crx", "cry", "xfx", "yfx", "hxw", "hyw", "w", mfx="fxm", mfy="fym",
                            damp=(dwx, dwy))
    ke = [
        "ub = 0.5 * dt * (uc[0, -1, 0] + uc)",
        "cub = select(ub > 0.0, ub * rdx[-1, 0], ub * rdx)",
        *ppm_flux("x", "u", "cub", "uu", "ku"),
        "vb = 0.5 * dt * (vc[-1, 0, 0] + vc)",
        "cvb = select(vb > 0.0, vb * rdy[0, -1], vb * rdy)",
        *ppm_flux("y", "v", "cvb", "vv", "kv"),
        "ked = 0.5 * (ub * uu + vb * vv)",
    ]
    vort = ["wk = f0 + rarea * (u * dx - u[0, 1, 0] * dx[0, 1] + v[1, 0, 0] * dy[1, 0] - v * dy)"]
    dvort, dvx, dvy = delnflux("wk", "v", NORD, "dampv")
    vort += dvort + fv_tp_2d("wk", "crx", "cry", "xfx", "yfx", "fxv", "fyv", "v", damp=(dvx, dvy))
    damp = [
        "divg = rarea_c * (u * dyc - u[-1, 0, 0] * dyc[-1, 0] + v * dxc - v[0, -1, 0] * dxc[0, -1])",
        "tens = rarea_c * (u * dyc - u[-1, 0, 0] * dyc[-1, 0] - v * dxc + v[0, -1, 0] * dxc[0, -1])",
        "smag = dt * sqrt(divg * divg + tens * tens)",
        "dmp = da_min * max(d2_bg, min(0.2, dddmp * smag))",
        "ddv = dmp * divg",
    ]
    update = [
        "cx = cx + crx",
        "cy = cy + cry",
        "xfa = xfa + xfx",
        "yfa = yfa + yfx",
        "mfx = mfx + fxm",
        "mfy = mfy + fym",
        "pt = (pt * delp + (gxp - gxp[1, 0, 0] + gyp - gyp[0, 1, 0]) * rarea) / delpn",
        "w = (w * delp + (hxw - hxw[1, 0, 0] + hyw - hyw[0, 1, 0]) * rarea) / delpn",
        "delp = delpn",
        "u = (u * dx + ked - ked[1, 0, 0] + fyv) * rdx + (ddv[1, 0, 0] - ddv) * rdx",
        "v = (v * dy + ked - ked[0, 1, 0] - fxv) * rdy + (ddv[0, 1, 0] - ddv) * rdy",
    ]
    return [
        ("d_sw_courant", [], [("PARALLEL", "...", courant)]),
        ("d_sw_mass", [], [("PARALLEL", "...", mass)]),
        ("d_sw_heat", [], [("PARALLEL", "...", heat)]),
        ("d_sw_vert", [], [("PARALLEL", "...", vert)]),
        ("d_sw_ke", [], [("PARALLEL", "...", ke)]),
        ("d_sw_vort", [], [("PARALLEL", "...", vort)]),
        ("d_sw_damp", [], [("PARALLEL", "...", damp)]),
        ("d_sw_update", [], [("PARALLEL", "...", update)]),
    ]


D_STATE = ["u", "v", "w", "delp", "pt", "uc", "vc", "cx", "cy", "xfa", "yfa", "mfx", "mfy"]


def d_sw_program() -> str:
    fields = [(n, IJK, False) for n in D_STATE] + [(m, IJ, False) for m in D_METRICS]
    st = d_sw_stencils()
    return program_text(COMMON_CONSTS + D_CONSTS, fields, st, [f"{x[0]}()" for x in st])


# ---------------------------------------------------------------------------
# D-grid nonhydrostatic update (FV3 riem_solver3 + nh_p_grad): the column
# solve updates w, gz and the interface pressure; after a halo exchange of
# pef/gz the pressure-gradient force is applied to the D-grid winds with
# corner-averaged pressure and geopotential.  Both run in nk+1 domains.
# ---------------------------------------------------------------------------


def nh_d_program() -> str:
    fields = [("delp", IJK, False), ("pt", IJK, False), ("w", IJK, False), ("gz", IJK, False),
              ("ws", IJ, False), ("pef", IJK, False)]
    st = riem_stencils("delp", "pt", "w", "gz", "ws", "pef", "gz", dt="dt", sfx="_d")
    st.append(("nh_d_w", [], [("PARALLEL", "0, -1", ["w = w2c_d"])]))
    return program_text(RIEM_CONSTS + [("dt", "15.0")], fields, st, [f"{x[0]}()" for x in st])


def p_grad_d_program() -> str:
    fields = [("u", IJK, False), ("v", IJK, False), ("pef", IJK, False), ("gz", IJK, False),
              ("rdx", IJ, False), ("rdy", IJ, False)]
    body = [
        "pkd = 0.25 * (pef + pef[-1, 0, 0] + pef[0, -1, 0] + pef[-1, -1, 0])",
        "gzd = 0.25 * (gz + gz[-1, 0, 0] + gz[0, -1, 0] + gz[-1, -1, 0])",
    ]
    layer = [
        "wkd = pkd[0, 0, 1] - pkd",
        "u = u + dt * rdx / (wkd + wkd[1, 0, 0]) * ((gzd[0, 0, 1] - gzd[1, 0, 0]) * (pkd[1, 0, 1] - pkd) + "
        "(gzd - gzd[1, 0, 1]) * (pkd[0, 0, 1] - pkd[1, 0, 0]))",
        "v = v + dt * rdy / (wkd + wkd[0, 1, 0]) * ((gzd[0, 0, 1] - gzd[0, 1, 0]) * (pkd[0, 1, 1] - pkd) + "
        "(gzd - gzd[0, 1, 1]) * (pkd[0, 0, 1] - pkd[0, 1, 0]))",
    ]
    st = [("p_grad_d_corners", [], [("PARALLEL", "...", body)]),
          ("p_grad_d", [], [("PARALLEL", "0, -1", layer)])]
    return program_text([("dt", "15.0")], fields, st, [f"{x[0]}()" for x in st])


def programs() -> dict:
    """name -> .stn text of every shipped program."""
    return {
        "copy": copy_program(),
        "fv_tp_2d": fv_tp_2d_program(),
        "tracer_2d": tracer_2d_program(),
        "riem_solver_c": riem_solver_c_program(),
        "remap_profile": remap_profile_program(),
        "remap_tracers": remap_tracers_program(),
        "c_sw": c_sw_program(),
        "c_grid": c_grid_program(),
        "d_sw": d_sw_program(),
        "nh_d": nh_d_program(),
        "p_grad_d": p_grad_d_program(),
    }


def write_all() -> list[Path]:
    progs = programs()
    paths = []
    for name, text in progs.items():
        p = HERE / f"{name}.stn"
        p.write_text(f"# generated by programs/templates.py ({name}); edit the template, not this file\n" + text)
        paths.append(p)
    return paths


if __name__ == "__main__":
    for p in write_all():
        print(p)
