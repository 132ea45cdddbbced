"""The B200 dycore timestep: device-resident state, the shipped programs'
hand-written kernels in the step order of ``config.py``, halo updates on
device, and CUDA-graph replay of whole timesteps.

State lives in the uniform device Layout (``device.Grid``): every 3-D field
has ``nk + 1`` levels and a 4-cell I/J halo, so layer programs (domain nk)
and interface programs (domain nk + 1) address the same buffers.  Fields a
kernel reads at horizontal offsets and rewrites (u, v, w, delp, pt, tracers)
are ping-ponged between two buffers; pointwise accumulators and in-place
column outputs are updated in place.  The state is the interior (layer fields
on levels < nk, interface fields on all nk + 1 levels): the halos and the
unused top slot of a ping-pong layer field are scratch between halo updates.

The CPU counterpart is ``oracle/dycore.py`` (tests only); the two agree
bitwise (tests/test_gpu_dycore.py).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .config import DIAG_3D, METRICS_2D, STATE_3D, RunConfig
from .device import Grid, capture_guard

C_METRICS = ("dx", "dy", "dxc", "dyc", "rdxc", "rdyc", "rarea", "rarea_c", "fc")
D_METRICS = ("dx", "dy", "dxc", "dyc", "rdx", "rdy", "rdxa", "rdya", "area", "rarea", "rarea_c", "f0", "del6_u",
             "del6_v")
PINGPONG = ("u", "v", "w", "delp", "pt")
ACCUM = ("cx", "cy", "xfa", "yfa", "mfx", "mfy")


class PeriodicHalo:
    """Single-rank doubly periodic halo update (one launch per group)."""

    def __init__(self, dycore: "Dycore"):
        self.d = dycore

    def update(self, names: list[str]) -> None:
        d = self.d
        for i in range(0, len(names), 32):
            fields = [d.f(n) for n in names[i : i + 32]]
            d.launch("halo", "fv3b_halo_periodic", fields, [float(d.cfg.halo)], d.dom_layers)


class Dycore:
    def __init__(self, cfg: RunConfig, state: dict[str, np.ndarray] | None = None, device: str = "cuda",
                 placement=(False, False, False, False), halo=None, tuned: bool = True):
        """``tuned``: apply the launch configuration tools/tune.py recorded
        for this device and shape (tuning.json), process-wide."""
        self.cfg = cfg
        if tuned and device != "cpu" and torch.cuda.is_available():
            from . import tuning

            self.tuning = tuning.apply(torch.cuda.get_device_name(), (cfg.ni, cfg.nj, cfg.nk))
        self.device = device
        self.grid = Grid(cfg.ni, cfg.nj, cfg.nk, halo=cfg.halo)
        self.placement = placement
        self.dom_layers = self.grid.domain(placement, nk=cfg.nk)
        self.dom_ifaces = self.grid.domain(placement, nk=cfg.nk + 1)
        g = self.grid
        names3 = STATE_3D + DIAG_3D + cfg.tracer_names() + [f"{q}_{a}" for q in cfg.remapped() + ["u", "v"]
                                                  for a in ("a2", "a3", "a4")]
        self.cur: dict[str, torch.Tensor] = {n: g.new3(device) for n in names3}
        self.cur.update({n: g.new2(device) for n in METRICS_2D})
        self.alt: dict[str, torch.Tensor] = {n: g.new3(device) for n in list(PINGPONG) + ["gz"] + cfg.tracer_names()}
        self.scratch = {n: g.new3(device) for n in ("delpcc", "ptcc", "wcc", "pkc", "gzc", "riem_scr", "du", "dv",
                                                     "dlnp", "lnpe1", "lnpe2")}
        # target coordinate of the vertical remapping (pe2 = ak + bk * ps)
        ak, bk = cfg.target_coordinate()
        self.coord = {"ak": torch.from_numpy(ak).to(device), "bk": torch.from_numpy(bk).to(device)}
        self.halo = halo or PeriodicHalo(self)
        self.stream = None
        self.overlap = False  # halo exchanges on their own stream (step_overlapped)
        self.launches = 0
        self.timer = None
        self._graphs: dict[tuple, tuple] = {}
        if state is not None:
            self.load(state)

    # -- state transfer (reference array convention, uniform halo) ----------

    def load(self, state: dict[str, np.ndarray]) -> None:
        h = self.cfg.halo
        for n, t in self.cur.items():
            if n in state:
                a = state[n]
                self.grid.put(t, a, ("I", "J", "K")[: a.ndim], (h, h, 0)[: a.ndim])

    def download(self, names=None) -> dict[str, np.ndarray]:
        h = self.cfg.halo
        out = {}
        for n in names or self.cur:
            t = self.cur[n]
            dims = ("I", "J", "K") if t.dim() == 3 else ("I", "J")
            shape = (self.cfg.ni + 2 * h, self.cfg.nj + 2 * h, self.cfg.nk + 1)[: t.dim()]
            out[n] = self.grid.get(t, dims, (h, h, 0)[: t.dim()], shape)
        return out

    # -- host I/O through pinned buffers (the end-to-end path) ---------------

    def prognostic(self) -> list[str]:
        """Fields a timestep evolves (the state a host caller owns).  The
        order is step_host's transfer order: gz (downloaded early), the other
        dynamics fields, then the tracers (uploaded during the substeps)."""
        return ["gz", "u", "v", "w", "delp", "pt"] + self.cfg.tracer_names()

    def host_buffers(self, names=None) -> dict[str, torch.Tensor]:
        """Pinned host tensors in the reference array convention (I, J, K,
        halo-inclusive, C order) for ``names`` (default: the prognostic
        state), as consecutive views of one pinned block, so step_host moves
        each run of fields it transfers together as one copy."""
        names = list(names or self.prognostic())
        block = torch.zeros((len(names),) + self._host_shape(), dtype=torch.float64).pin_memory()
        return {n: block[t] for t, n in enumerate(names)}

    def _host_shape(self) -> tuple[int, int, int]:
        h, c = self.cfg.halo, self.cfg
        return (c.ni + 2 * h, c.nj + 2 * h, c.nk + 1)

    @staticmethod
    def _runs(names, a: dict, b: dict) -> list[tuple[torch.Tensor, torch.Tensor]]:
        """(a-view, b-view) pairs covering ``names`` in order, consecutive
        fields merged into one flat view wherever both sides are adjacent in
        one storage (one DMA instead of one per field)."""
        out = []
        for n in names:
            x, y = a[n], b[n]
            if out:
                px, py, pn = out[-1]
                if (x.untyped_storage().data_ptr() == px.untyped_storage().data_ptr()
                        and y.untyped_storage().data_ptr() == py.untyped_storage().data_ptr()
                        and x.is_contiguous() and y.is_contiguous()
                        and x.storage_offset() == px.storage_offset() + px.numel()
                        and y.storage_offset() == py.storage_offset() + py.numel()):
                    out[-1] = (torch.empty(0, dtype=x.dtype, device=x.device).set_(
                                   x.untyped_storage(), px.storage_offset(), (px.numel() + x.numel(),)),
                               torch.empty(0, dtype=y.dtype, device=y.device).set_(
                                   y.untyped_storage(), py.storage_offset(), (py.numel() + y.numel(),)),
                               pn + [n])
                    continue
            out.append((x.reshape(-1) if x.is_contiguous() else x, y.reshape(-1) if y.is_contiguous() else y, [n]))
        return [(x, y) for x, y, _ in out]

    def _staging(self) -> torch.Tensor:
        if getattr(self, "_stage", None) is None:
            h, c = self.cfg.halo, self.cfg
            self._stage = torch.empty((c.ni + 2 * h, c.nj + 2 * h, c.nk + 1), dtype=torch.float64,
                                      device=self.device)
        return self._stage

    def _window(self, t: torch.Tensor) -> torch.Tensor:
        g = self.grid
        a = g.i0 - self.cfg.halo
        return t[:, :, a : a + self.cfg.ni + 2 * self.cfg.halo].permute(2, 1, 0)

    def _transpose(self, src: torch.Tensor, dst: torch.Tensor) -> None:
        """Reference-convention (I, J, K) array <-> Layout window copy on the
        device (fv3b_transpose, current stream); both are (I, J, K) views."""
        fs = []
        for t in (src, dst):
            f = _lib.Field()
            f.data = t.data_ptr()
            f.stride[:] = list(t.stride())
            f.shape[:] = list(t.shape)
            f.halo_lo[:] = [0, 0, 0]
            f.rank = 3
            fs.append(f)
        d = _lib.Domain()
        d.ni, d.nj, d.nk = src.shape
        self.launch("transpose", "fv3b_transpose", fs, [], d)

    def load_host(self, host: dict[str, torch.Tensor]) -> None:
        """Enqueue host -> device copies (pinned, async) of ``host`` fields
        into the current state, then the layout transpose on the device."""
        st = self._staging()
        for n, src in host.items():
            st.copy_(src, non_blocking=True)
            self._transpose(st, self._window(self.cur[n]))

    def store_host(self, host: dict[str, torch.Tensor]) -> None:
        """Enqueue device -> host copies of the current state into ``host``."""
        st = self._staging()
        for n, dst in host.items():
            self._transpose(self._window(self.cur[n]), st)
            dst.copy_(st, non_blocking=True)

    def _io_stages(self, names) -> tuple[dict, dict, list]:
        """Device staging for step_host of the current call: input stage i
        (three-deep ring: a call's uploads never wait for the compute of the
        call before last), output stage o (two-deep), and the slots' free events."""
        if getattr(self, "_io", None) is None or set(self._io[0][0]) != set(names):
            shape = self._host_shape()

            def mk():  # one device block per stage, fields in transfer order (see _runs)
                block = torch.empty((len(names),) + shape, dtype=torch.float64, device=self.device)
                return {n: block[t] for t, n in enumerate(names)}

            self._io = ([mk() for _ in range(3)], [mk() for _ in range(2)])
            self._io_free = ([None] * 3, [None] * 2)  # inputs consumed / outputs downloaded
        return self._io

    def _io_streams(self) -> tuple[torch.cuda.Stream, torch.cuda.Stream]:
        if getattr(self, "_up", None) is None:
            self._up, self._down, self._xs = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
            self._io_calls, self._prev_out, self._prev_done, self._prev_x = 0, set(), None, None
            self._dl_events = {}  # host data_ptr -> the last call's download event of that buffer
        return self._up, self._down

    def _halo_refreshed(self) -> set[str]:
        """Fields whose every halo cell a step rewrites before reading one
        (periodic halo only): the dynamics fields of the first halo point and
        the tracers of the tracer point."""
        if not isinstance(self.halo, PeriodicHalo):
            return set()
        return {"u", "v", "w", "delp", "pt", "gz"} | set(self.cfg.tracer_names())

    def _interior_rows(self) -> tuple[int, int, int, int]:
        return interior_rows(self.cfg)

    def host_io_bytes(self, h_in: dict[str, torch.Tensor]) -> tuple[int, int]:
        """(uploaded, downloaded) bytes of one step_host call with these host
        buffers (the refreshed fields' halos are not uploaded)."""
        fresh = self._halo_refreshed()
        _, width, rows, _ = self._interior_rows()
        up = sum(width * rows if n in fresh else t.numel() * t.element_size() for n, t in h_in.items())
        return up, sum(t.numel() * t.element_size() for t in h_in.values())

    def step_host(self, h_in: dict[str, torch.Tensor], h_out: dict[str, torch.Tensor]) -> torch.cuda.Event:
        """One timestep from pinned host state ``h_in`` to pinned host state
        ``h_out`` (reference array convention, host_buffers()).  Returns an
        event that completes when ``h_out`` holds the result; the host buffers
        must stay untouched until then.

        Transfers run on an upload and a download stream (both PCIe
        directions at once) and overlap the compute they do not feed: the
        tracers' uploads run during the acoustic substeps (first needed by
        tracer_2d); gz is final after the substeps and downloads during
        tracer advection and remapping; everything the remapping rewrites
        (tracers, delp, pt, w, u, v) downloads at the end of the step.
        Device staging is a ring (three input stages, two output stages), so
        successive calls pipeline: the next call's uploads overlap this
        call's compute, this call's downloads the next call's compute.  A
        call whose inputs are the previous call's outputs (a chained
        integration) waits for those downloads before uploading.

        The layout transposes off the compute path run on a third stream:
        the tracers' (during the substeps), and every output's.  Inputs land
        in the other buffer of each ping-pong pair (cur / alt swapped first),
        so the previous call's output transposes, still reading the old
        buffers, overlap this call's start; the first program that writes a
        ping-pong buffer (d_sw) waits for them."""
        comp = torch.cuda.current_stream()
        up, down = self._io_streams()
        xs = self._xs
        tracers = set(self.cfg.tracer_names())
        trc = [n for n in h_in if n in tracers]           # uploaded during the substeps
        dyn = [n for n in h_in if n not in tracers]       # uploaded before the step
        late = [n for n in h_in if n in tracers or n in ("delp", "pt", "w", "u", "v")]  # rewritten by the remap
        early = [n for n in h_in if n not in late]
        stages = self._io_stages(list(h_in))
        si, so = self._io_calls % 3, self._io_calls % 2
        self._io_calls += 1
        sin, sout = stages[0][si], stages[1][so]
        in_free, out_free = self._io_free
        if in_free[si] is not None:  # consumed by the compute three calls ago
            up.wait_event(in_free[si])
        # a chained call (inputs are the last call's outputs) moves field by
        # field: each upload waits only for the download of its own buffer, so
        # the dynamics fields (downloaded first) travel back up while the
        # tracers are still coming down, and the compute starts before they land
        chained = self._prev_done is not None and bool(self._prev_out & {t.data_ptr() for t in h_in.values()})
        dl = self._dl_events
        # a periodic domain's first halo points (the substeps' start for the
        # dynamics fields, the tracer point for the tracers) rewrite every
        # halo cell of these fields before anything reads one: only their
        # interior columns travel up (one pitched copy per field, rows of
        # nj x (nk + 1) values)
        fresh = self._halo_refreshed()

        def upload(names):
            if not chained and not fresh & set(names):
                for dst, src in self._runs(names, sin, h_in):
                    dst.copy_(src, non_blocking=True)
                return
            for n in names:
                p = h_in[n].data_ptr()
                if chained and p in dl:
                    up.wait_event(dl[p])
                elif chained and p in self._prev_out:
                    up.wait_event(self._prev_done)
                if n in fresh:
                    off, width, rows, pitch = self._interior_rows()
                    _lib.memcpy2d(sin[n].data_ptr() + off, pitch, p + off, pitch, width, rows, up.cuda_stream)
                else:
                    sin[n].copy_(h_in[n], non_blocking=True)

        with torch.cuda.stream(up):
            upload(dyn)
            e_dyn = up.record_event()
            upload(trc)
            e_trc = up.record_event()
        # inputs into the other buffer of each pair (the previous outputs stay
        # readable); a field without a second buffer waits for the readers
        pairs = all(n in self.alt for n in h_in)
        if pairs:
            self.swap(*h_in)
        elif self._prev_x is not None:
            comp.wait_event(self._prev_x)
        comp.wait_event(e_dyn)
        for n in dyn:
            self._transpose(sin[n], self._window(self.cur[n]))
        start = comp.record_event()
        xs.wait_event(start)  # (the tracers' buffers are this call's from here on)
        xs.wait_event(e_trc)
        with torch.cuda.stream(xs):
            for n in trc:
                self._transpose(sin[n], self._window(self.cur[n]))
        e_xtrc = xs.record_event()
        if out_free[so] is not None:  # downloaded two calls ago
            xs.wait_event(out_free[so])

        new_dl = {}

        def out(names):  # device transpose on the transpose stream, download on the download stream
            if not names:
                return
            xs.wait_event(comp.record_event())
            # one merged download (pipelined calls: the fewest DMAs), or field
            # by field in a chained integration (see upload)
            e_out = None
            for group in ([[n] for n in names] if chained else [names]):
                with torch.cuda.stream(xs):
                    for n in group:
                        self._transpose(self._window(self.cur[n]), sout[n])
                e_out = xs.record_event()
                down.wait_event(e_out)
                with torch.cuda.stream(down):
                    for dst, src in self._runs(group, h_out, sout):
                        dst.copy_(src, non_blocking=True)
                e_dl = down.record_event()
                for n in group:
                    new_dl[h_out[n].data_ptr()] = e_dl
            return e_out

        tracer_point, consumed, point = set(self.cfg.tracer_names()), False, 0
        for names in self.phases():
            point += 1
            if point == 2 and self._prev_x is not None:  # before the first ping-pong write (d_sw)
                comp.wait_event(self._prev_x)
            if tracer_point & set(names):  # the tracer halo point: substeps done
                comp.wait_event(e_xtrc)
                in_free[si], consumed = comp.record_event(), True
                out(early)
            self.halo.update(names)
        if not consumed:  # no tracers in the run
            comp.wait_event(e_xtrc)
            in_free[si] = comp.record_event()
            out(early)
        e_late = out(late)
        # the next call may not overwrite what the output transposes read
        self._prev_x = e_late if e_late is not None else xs.record_event()
        done = down.record_event()
        out_free[so] = done
        self._prev_done, self._prev_out = done, {t.data_ptr() for t in h_out.values()}
        self._dl_events = new_dl
        return done

    # -- launch helpers -----------------------------------------------------

    def f(self, name: str) -> _lib.Field:
        return self.grid.abi(self.cur[name])

    def a(self, name: str) -> _lib.Field:
        return self.grid.abi(self.alt[name])

    def s(self, name: str) -> _lib.Field:
        return self.grid.abi(self.scratch[name])

    def swap(self, *names: str) -> None:
        for n in names:
            self.cur[n], self.alt[n] = self.alt[n], self.cur[n]

    def launch(self, node: str, entry: str, fields, scalars, dom) -> None:
        stream = torch.cuda.current_stream().cuda_stream
        if self.timer is not None:
            self.timer.start(node)
        _lib.call(entry, fields, scalars, dom, stream)
        if self.timer is not None:
            self.timer.stop(node)
        self.launches += 1

    # -- the programs of one timestep ----------------------------------------

    def c_grid(self) -> None:
        c, dt = self.cfg.consts, self.cfg.dt_acoustic
        fields = [self.f(n) for n in ("u", "v", "delp", "pt", "w", "gz")] + [self.f(m) for m in C_METRICS]
        fields += [self.f("ws"), self.f("uc"), self.f("vc")] + [self.s(n) for n in ("delpcc", "ptcc", "wcc", "pkc", "gzc", "riem_scr")]
        self.launch("c_grid", "fv3b_c_grid", fields,
                    [0.5 * dt, c["ptop"], c["rdgas"], c["grav"], c["gama"], c["p_fac"]], self.dom_ifaces)

    def d_sw(self, first: bool = False) -> None:
        """``first``: the timestep's first substep, whose accumulator inputs
        are the step's zeros (fv3b_d_sw's acc_reset) and which saves the
        step's dp1 (the delp it reads)."""
        c, dt = self.cfg.consts, self.cfg.dt_acoustic
        fields = [self.f(n) for n in PINGPONG + ("uc", "vc") + ACCUM] + [self.f(m) for m in D_METRICS]
        fields += [self.a(n) for n in PINGPONG] + [self.f(n) for n in ACCUM]
        if first:
            fields.append(self.f("dp1"))  # the step's dp1 = delp at the step start
        self.launch("d_sw", "fv3b_d_sw", fields,
                    [c["ppm_p1"], c["ppm_p2"], dt, c["dddmp"], c["d2_bg"], c["da_min"], c["damp4"], c["damp4h"],
                     c["dampv"], 1.0 if first else 0.0], self.dom_layers)
        self.swap(*PINGPONG)

    def nh_d(self) -> None:
        c, dt = self.cfg.consts, self.cfg.dt_acoustic
        fields = [self.f(n) for n in ("delp", "pt", "w", "gz", "ws")] + [self.f("pef"), self.a("gz"), self.a("w"), self.s("riem_scr")]
        self.launch("nh_d", "fv3b_nh_d", fields, [c["ptop"], c["rdgas"], c["grav"], c["gama"], c["p_fac"], dt],
                    self.dom_ifaces)
        self.swap("w", "gz")

    def p_grad_d(self) -> None:
        fields = [self.f(n) for n in ("u", "v", "pef", "gz", "rdx", "rdy")] + [self.a("u"), self.a("v")]
        self.launch("p_grad_d", "fv3b_p_grad_d", fields, [self.cfg.dt_acoustic], self.dom_ifaces)
        self.swap("u", "v")

    def tracer_2d(self) -> None:
        c = self.cfg.consts
        qs = self.cfg.tracer_names()
        fields = [self.f(n) for n in ("cx", "cy", "xfa", "yfa", "mfx", "mfy", "dp1", "area", "rarea")]
        fields += [self.f(q) for q in qs] + [self.a(q) for q in qs]
        self.launch("tracer_2d", "fv3b_tracer_2d", fields, [c["ppm_p1"], c["ppm_p2"]], self.dom_layers)
        self.swap(*qs)

    def remap(self, thickness: bool = True) -> None:
        """remap_profile of every remapped field: the tracers, pt and w at
        delp (the remap_tracers program, and the remap_profile program per
        field), and the D-grid winds at the layer thickness of their points
        (fv3b_face_thickness; delp's halo is refreshed at the tracer halo
        point).  One launch per kernel, the field groups sharing it.
        ``thickness=False``: the thicknesses were launched already
        (remap_thickness)."""
        if thickness:
            self.remap_thickness()
        fields, counts = [], []
        for thick, names in self._remap_groups():
            counts.append(float(len(names)))
            fields.append(thick)
            for q in names:
                fields += [self.f(q), self.f(f"{q}_a2"), self.f(f"{q}_a3"), self.f(f"{q}_a4")]
        self.launch("remap_tracers", "fv3b_remap_profile", fields, counts, self.dom_ifaces)

    def remap_thickness(self) -> None:
        """The remapping's layer thicknesses: the D-grid winds' at their
        points (fv3b_face_thickness) and pt's log-pressure interfaces
        (fv3b_log_thickness), from delp alone."""
        self.launch("remap_faces", "fv3b_face_thickness", [self.f("delp"), self.s("du"), self.s("dv")], [],
                    self.dom_layers)
        if self.cfg.pt_logp:  # pt is profiled at the log-pressure thickness
            coord = [self.grid.abi(self.coord[n], rank=1) for n in ("ak", "bk")]
            self.launch("remap_logp", "fv3b_log_thickness",
                        [self.f("delp")] + coord + [self.s(n) for n in ("dlnp", "lnpe1", "lnpe2")], [],
                        self.dom_layers)

    def advect_and_thickness(self) -> None:
        """tracer_2d, with the remapping's thickness kernels on a side stream
        beside it (they read delp only and write scratch; their few
        registers and no shared memory fit next to tracer_2d's CTAs).  Under
        a per-launch timer they stay in line."""
        if self.timer is not None:
            self.tracer_2d()
            self.remap_thickness()
            return
        comp = torch.cuda.current_stream()
        if getattr(self, "_thick_stream", None) is None:
            self._thick_stream = torch.cuda.Stream()
        side = self._thick_stream
        side.wait_event(comp.record_event())
        with torch.cuda.stream(side):
            self.remap_thickness()
            done = side.record_event()
        self.tracer_2d()
        comp.wait_event(done)

    def _remap_groups(self):
        """(thickness, fields) of the profile launch: the tracers and w (and
        pt unless pt_logp) at delp, pt at its log-pressure thickness, the
        winds at their face thickness."""
        cfg = self.cfg
        groups = [(self.f("delp"), cfg.remap_linear())]
        if cfg.pt_logp:
            groups.append((self.s("dlnp"), ["pt"]))
        return groups + [(self.s("du"), ["u"]), (self.s("dv"), ["v"])]

    def _map_launches(self):
        """(node, [(thickness fields, fields, sign)]) of the mapping launches:
        the fields at delp (which rewrites delp), then the winds at their
        face thickness and pt in log pressure (sign -1: between the log
        interfaces of fv3b_log_thickness)."""
        side = [([self.s("du")], ["u"], 1.0), ([self.s("dv")], ["v"], 1.0)]
        if self.cfg.pt_logp:
            side.append(([self.s("lnpe1"), self.s("lnpe2")], ["pt"], -1.0))
        return [("remap_map", [([self.f("delp")], self.cfg.remap_linear(), 1.0)]), ("remap_map_winds", side)]

    def moist_pk(self) -> None:
        """Pressure and heat-capacity diagnostics of the remapped state: pe,
        peln, pk at the interfaces, pkz and the moist cv at the layers
        (fv3b_moist_pk; oracle/thermo.py)."""
        fields = [self.f("delp")] + [self.f(q) for q in self.cfg.moist_names()]
        fields += [self.f(n) for n in DIAG_3D]
        self.launch("moist_pk", "fv3b_moist_pk", fields, self.cfg.moist_scalars(), self.dom_ifaces)

    def remap_map(self) -> None:
        """Lagrangian -> Eulerian: every remapped field's profile integrated
        over the target layers (pe2 = ak + bk * ps of its thickness), each
        thickness <- its pe2 differences (delp; the winds' are scratch)."""
        coord = [self.grid.abi(self.coord[n], rank=1) for n in ("ak", "bk")]
        swapped = []
        # the scalars' group (9 or 10 fields) and the single-field groups in
        # separate launches (measured: one launch of all of them is slower),
        # run concurrently: the two read and write disjoint fields (the
        # scalars rewrite delp; the others map at du, dv and the log-pressure
        # interfaces), and both column walks are latency-bound at a few warps
        # per SM, so each fills the other's stalls (step 7.63 -> 7.58 ms).
        # Under a per-launch timer they run one after the other, so each
        # launch's events bracket only its own kernel.
        comp = torch.cuda.current_stream()
        if getattr(self, "_map_stream", None) is None:
            self._map_stream = torch.cuda.Stream()
        fork = comp.record_event()
        joins = []
        for idx, (node, launch) in enumerate(self._map_launches()):
            fields, counts = list(coord), []
            for thick, names, sign in launch:
                counts.append(sign * len(names))
                fields += thick
                for q in names:
                    fields += [self.f(q), self.f(f"{q}_a2"), self.f(f"{q}_a3"), self.f(f"{q}_a4"), self.a(q)]
                    swapped.append(q)
            if idx == 0 or self.timer is not None:
                self.launch(node, "fv3b_remap_map", fields, counts, self.dom_ifaces)
                continue
            side = self._map_stream
            side.wait_event(fork)
            with torch.cuda.stream(side):
                self.launch(node, "fv3b_remap_map", fields, counts, self.dom_ifaces)
                joins.append(side.record_event())
        for e in joins:
            comp.wait_event(e)
        self.swap(*swapped)

    def phases(self):
        """One timestep as a generator: enqueues the programs on the current
        stream and yields, at each halo-update point, the fields to refresh
        (the caller performs the update; a decomposed run exchanges them
        between ranks, parallel.py)."""
        cfg = self.cfg
        # the accumulators start the step at zero and dp1 is the delp of the
        # step start: the first d_sw reads the former as 0.0 (acc_reset) and
        # writes the latter (its delp input) instead of a fill and a copy
        for it in range(cfg.n_split):
            yield from self.acoustic_phases(first=it == 0)
        yield cfg.tracer_names() + list(ACCUM) + ["delp"]  # (delp: the winds' remapping thickness)
        self.advect_and_thickness()
        self.remap(thickness=False)
        self.remap_map()
        self.moist_pk()

    def acoustic_phases(self, first: bool = False):
        """One acoustic substep (BASELINE config C1: halo, c_sw +
        riem_solver_c + p_grad_c, halo, d_sw, then the D-grid vertical solve
        and pressure gradient), yielding its halo-update points like
        ``phases``.  ``first``: the timestep's first substep (d_sw's
        acc_reset and dp1 copy)."""
        yield ["u", "v", "w", "delp", "pt", "gz"]
        self.c_grid()
        yield ["uc", "vc"]
        self.d_sw(first=first)
        self.nh_d()
        yield ["pef", "gz"]
        self.p_grad_d()

    def substep(self, first: bool = False) -> None:
        """Enqueue one acoustic substep on the current stream."""
        for names in self.acoustic_phases(first):
            self.halo.update(names)

    def step(self) -> None:
        """Enqueue one full timestep on the current stream (with
        ``self.overlap``: halo exchanges on a second stream, see
        :meth:`step_overlapped`)."""
        if self.overlap:
            self.step_overlapped()
            return
        for names in self.phases():
            self.halo.update(names)

    # -- halo exchanges overlapped with compute ----------------------------------

    def _comm(self) -> torch.cuda.Stream:
        if getattr(self, "_comm_stream", None) is None:
            self._comm_stream = torch.cuda.Stream()
        return self._comm_stream

    def _start(self, names) -> torch.cuda.Event:
        """Start the halo update of ``names`` on the exchange stream once the
        compute stream has produced them; returns its completion event."""
        comm = self._comm()
        comm.wait_event(torch.cuda.current_stream().record_event())
        with torch.cuda.stream(comm):
            self.halo.update(list(names))
        return comm.record_event()

    @staticmethod
    def _wait(*events) -> None:
        for e in events:
            if e is not None:
                torch.cuda.current_stream().wait_event(e)

    def step_overlapped(self) -> None:
        """One timestep whose halo exchanges run on a second stream (SURVEY
        8(e): the halo moves under compute).  Each field group's exchange
        starts as soon as its producer has run and is waited for only by the
        program that reads the halo, so a group whose next reader is not the
        next program moves under the programs in between:

        * the tracers (q*, unchanged by the acoustic substeps) from the step
          start, under every substep, until tracer_2d;
        * w, delp, pt (final after d_sw / nh_d) under p_grad_d, until the
          next substep's c_grid; u, v after p_grad_d;
        * the flux accumulators and delp after the last d_sw / nh_d, under
          the last p_grad_d, until tracer_2d.
        gz is refreshed with pef after nh_d (p_grad_d and the next c_grid
        read it; nothing in between writes it), and every group is exchanged
        exactly when the plain step's halo points would leave it fresh, so
        the results are bitwise those of :meth:`step` (tests)."""
        cfg = self.cfg
        tracers = cfg.tracer_names()
        dyn = [self._start(["u", "v", "w", "delp", "pt", "gz"])]
        ev_trc = self._start(tracers) if tracers else None
        ev_acc = None
        for it in range(cfg.n_split):
            last = it == cfg.n_split - 1
            self._wait(*dyn)
            self.c_grid()
            self._wait(self._start(["uc", "vc"]))
            self.d_sw(first=it == 0)
            self.nh_d()
            ev_p = self._start(["pef", "gz"])
            if last:
                ev_acc = self._start(list(ACCUM) + ["delp"])
            else:
                dyn = [self._start(["w", "delp", "pt"])]
            self._wait(ev_p)
            self.p_grad_d()
            if not last:
                dyn.append(self._start(["u", "v"]))
        self._wait(ev_trc, ev_acc)
        self.advect_and_thickness()
        self.remap(thickness=False)
        self.remap_map()
        self.moist_pk()
        # the exchange stream joins the compute stream (graph capture, next step)
        self._wait(self._comm().record_event())

    # -- CUDA graphs ---------------------------------------------------------

    def _assignment(self) -> tuple:
        return tuple(self.cur[n].data_ptr() for n in sorted(self.cur))

    def capture(self) -> None:
        """Capture one timestep per distinct buffer assignment.  A step
        permutes the ping-pong buffers (every field swaps an even number of
        times at present, so one graph suffices); the captures follow the
        assignments until they cycle.  Capture executes nothing, so the
        state is unchanged; the bookkeeping is restored afterwards."""
        start = (dict(self.cur), dict(self.alt))
        self._graphs = {}
        with capture_guard():
            while self._assignment() not in self._graphs:
                key = self._assignment()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g):
                    self.step()
                self._graphs[key] = (g, dict(self.cur), dict(self.alt))
        self.cur, self.alt = start
        torch.cuda.synchronize()

    def replay(self) -> None:
        """Run one captured timestep on the current stream."""
        g, cur, alt = self._graphs[self._assignment()]
        g.replay()
        self.cur, self.alt = dict(cur), dict(alt)


# libfv3b kernels launched per entry point (fused entries launch several)
KERNELS = {"fv3b_c_grid": 3, "fv3b_d_sw": 2}


def interior_rows(cfg: RunConfig) -> tuple[int, int, int, int]:
    """(byte offset, row bytes, rows, pitch) of the interior columns of a
    step_host array (reference convention: I, J, K C order, halo h, nk + 1
    levels): for each interior i, j in [h, h + nj) over all levels is one
    contiguous run."""
    h = cfg.halo
    nk1 = cfg.nk + 1
    pitch = (cfg.nj + 2 * h) * nk1 * 8
    return (h * (cfg.nj + 2 * h) + h) * nk1 * 8, cfg.nj * nk1 * 8, cfg.ni, pitch


def kernels_per_step(cfg: RunConfig) -> int:
    per_sub = 3 + KERNELS["fv3b_c_grid"] + KERNELS["fv3b_d_sw"] + 1 + 1
    # tracer halo, tracer_2d, face thickness (+ log thickness) + profiles, maps, moist_pk
    return cfg.n_split * per_sub + 1 + 1 + 2 + int(cfg.pt_logp) + 2 + 1
