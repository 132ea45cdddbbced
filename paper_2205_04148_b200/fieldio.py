"""Field I/O and dycore checkpoints in the reference's format.

``save_field`` / ``load_field`` follow ``stencilkit.executor.buffers``
(``buffers.py:83-116``): the halo-inclusive field content in the reference
array convention (axes in declared I, J, K order, C order) as raw binary,
plus a ``<path>.json`` sidecar with the field name, element type, shape and
the reference ``Layout`` (``scheduling.py:323-407``) of the field; text mode
writes one value per line after a header.  Files written here load with the
reference's ``load_field`` and vice versa (tests/test_perf_model.py).

``save_state`` / ``load_state`` checkpoint a :class:`~.dycore.Dycore` (every
state field, one file each, plus ``run.json`` with the run configuration) —
the restart / golden-state capture of SURVEY 8f #3.
"""

from __future__ import annotations

import json
from dataclasses import asdict
from pathlib import Path

import numpy as np

_DTYPES = {"float64": np.float64, "float32": np.float32}


def reference_layout(dims, shape, halo_lo, alignment: int = 8) -> dict:
    """The reference ``allocate_layout`` rule (scheduling.py:377-407) as its
    ``Layout.to_json`` document."""
    padded = list(shape)
    if dims:
        padded[0] = -(-shape[0] // alignment) * alignment
    strides, acc = [], 1
    for n in padded:
        strides.append(acc)
        acc *= n
    pre_pad = (alignment - (halo_lo[0] % alignment)) % alignment if dims else 0
    return {"dims": list(dims), "shape": list(shape), "halo_lo": list(halo_lo), "strides": strides,
            "pre_pad": pre_pad, "alignment": alignment}


def save_field(name: str, data: np.ndarray, path, dims=("I", "J", "K"), halo_lo=(0, 0, 0), text: bool = False):
    path = Path(path)
    data = np.ascontiguousarray(data)
    dtype = "float32" if data.dtype == np.float32 else "float64"
    if text:
        with open(path, "w") as fh:
            fh.write(f"# field {name} dtype {dtype} shape {list(data.shape)}\n")
            for v in data.ravel():
                fh.write(f"{v!r}\n")
        return
    data.astype(_DTYPES[dtype], copy=False).tofile(path)
    dims = tuple(dims)[: data.ndim]
    sidecar = {"field": name, "dtype": dtype, "shape": list(data.shape),
               "layout": reference_layout(dims, data.shape, tuple(halo_lo)[: data.ndim])}
    with open(path.with_suffix(path.suffix + ".json"), "w") as fh:
        json.dump(sidecar, fh, indent=2, sort_keys=True)


def load_field(path):
    """(name, layout document, array) of a binary field file."""
    path = Path(path)
    with open(path.with_suffix(path.suffix + ".json")) as fh:
        sidecar = json.load(fh)
    data = np.fromfile(path, dtype=_DTYPES[sidecar["dtype"]]).reshape(sidecar["shape"])
    return sidecar["field"], sidecar["layout"], data


def save_state(dycore, directory) -> None:
    """Checkpoint every state field of a Dycore (device -> files)."""
    d = Path(directory)
    d.mkdir(parents=True, exist_ok=True)
    h = dycore.cfg.halo
    arrays = dycore.download()
    for name, a in arrays.items():
        save_field(name, a, d / f"{name}.bin", ("I", "J", "K"), (h, h, 0))
    cfg = asdict(dycore.cfg)
    (d / "run.json").write_text(json.dumps({"config": cfg, "fields": sorted(arrays)}, indent=1, sort_keys=True))


def load_state(directory) -> tuple[dict, dict[str, np.ndarray]]:
    """(run config dict, {field: array}) of a checkpoint; pass the arrays to
    ``Dycore(cfg, state)`` or ``Dycore.load``."""
    d = Path(directory)
    meta = json.loads((d / "run.json").read_text())
    state = {}
    for name in meta["fields"]:
        fname, _, a = load_field(d / f"{name}.bin")
        state[fname] = a
    return meta["config"], state
