"""Tuned launch configurations (tools/tune.py), keyed by device and shape.

``tuning.json`` holds, per ``"<device name>|<ni>x<nj>x<nk>"``, the
fv3b_tune_set knobs the tuner kept (only values that beat the automatic
choice on the whole step), with the sweep that chose them.  ``apply`` sets
the knobs of the matching entry process-wide (``_lib.tune_set``); shapes or
devices without an entry keep the automatic choices.
"""

from __future__ import annotations

import json
from pathlib import Path

from . import _lib

PATH = Path(__file__).resolve().parent / "tuning.json"


def _key(device: str, shape) -> str:
    return f"{device}|{shape[0]}x{shape[1]}x{shape[2]}"


def load() -> dict:
    return json.loads(PATH.read_text()) if PATH.exists() else {}


def lookup(device: str, shape) -> dict:
    return load().get(_key(device, shape), {}).get("knobs", {})


def apply(device: str, shape) -> dict:
    """Set the tuned knobs for (device, shape); returns them ({} = automatic)."""
    knobs = lookup(device, shape)
    for k, v in knobs.items():
        _lib.tune_set(k, int(v))
    return knobs


def record(device: str, shape, entry: dict) -> None:
    table = load()
    table[_key(device, shape)] = entry
    PATH.write_text(json.dumps(table, indent=1, sort_keys=True) + "\n")
