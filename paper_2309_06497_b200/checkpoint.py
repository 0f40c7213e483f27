"""Reference checkpoint interop: the one-file JSON-hex format of ``minishampoo.checkpoint``.

Format (checkpoint.py:1-144): one JSON object ``{"format_version": 1, "step": t, "params": [array,
...], "state": {"t": t, "params": {"i": {"b": {name: value}}}}}``; an array is ``{"shape": [...],
"dtype": "<f8" | "<f4", "hex": little-endian bytes as hex}``; keys sorted, compact separators, one
trailing newline -- so save -> load -> save is byte-identical, and a file written here is the file
the reference would write for the same state.  Parsing is strict: unknown keys, unknown state names,
a wrong version, an unsupported dtype or a payload of the wrong length raise ``CheckpointError``.

The state tree is the ``state_tree()`` nesting (optim.py:387-423).  ``merge_state_trees`` is the
sharded union of the reference trainer (train.py:346-353): the trees of one replica group's ranks,
each holding its owned blocks, merged so every block appears once.  Pure host code (numpy).
"""

from __future__ import annotations

import json
import re
from typing import Iterable

import numpy as np

__all__ = ["CheckpointError", "FORMAT_VERSION", "save_checkpoint", "load_checkpoint", "encode_array",
           "decode_array", "merge_state_trees", "dumps_checkpoint"]

FORMAT_VERSION = 1

_DTYPES = {np.dtype("<f8"): "<f8", np.dtype("<f4"): "<f4"}
_SCALARS = frozenset({"kind", "graft_step", "step", "last_inverse_step"})
_ARRAYS = frozenset({"graft_accumulator", "filtered_grad", "momentum", "accumulator"})
_PER_MODE = re.compile(r"(?:factor|inv_factor|diag)[0-9]+")


class CheckpointError(ValueError):
    """Malformed checkpoint (checkpoint.py:32-33)."""


def encode_array(a) -> dict:
    a = np.ascontiguousarray(a)
    code = _DTYPES.get(a.dtype.newbyteorder("<") if a.dtype.byteorder == ">" else a.dtype)
    if code is None:
        raise CheckpointError(f"cannot store arrays of dtype {a.dtype} (float64/float32 only)")
    raw = a.astype(np.dtype(code), copy=False).tobytes()
    return {"shape": [int(d) for d in a.shape], "dtype": code, "hex": raw.hex()}


def decode_array(obj, where: str = "array") -> np.ndarray:
    if not isinstance(obj, dict) or set(obj) != {"shape", "dtype", "hex"}:
        raise CheckpointError(f"{where}: an array needs exactly the keys dtype, hex, shape")
    code = obj["dtype"]
    if code not in ("<f8", "<f4"):
        raise CheckpointError(f"{where}: dtype {code!r} is not <f8 or <f4")
    shape = tuple(int(d) for d in obj["shape"])
    try:
        raw = bytes.fromhex(obj["hex"])
    except (TypeError, ValueError) as exc:
        raise CheckpointError(f"{where}: hex payload does not decode") from exc
    dt = np.dtype(code)
    need = int(np.prod(shape, dtype=np.int64)) * dt.itemsize
    if len(raw) != need:
        raise CheckpointError(f"{where}: {len(raw)} payload bytes, shape {shape} x {dt.itemsize} needs {need}")
    return np.frombuffer(raw, dtype=dt).reshape(shape).copy()


def _state_to_json(tree: dict) -> dict:
    params = {}
    for i, blocks in tree["params"].items():
        params[str(int(i))] = {
            str(int(b)): {name: (encode_array(v) if isinstance(v, np.ndarray) else v) for name, v in entry.items()}
            for b, entry in blocks.items()}
    return {"t": int(tree["t"]), "params": params}


def _state_from_json(obj) -> dict:
    if not isinstance(obj, dict) or set(obj) != {"t", "params"}:
        raise CheckpointError("state: expected exactly the keys params, t")
    out = {"t": int(obj["t"]), "params": {}}
    for i, blocks in obj["params"].items():
        row = out["params"].setdefault(int(i), {})
        for b, entry in blocks.items():
            dec = {}
            for name, v in entry.items():
                where = f"state[{i}][{b}][{name}]"
                if not (name in _SCALARS or name in _ARRAYS or _PER_MODE.fullmatch(name)):
                    raise CheckpointError(f"{where}: unknown state name")
                dec[name] = decode_array(v, where) if isinstance(v, dict) else v
            row[int(b)] = dec
    return out


def dumps_checkpoint(step: int, params: Iterable, state: dict) -> str:
    """The file contents save_checkpoint writes (sorted keys, compact separators, trailing newline)."""
    doc = {"format_version": FORMAT_VERSION, "step": int(step),
           "params": [encode_array(np.asarray(p)) for p in params], "state": _state_to_json(state)}
    return json.dumps(doc, sort_keys=True, separators=(",", ":")) + "\n"


def save_checkpoint(path: str, step: int, params: Iterable, state: dict) -> None:
    """Write a reference-format checkpoint (checkpoint.py:114-126)."""
    text = dumps_checkpoint(step, params, state)
    with open(path, "w") as fh:
        fh.write(text)


def load_checkpoint(path: str):
    """Read a reference-format checkpoint (checkpoint.py:129-144) -> (step, params, state tree)."""
    with open(path) as fh:
        doc = json.load(fh)
    keys = {"format_version", "step", "params", "state"}
    if not isinstance(doc, dict) or set(doc) != keys:
        raise CheckpointError(f"top level: expected exactly the keys {sorted(keys)}")
    if doc["format_version"] != FORMAT_VERSION:
        raise CheckpointError(f"format_version {doc['format_version']!r} is not {FORMAT_VERSION}")
    params = [decode_array(p, f"params[{k}]") for k, p in enumerate(doc["params"])]
    return int(doc["step"]), params, _state_from_json(doc["state"])


def merge_state_trees(trees: Iterable[dict]) -> dict:
    """Union of per-rank state trees of ONE replica group (train.py:346-353): every block appears in
    exactly one rank's tree; the merged tree holds them all (step count of the first tree)."""
    trees = list(trees)
    if not trees:
        raise ValueError("no state trees to merge")
    merged = {"t": int(trees[0]["t"]), "params": {}}
    for tr in trees:
        if int(tr["t"]) != merged["t"]:
            raise CheckpointError("state trees disagree on the step count")
        for i, blocks in tr["params"].items():
            row = merged["params"].setdefault(int(i), {})
            for b, entry in blocks.items():
                if int(b) in row:
                    raise CheckpointError(f"block ({i}, {b}) is owned by more than one rank")
                row[int(b)] = entry
    return merged
