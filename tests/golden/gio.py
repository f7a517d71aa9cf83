"""Tiny nested-structure <-> .npz codec for the golden fixtures.

A fixture is a nested dict/list of numpy arrays, numbers, strings, bools
and None.  Arrays go into the .npz; the structure (with array references)
is stored as JSON under the key ``__tree__``.
"""

from __future__ import annotations

import json

import numpy as np


def save(path, obj) -> None:
    arrays = {}

    def enc(x):
        if isinstance(x, dict):
            return {"d": {str(k): enc(v) for k, v in x.items()}}
        if isinstance(x, (list, tuple)):
            return {"l": [enc(v) for v in x]}
        if isinstance(x, np.ndarray):
            key = f"a{len(arrays)}"
            arrays[key] = x
            return {"a": key}
        if isinstance(x, (np.floating, float)):
            return {"f": float(x).hex()}
        if isinstance(x, (np.integer, int)) and not isinstance(x, bool):
            return {"i": int(x)}
        if isinstance(x, (bool, np.bool_)):
            return {"b": bool(x)}
        if x is None:
            return {"n": 0}
        if isinstance(x, str):
            return {"s": x}
        raise TypeError(f"cannot encode {type(x)}")

    tree = enc(obj)
    arrays["__tree__"] = np.frombuffer(json.dumps(tree).encode(), dtype=np.uint8)
    np.savez_compressed(path, **arrays)


def load(path):
    with np.load(path, allow_pickle=False) as z:
        arrays = {k: z[k] for k in z.files}
    tree = json.loads(arrays.pop("__tree__").tobytes().decode())

    def dec(x):
        (kind, val), = x.items()
        if kind == "d":
            return {k: dec(v) for k, v in val.items()}
        if kind == "l":
            return [dec(v) for v in val]
        if kind == "a":
            return arrays[val]
        if kind == "f":
            return float.fromhex(val)
        if kind == "i":
            return int(val)
        if kind == "b":
            return bool(val)
        if kind == "n":
            return None
        if kind == "s":
            return val
        raise ValueError(kind)

    return dec(tree)
