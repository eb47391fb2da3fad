"""Load the frozen golden fixtures (tests/golden/*.json + *_hist.npz).

Fixtures were produced in the dev container by ``oracle/gen_golden.py``
from the live reference (2-D) or the oracle restatement (3-D); histories
live in a sibling ``<group>_hist.npz`` (one float64 array (k, 4) per case:
iteration, Re sigma*, Im sigma*, residual) to keep the JSON small.
"""

from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load_group(name: str) -> dict:
    path = os.path.join(GOLDEN, f"{name}.json")
    if not os.path.exists(path):
        return {}
    with open(path) as f:
        recs = json.load(f)
    hp = os.path.join(GOLDEN, f"{name}_hist.npz")
    hist = np.load(hp) if os.path.exists(hp) else None
    out = {}
    for r in recs:
        nm = r["case"]["name"]
        if "history" not in r:
            r["history"] = hist[nm] if hist is not None and nm in hist.files else np.zeros((0, 4))
        else:
            r["history"] = np.asarray(r["history"], dtype=np.float64).reshape(-1, 4)
        out[nm] = r
    return out


def compact(name: str):
    """Move histories of a JSON group into <group>_hist.npz (idempotent)."""
    path = os.path.join(GOLDEN, f"{name}.json")
    with open(path) as f:
        recs = json.load(f)
    hp = os.path.join(GOLDEN, f"{name}_hist.npz")
    arrays = dict(np.load(hp)) if os.path.exists(hp) else {}
    for r in recs:
        if "history" in r:
            arrays[r["case"]["name"]] = np.asarray(r.pop("history"), dtype=np.float64).reshape(-1, 4)
    np.savez_compressed(hp, **arrays)
    with open(path + ".tmp", "w") as f:
        json.dump(recs, f, indent=0)
    os.replace(path + ".tmp", path)


if __name__ == "__main__":
    import sys

    for g in sys.argv[1:]:
        compact(g)
