"""Loader for the golden fixtures in tests/golden/ (made by make_golden.py
from the unmodified reference package)."""

from __future__ import annotations

import glob
import hashlib
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


class Fixture:
    def __init__(self, path):
        self.name = os.path.basename(path)[:-4]
        z = np.load(path)
        self.meta = json.loads(str(z["meta"]))
        self.arrays = {k: z[k] for k in z.files if k != "meta"}

    def __getitem__(self, k):
        a = self.arrays[k]
        if k in ("input", "outliers", "work_c", "work_d", "dense", "recon",
                 "err_sum") and a.dtype == np.float32 and self.meta.get("kind") != "pipeline":
            return a.astype(np.float64)
        if k == "codes":
            return a.astype(np.int32)
        if k == "symbols":
            return a.astype(np.int64)
        if k == "input" and self.meta.get("kind") == "pipeline":
            return a.astype({"f32": np.float32, "f64": np.float64, "i32": np.int32,
                             "i64": np.int64}[self.meta["grid_kind"]])
        return a

    def __contains__(self, k):
        return k in self.arrays or k in self.meta.get("sha", {})

    def check(self, k, value) -> bool:
        """Exact comparison against the stored array or its SHA-256."""
        value = np.ascontiguousarray(value)
        if k in self.meta.get("sha", {}):
            digest, dtype, shape = self.meta["sha"][k]
            value = value.astype(dtype).reshape(shape)
            return hashlib.sha256(value.tobytes()).hexdigest() == digest
        ref = self[k]
        return ref.shape == value.shape and ref.tobytes() == value.astype(ref.dtype).tobytes()


def fixtures(kind: str):
    out = []
    for p in sorted(glob.glob(os.path.join(GOLDEN, "*.npz"))):
        f = Fixture(p)
        if f.meta["kind"] == kind:
            out.append(f)
    return out


def level_tuples(meta):
    return [tuple(x) for x in meta["levels"]]
