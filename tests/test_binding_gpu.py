"""INTEGRATION.md §1 exercised for real: the UNMODIFIED reference package
(installed into baseline/_ref with pip) has its hot path
rebound to the B200 drop-ins by paper_2311_12133_b200.binding, and its own
hpez.compress / hpez.decompress must produce byte-identical archives
(SHA-256) and identical reconstructions to the unbound reference."""

import hashlib
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "baseline", "_ref")

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(
    not os.path.isdir(os.path.join(REF, "hpez")), reason="baseline/_ref (pip install of the reference) absent")]

SCRIPT = r"""
import hashlib, json, sys
sys.path.insert(0, {ref!r}); sys.path.insert(0, {root!r})
import numpy as np
import hpez
import synthetic as syn
from hpez.grid import BoundMode, ElementKind, ErrorBoundSpec, ScalarGrid
cases = [
    ("cfg4_small", syn.config_field(4, dims=(64, 72, 80)), ElementKind.F32, BoundMode.REL, 1e-3),
    ("cfg2_small", syn.config_field(2, dims=(48, 56, 64)), ElementKind.F32, BoundMode.REL, 1e-4),
    ("f64_abs", syn.config_field(3, dims=(40, 50, 60)).astype(np.float64), ElementKind.F64, BoundMode.ABS, 0.05),
    ("i32", (syn.config_field(1, dims=(40, 44, 48)) * 1000).astype(np.int32), ElementKind.I32, BoundMode.ABS, 3.0),
]
def run():
    out = {{}}
    for name, a, kind, mode, eps in cases:
        g = ScalarGrid(a.shape, kind, a)
        res = hpez.compress(g, ErrorBoundSpec(mode, eps))
        back = hpez.decompress(res.archive)
        out[name] = [hashlib.sha256(res.archive).hexdigest(),
                     hashlib.sha256(back.data.tobytes()).hexdigest(),
                     hashlib.sha256(res.reconstruction.data.tobytes()).hexdigest()]
    return out
ref = run()
from paper_2311_12133_b200 import binding
binding.enable(hpez)
import hpez.interp
assert hpez.interp.run_levels.__module__.startswith("paper_2311_12133_b200")
b2 = run()
print(json.dumps({{"ref": ref, "b200": b2}}))
"""


def test_reference_package_with_b200_binding_is_byte_identical():
    code = SCRIPT.format(ref=REF, root=ROOT)
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    import json
    d = json.loads(r.stdout.strip().splitlines()[-1])
    assert d["b200"] == d["ref"]
