"""The module-level binding a maintainer adds to the reference package
(INTEGRATION.md §1): it rebinds the hot-path entry points of an imported
``hpez`` to the B200 drop-ins, by name at every call site the reference
uses (pipeline.py:17-26 and tuner.py:19-27 import them by name).

    import hpez
    from paper_2311_12133_b200 import binding
    binding.enable(hpez)     # hpez.compress / decompress now run on the GPU

The archives are byte-identical to the unbound reference's
(tests/test_binding_gpu.py checks SHA-256 equality).
"""

from __future__ import annotations

import importlib

_PATCHED = {}


def enable(hpez) -> None:
    from . import container as c2
    from . import interp as i2
    from . import lorenzo as l2
    from . import tuner as t2
    from . import errors as e2
    mods = {m: importlib.import_module(f"{hpez.__name__}.{m}")
            for m in ("container", "interp", "lorenzo", "pipeline", "tuner", "errors")}
    table = [
        ("interp", "run_levels", i2.run_levels),        # interp.py:440
        ("pipeline", "run_levels", i2.run_levels),      # bound by name at pipeline.py:21
        ("tuner", "run_levels", i2.run_levels),         # bound by name at tuner.py:20
        ("lorenzo", "lorenzo_pass", l2.lorenzo_pass),   # lorenzo.py:145
        ("pipeline", "lorenzo_pass", l2.lorenzo_pass),
        ("tuner", "lorenzo_pass", l2.lorenzo_pass),
        ("container", "pack_codes", c2.pack_codes),     # container.py:70
        ("container", "unpack_codes", c2.unpack_codes),  # container.py:88
        ("pipeline", "pack_codes", c2.pack_codes),
        ("pipeline", "unpack_codes", c2.unpack_codes),
        ("tuner", "tune_blocks", t2.tune_blocks),       # tuner.py:414
        ("tuner", "analyze_samples", t2.analyze_samples),  # tuner.py:86
    ]
    for mod, name, fn in table:
        m = mods[mod]
        if hasattr(m, name):
            _PATCHED.setdefault((m, name), getattr(m, name))
            setattr(m, name, fn)
    # the drop-ins raise the reference's own exception classes
    for name in ("CorruptStream", "OutlierUnderflow", "EmptyInput", "InvalidTable", "TruncatedStream"):
        if hasattr(mods["errors"], name):
            _PATCHED.setdefault((e2, name), getattr(e2, name))
            setattr(e2, name, getattr(mods["errors"], name))


def disable() -> None:
    for (m, name), fn in _PATCHED.items():
        setattr(m, name, fn)
    _PATCHED.clear()
