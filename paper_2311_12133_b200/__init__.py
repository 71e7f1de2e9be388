"""B200-native (sm_100a) hot path of HPEZ / QoZ 2.0 (arXiv 2311.12133).

Drop-in for the reference package's interpolation sweep and its callers:
``run_levels`` / ``run_levels_device`` (interp.run_levels), ``lorenzo_pass``,
GPU histogram + canonical Huffman (``pack_codes``), GPU block-wise tuning
(``tune`` / ``tune_blocks``), and the unchanged ``compress`` / ``decompress``
archive API on top.  There is no CPU fallback: every hot-path call needs the
in-tree libhpez_b200.so and a CUDA device.
"""

from .errors import HpezError  # noqa: F401
from .grid import (BoundMode, ElementKind, ErrorBoundSpec, ScalarGrid,  # noqa: F401
                   load_raw, value_range)
from .interp import (CodeSource, PassStats, TRAVERSAL_DIM_MAJOR,  # noqa: F401
                     TRAVERSAL_FVFI, block_grid_shape, run_levels, run_levels_device)
from .plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM, PARADIGM_ONED,  # noqa: F401
                   CompressionConfig, InterpKernel, KernelTag, LevelConfig, LevelSpec,
                   build_level_plan, decode_tag, encode_tag)
from .quant import DEFAULT_RADIUS, ROUND_F32, ROUND_INT, ROUND_NONE  # noqa: F401


def __getattr__(name):
    # heavier modules load lazily so `import paper_2311_12133_b200` stays cheap
    if name in ("compress", "decompress", "CompressResult"):
        from . import pipeline
        return getattr(pipeline, name)
    if name in ("tune", "TunerOptions", "QualityTarget", "tune_blocks"):
        from . import tuner
        return getattr(tuner, name)
    if name in ("lorenzo_pass", "lorenzo_pass_device"):
        from . import lorenzo
        return getattr(lorenzo, name)
    if name in ("pack_codes", "unpack_codes"):
        from . import container
        return getattr(container, name)
    raise AttributeError(name)


__version__ = "0.1.0"
