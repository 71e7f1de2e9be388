"""B200-native (sm_100a) hot path of HPEZ / QoZ 2.0 (arXiv 2311.12133).

Drop-in for the reference package's interpolation sweep and its callers:
``run_levels`` / ``run_levels_device`` (interp.run_levels), Lorenzo,
histogram + canonical Huffman, block-wise tuning, and the unchanged
``compress`` / ``decompress`` archive API on top.
"""

from .errors import HpezError  # noqa: F401
from .interp import (CodeSource, PassStats, TRAVERSAL_DIM_MAJOR,  # noqa: F401
                     TRAVERSAL_FVFI, block_grid_shape, run_levels, run_levels_device)
from .plan import (KERNEL_VARIANTS, PARADIGM_MULTIDIM, PARADIGM_ONED,  # noqa: F401
                   CompressionConfig, InterpKernel, KernelTag, LevelConfig, LevelSpec,
                   build_level_plan, decode_tag, encode_tag)
from .quant import DEFAULT_RADIUS, ROUND_F32, ROUND_INT, ROUND_NONE  # noqa: F401

__version__ = "0.1.0"
