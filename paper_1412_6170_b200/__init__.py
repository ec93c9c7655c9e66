"""B200-native per-tick repeated k-NN join (arXiv 1412.6170), drop-in for the
reference package ``mknn``'s tick API (Engine / EngineConfig / TickResult /
TickMetrics).  All tick work runs in libmknn_b200.so (hand-written sm_100a
kernels behind the C-ABI in include/mknn_b200.h)."""

from .engine import Engine, EngineConfig, TickMetrics, TickResult, resolve_th_quad
from .geometry import Point, Rect
from .index import QuadIndex, should_rebuild

__version__ = "0.1.0"

__all__ = [
    "Engine",
    "EngineConfig",
    "Point",
    "QuadIndex",
    "Rect",
    "TickMetrics",
    "TickResult",
    "__version__",
    "resolve_th_quad",
    "should_rebuild",
]
