"""B200-native Kino-PAX+ planning iteration (arXiv 2602.02846), drop-in for the
reference `kinoplan` CPU planner.  The planner itself is the sm_100a library
lib/libkinoplan_b200.so behind the C-ABI include/kinoplan_b200.h; this package
holds the ctypes mirror of that ABI, the Python mirror of the reference API and
the bundled scenario files."""
from . import scenarios  # noqa: F401
from .planner import (  # noqa: F401
    BatchPlanner,
    ConfigError,
    DeviceError,
    GridTooFineError,
    InvalidProblemError,
    InvalidSegmentError,
    Planner,
    SchemaError,
    plan,
)

__all__ = ["Planner", "BatchPlanner", "plan", "scenarios", "SchemaError", "InvalidProblemError", "ConfigError",
           "GridTooFineError", "InvalidSegmentError", "DeviceError"]
