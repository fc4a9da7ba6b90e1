"""tilejoin.grid -> the device grid index exported in the reference's shape."""
import sys

from paper_2209_11287_b200 import grid as _impl

sys.modules[__name__] = _impl
