"""tilejoin.errors -> the drop-in's exception taxonomy."""
import sys

from paper_2209_11287_b200 import errors as _impl

sys.modules[__name__] = _impl
