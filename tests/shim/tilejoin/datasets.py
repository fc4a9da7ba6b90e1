"""tilejoin.datasets -> the drop-in's dataset types, generator and readers."""
import sys

from paper_2209_11287_b200 import datasets as _impl

sys.modules[__name__] = _impl
