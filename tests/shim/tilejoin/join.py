"""tilejoin.join -> the drop-in (join.py:150 self_join and its types)."""
import sys

from paper_2209_11287_b200 import join as _impl

sys.modules[__name__] = _impl
