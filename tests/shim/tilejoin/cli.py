"""tilejoin.cli -> the drop-in CLI (the same module object, so monkeypatching
tilejoin.cli.self_join patches what the commands call)."""
import sys

from paper_2209_11287_b200 import cli as _impl

sys.modules[__name__] = _impl
