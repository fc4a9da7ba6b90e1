"""`tilejoin` import shim (test infrastructure): maps the reference package's module
paths onto paper_2209_11287_b200 so the reference's own test files
(pkg/tests/test_join.py, test_cli.py) run unchanged against the GPU drop-in.
Used by tools/run_reference_tests.sh; never imported by the product."""

from paper_2209_11287_b200 import *  # noqa: F401,F403
from paper_2209_11287_b200 import __version__  # noqa: F401
