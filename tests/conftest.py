"""Shared fixtures.  GPU tests carry @pytest.mark.gpu and call the CUDA path
through libtedjoin.so; everything else runs on CPU (oracle, host logic, ABI)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) and libtedjoin.so")
    config.addinivalue_line("markers", "slow: multi-second case")


def load_json(name):
    return json.loads((GOLDEN / name).read_text())


@pytest.fixture(scope="session")
def golden_sweep():
    return load_json("sweep.json")


@pytest.fixture(scope="session")
def golden_generator():
    return load_json("generator.json")


def sha_pairs(pairs) -> str:
    import hashlib

    return hashlib.sha256(np.ascontiguousarray(pairs, dtype="<i8").tobytes()).hexdigest()


def csr_equal(off_a, nb_a, off_b, nb_b) -> bool:
    off_a, off_b = np.asarray(off_a, np.int64), np.asarray(off_b, np.int64)
    if not np.array_equal(off_a, off_b):
        return False
    m = int(off_a[-1])
    return np.array_equal(np.asarray(nb_a[:m], np.int64), np.asarray(nb_b[:m], np.int64))
