"""tilejoin.oracle.brute_force_join (oracle.py:55-86) -> the repo's numpy restatement
(oracle/__init__.py brute_force): the reference tests' ground truth."""
from dataclasses import dataclass

import numpy as np

import oracle as _oracle
from paper_2209_11287_b200.errors import ResourceError

BRUTE_FORCE_GUARD = 50_000


@dataclass(frozen=True)
class OraclePairSet:
    pairs: np.ndarray

    @property
    def total_pairs(self) -> int:
        return len(self.pairs)

    def __len__(self) -> int:
        return len(self.pairs)


def brute_force_join(dataset, epsilon: float, force: bool = False) -> OraclePairSet:
    n = len(getattr(dataset, "coords", dataset))
    if n > BRUTE_FORCE_GUARD and not force:
        raise ResourceError(f"n={n} exceeds the brute-force guard of {BRUTE_FORCE_GUARD}")
    return OraclePairSet(_oracle.brute_force(dataset, epsilon))
