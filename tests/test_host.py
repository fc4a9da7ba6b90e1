"""CPU: host-side logic of the drop-in (validation, batching, partitioning, ABI)."""

import re

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from conftest import ROOT
from paper_2209_11287_b200 import (
    Dataset,
    JoinConfig,
    ValidationError,
    plan_from_estimates,
    self_join,
)
from paper_2209_11287_b200 import _native
from paper_2209_11287_b200.distributed import balanced_cell_ranges


def greedy_reference(est, batch_size):
    """join.py:128-147 restated literally (per-cell loop)."""
    if batch_size is None:
        return [(0, len(est))], [sum(est)]
    batches, estimates, start, acc = [], [], 0, 0
    for i, e in enumerate(est):
        acc += e
        if acc >= batch_size:
            batches.append((start, i + 1))
            estimates.append(acc)
            start, acc = i + 1, 0
    if start < len(est):
        batches.append((start, len(est)))
        estimates.append(acc)
    return batches, estimates


@settings(max_examples=200, deadline=None)
@given(est=st.lists(st.integers(1, 1000), min_size=1, max_size=300),
       batch=st.one_of(st.none(), st.integers(1, 5000)))
def test_plan_matches_reference_greedy(est, batch):
    plan = plan_from_estimates(est, batch)
    b, e = greedy_reference(est, batch)
    assert plan.batches == b
    assert plan.estimated_pairs == e


def test_plan_rejects_bad_batch_size():
    with pytest.raises(ValidationError):
        plan_from_estimates([1, 2], 0)


@settings(max_examples=200, deadline=None)
@given(costs=st.lists(st.integers(1, 10**6), min_size=1, max_size=400), parts=st.integers(1, 9))
def test_balanced_cell_ranges_partition(costs, parts):
    ranges = balanced_cell_ranges(costs, parts)
    assert len(ranges) == parts
    assert ranges[0][0] == 0 and ranges[-1][1] == len(costs)
    for (a, b), (c, d) in zip(ranges, ranges[1:]):
        assert b == c and a <= b
    total = sum(costs)
    for a, b in ranges:  # each share within one cell of the ideal
        assert sum(costs[a:b]) <= total / parts + max(costs) + 1


@pytest.mark.parametrize("cfg", [
    JoinConfig(epsilon=0.0), JoinConfig(epsilon=float("nan")), JoinConfig(epsilon=0.1, kernel="simd"),
    JoinConfig(epsilon=0.1, batch_size=0), JoinConfig(epsilon=0.1, thread_count=0),
    JoinConfig(epsilon=0.1, k_idx=7), JoinConfig(epsilon=0.1, k_idx=0),
])
def test_config_validation_before_any_device_work(cfg):
    data = Dataset(np.random.default_rng(0).random((5, 6)))
    if cfg.k_idx == 7:
        data = Dataset(np.random.default_rng(0).random((5, 2)))
    with pytest.raises(ValidationError):
        self_join(data, cfg)


def test_dataset_validation_messages():
    with pytest.raises(ValidationError, match="point 2, dimension 3"):
        pts = np.zeros((4, 5))
        pts[2, 3] = np.inf
        Dataset(pts)
    with pytest.raises(ValidationError):
        Dataset(np.zeros(3))
    ds = Dataset([[1.0, 2.0, 3.0, 4.0, 5.0]])
    assert ds.d == 5 and ds.d_padded == 8 and ds.coords.shape == (1, 8)
    assert np.array_equal(ds.logical, [[1.0, 2.0, 3.0, 4.0, 5.0]])


def test_dataset_does_not_alias_input():
    src = np.random.default_rng(1).random((4, 4))
    ds = Dataset(src)
    src[0, 0] = 99.0
    assert ds.coords[0, 0] != 99.0


def test_cpu_only_box_fails_loudly():
    """No CPU fallback: without a CUDA device the product path raises."""
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    with pytest.raises(RuntimeError, match="CUDA"):
        self_join(Dataset(np.random.default_rng(0).random((10, 2))), JoinConfig(epsilon=0.1))


def test_abi_exports_every_declared_symbol():
    header = (ROOT / "include" / "tedjoin.h").read_text()
    declared = set(re.findall(r"\b(tj_[a-z0-9_]+)\s*\(", header))
    assert declared == set(_native.SIGNATURES), declared ^ set(_native.SIGNATURES)
    lib = _native.load_library()
    for name in declared:
        assert hasattr(lib, name), name
    assert lib.tj_version() >= 100


def test_abi_error_path_without_gpu():
    """tj_ctx_create on a box without a GPU returns an error status, not a crash."""
    import ctypes

    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    lib = _native.load_library()
    h = ctypes.c_void_p()
    st = lib.tj_ctx_create(0, ctypes.byref(h))
    assert st != _native.TJ_OK
    assert lib.tj_last_error(None)


def test_library_is_built_for_sm100a():
    import subprocess

    lib = _native.LIB_PATH
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_auto_kernel_dispatch():
    """kernel='auto' picks from measured throughput; DMMA wins at every measured d."""
    from paper_2209_11287_b200.join import resolve_kernel

    assert resolve_kernel("tile", 3) == "tile" and resolve_kernel("scalar", 3) == "scalar"
    assert all(resolve_kernel("auto", d) == "tile" for d in (1, 2, 4, 8, 16, 33, 64))
    assert resolve_kernel("auto", 65) == "scalar"
