"""CPU: pin the oracle (and the restated generator) to the reference's own outputs.

The fixtures in tests/golden were produced by importing the reference tilejoin
package (tests/golden/make_golden.py); nothing here reads /root/reference."""

import numpy as np
import pytest

import oracle
from conftest import load_json, sha_pairs
from paper_2209_11287_b200.datasets import Dataset, GenSpec, generate

SMALL_SPECS = [("uniform", 1000, 2, 17), ("exponential", 800, 3, 23),
               ("uniform", 600, 3, 77), ("exponential", 400, 8, 5)]


@pytest.mark.parametrize("spec", SMALL_SPECS, ids=lambda s: "%s_%d_%d_%d" % s)
def test_generator_matches_reference_small(spec, golden_generator):
    assert generate(GenSpec(*spec)).checksum() == golden_generator["%s_%d_%d_%d" % spec]["checksum"]


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4d2", "c4d8", "c4d16", "c4d32", "c4d64", "c5"])
def test_generator_matches_reference_bench_configs(name, golden_generator):
    g = golden_generator[name]
    assert generate(GenSpec(g["dist"], g["n"], g["d"], seed=0)).checksum() == g["checksum"]


def _ds(case):
    return generate(GenSpec(case["dist"], case["n"], case["d"], seed=case["seed"]))


def test_sweep_reference_consistency(golden_sweep):
    """The reference's own kernels agree on every sweep instance (pick_epsilon keeps
    pairs away from the shell), so one pair-set hash pins all three."""
    assert len(golden_sweep) == 60
    assert all(c["tile_equal"] and c["scalar_equal"] for c in golden_sweep)


def test_oracle_join_matches_reference_sweep(golden_sweep):
    for case in golden_sweep:
        ds = _ds(case)
        assert ds.checksum() == case["checksum"]
        off, nb = oracle.join_csr(ds, case["eps"])
        pairs = oracle.csr_to_pairs(off, nb)
        assert len(pairs) == case["pairs"]
        assert sha_pairs(pairs) == case["sha_pairs"], case


def test_numpy_brute_force_matches_reference(golden_sweep):
    for case in golden_sweep:
        if case["n"] != 500:
            continue
        ds = _ds(case)
        assert sha_pairs(oracle.brute_force(ds, case["eps"])) == case["sha_pairs"]


def test_oracle_grid_matches_reference(golden_sweep):
    for case in golden_sweep:
        ds = _ds(case)
        order, cstart, ccoord, cand = oracle.grid(ds, case["eps"])
        assert len(cstart) - 1 == case["n_cells"]
        assert sha_pairs(order.astype(np.int64)) == case["sha_point_order"]
        assert sha_pairs(ccoord) == case["sha_cells"]
        assert sha_pairs(cand) == case["sha_cand_counts"]
        assert sha_pairs(np.diff(cstart)) == case["sha_cell_sizes"]
        nq = np.diff(cstart)
        assert int(np.sum(-(-nq // 8) * -(-cand // 8))) == case["tiles"]
        assert int(np.sum(nq * cand)) == case["candidates"]


def test_oracle_config1_matches_reference():
    c1 = load_json("config1.json")
    ds = generate(GenSpec("uniform", 100_000, 2, seed=0))
    assert ds.checksum() == c1["checksum"]
    off, nb = oracle.join_csr(ds, c1["eps"])
    assert int(off[-1]) == c1["scalar"]["pairs"] == c1["tile"]["pairs"] == 6_502_052
    assert sha_pairs(oracle.csr_to_pairs(off, nb)) == c1["scalar"]["sha_pairs"]
    assert sha_pairs(np.diff(off)) == c1["scalar"]["sha_counts"]


def test_oracle_sampled_rows_match_reference():
    """Rows of sampled queries on the big configs, from the reference's own refiner."""
    try:
        metas = load_json("sampled.json")
    except FileNotFoundError:
        pytest.skip("sampled fixtures not generated")
    arr = np.load(oracle.HERE.parent / "tests" / "golden" / "sampled.npz")
    for meta in metas:
        if meta["n"] > 5_000_000:
            continue  # c5 is checked on the GPU box only (CPU suite stays fast)
        name = meta["config"]
        ds = generate(GenSpec(meta["dist"], meta["n"], meta["d"], seed=0))
        q, cnt, nbrs = arr[f"{name}_qids"], arr[f"{name}_counts"], arr[f"{name}_nbrs"]
        counts, got = oracle.rows(ds, meta["eps"], q)
        assert np.array_equal(counts, cnt), name
        assert np.array_equal(got.astype(np.int64), nbrs), name


def test_oracle_known_answers():
    # test_join.py:29-32 boundary inclusion, :35-40 identical points, :69-72 singleton
    off, nb = oracle.join_csr(Dataset([[0.0, 0.0], [0.25, 0.0]]), 0.25)
    assert oracle.csr_to_pairs(off, nb).tolist() == [[0, 0], [0, 1], [1, 0], [1, 1]]
    pts = np.tile(np.random.default_rng(2024).random(3), (30, 1))
    off, _ = oracle.join_csr(Dataset(pts), 0.1)
    assert off[-1] == 900
    off, nb = oracle.join_csr(Dataset([[0.5, 0.5]]), 0.1)
    assert oracle.csr_to_pairs(off, nb).tolist() == [[0, 0]]
    # kernels.py known answers: 3-4-5
    assert oracle.sqdist(Dataset([[0.0, 0.0], [3.0, 4.0]]), 0, 1) == 25.0


def test_digest_implementations_agree():
    """oracle_digest (C, streaming), tests/digest.py numpy and torch: one digest."""
    import torch

    from digest import csr_digest_numpy, csr_digest_torch, keys_digest_torch

    ds = generate(GenSpec("exponential", 3000, 3, seed=9))
    off, nb = oracle.join_csr(ds, 0.04)
    want = oracle.digest(ds, 0.04)
    got_np = csr_digest_numpy(off, nb)
    got_t = csr_digest_torch(torch.from_numpy(off), torch.from_numpy(nb.astype(np.int32)))
    assert got_t.pop("ascending")
    assert got_np == got_t == want
    keys = (oracle.csr_to_pairs(off, nb)[:, 0].astype(np.uint64) << np.uint64(32)) | nb.astype(np.uint64)
    kd = oracle.digest_keys(keys)
    assert kd == {k: want[k] for k in ("pairs", "s1", "s2")}
    assert keys_digest_torch(torch.from_numpy(keys.view(np.int64))) == kd


def test_full_digest_fixture_pinned_to_reference_config1():
    """full_digests.json's c1 entry is the digest of the reference's own config-1 pair set
    (config1.json SHA-256 of the reference self_join pairs)."""
    import json

    from digest import csr_digest_numpy

    full = json.loads((oracle.HERE.parent / "tests" / "golden" / "full_digests.json").read_text())
    c1 = load_json("config1.json")
    ds = generate(GenSpec("uniform", 100_000, 2, seed=0))
    off, nb = oracle.join_csr(ds, c1["eps"])
    assert sha_pairs(oracle.csr_to_pairs(off, nb)) == c1["scalar"]["sha_pairs"]
    dg = csr_digest_numpy(off, nb)
    for key in ("pairs", "s1", "s2", "max_row"):
        assert dg[key] == full["c1"][key]
    assert full["c2"]["pairs"] == 129_482_252 and full["c5"]["pairs"] == 3_524_665_904
