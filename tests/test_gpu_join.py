"""GPU parity: the CUDA self-join through libtedjoin.so vs the oracle and the
reference's own known answers (test_join.py cases restated, golden fixtures).

The bar is bit-exact pair sets: both kernels decide with the reference direct
form (the tile path re-decides guard-band pairs), so no epsilon-boundary
tolerance is needed."""

import math

import numpy as np
import pytest

import oracle
from conftest import csr_equal, load_json, sha_pairs
from paper_2209_11287_b200 import (
    Dataset,
    GenSpec,
    JoinConfig,
    ResourceError,
    ValidationError,
    generate,
    join_stats,
    selectivity,
    self_join,
)
from paper_2209_11287_b200 import grid as tgrid

pytestmark = pytest.mark.gpu
KERNELS = ("tile", "scalar")
ALL_KERNELS = ("tile", "scalar", "core_fma", "core_expanded")  # + the CUDA-core comparison variants


def assert_oracle_equal(res, ds, eps, k_idx=None):
    off, nb = oracle.join_csr(ds, eps, k_idx=k_idx)
    assert res.total_pairs == int(off[-1])
    assert csr_equal(res.offsets, res.neighbors, off, nb)


# --------------------------------------------------------- reference known answers


@pytest.mark.parametrize("kernel", KERNELS)
def test_boundary_distance_is_included(kernel):  # test_join.py:29-32
    r = self_join(Dataset([[0.0, 0.0], [0.25, 0.0]]), JoinConfig(epsilon=0.25, kernel=kernel))
    assert r.pairs.tolist() == [[0, 0], [0, 1], [1, 0], [1, 1]]


@pytest.mark.parametrize("kernel", KERNELS)
def test_identical_points_complete_graph(kernel):  # test_join.py:35-40
    rng = np.random.default_rng(2024)
    n = 30
    r = self_join(Dataset(np.tile(rng.random(3), (n, 1))), JoinConfig(epsilon=0.1, kernel=kernel))
    assert r.total_pairs == n * n
    assert r.selectivity == n - 1


@pytest.mark.parametrize("kernel", KERNELS)
def test_single_point(kernel):  # test_join.py:69-72
    r = self_join(Dataset([[0.5, 0.5]]), JoinConfig(epsilon=0.1, kernel=kernel))
    assert r.pairs.tolist() == [[0, 0]]
    assert r.selectivity == 0.0


@pytest.mark.parametrize("kernel", KERNELS)
def test_uniform_2d_matches_brute_force(kernel):  # test_join.py:43-49
    g = load_json("generator.json")
    ds = generate(GenSpec("uniform", 1000, 2, seed=17))
    assert ds.checksum() == g["uniform_1000_2_17"]["checksum"]
    eps = 0.0402  # fixed radius, parity against the restated brute force
    r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
    truth = oracle.brute_force(ds, eps)
    assert np.array_equal(r.pairs, truth)
    assert 4 < r.selectivity < 20


@pytest.mark.parametrize("kernel", KERNELS)
def test_self_pairs_and_symmetry(kernel):  # test_join.py:60-66
    ds = generate(GenSpec("uniform", 300, 4, seed=4))
    r = self_join(ds, JoinConfig(epsilon=0.3, kernel=kernel))
    p = r.pairs
    assert np.all(np.isin(np.arange(300), p[p[:, 0] == p[:, 1], 0]))
    fwd = set(map(tuple, p.tolist()))
    assert all((j, i) in fwd for i, j in fwd)


def test_selectivity_values():  # test_join.py:219-225
    r = self_join(Dataset(np.tile([0.1, 0.2], (100, 1))), JoinConfig(epsilon=0.5))
    assert selectivity(r, 100) == 99.0
    spread = Dataset(np.column_stack([np.arange(50.0), np.zeros(50)]))
    assert selectivity(self_join(spread, JoinConfig(epsilon=0.5)), 50) == 0.0


def test_capacity_guard_names_the_batch():  # test_join.py:169-172
    ds = generate(GenSpec("uniform", 300, 2, seed=12))
    with pytest.raises(ResourceError, match="batch 0"):
        self_join(ds, JoinConfig(epsilon=0.5), max_result_pairs=10)


def test_capacity_guard_later_batch():
    ds = generate(GenSpec("uniform", 2000, 2, seed=12))
    full = self_join(ds, JoinConfig(epsilon=0.05))
    cap = full.total_pairs // 2
    with pytest.raises(ResourceError, match=r"batch [1-9]"):
        self_join(ds, JoinConfig(epsilon=0.05, batch_size=500), max_result_pairs=cap)


def test_config_validation():  # test_join.py:239-250
    data = Dataset(np.random.default_rng(0).random((5, 2)))
    for cfg in (JoinConfig(epsilon=0.0), JoinConfig(epsilon=0.1, kernel="simd"),
                JoinConfig(epsilon=0.1, batch_size=0), JoinConfig(epsilon=0.1, thread_count=0),
                JoinConfig(epsilon=0.1, k_idx=7)):
        with pytest.raises(ValidationError):
            self_join(data, cfg)


# -------------------------------------------------------------- invariances


@pytest.fixture(scope="module")
def case600():
    ds = generate(GenSpec("uniform", 600, 3, seed=77))
    eps = 0.0731
    return ds, eps, self_join(ds, JoinConfig(epsilon=eps))


@pytest.mark.parametrize("cfg", [
    dict(short_circuit=False), dict(batch_size=1), dict(batch_size=64), dict(thread_count=4),
    dict(reorder_dims=True), dict(k_idx=1), dict(k_idx=2), dict(k_idx=3), dict(kernel="scalar"),
    dict(kernel="scalar", short_circuit=False), dict(kernel="scalar", batch_size=7),
])
def test_knobs_do_not_change_pairs(case600, cfg):  # test_join.py:78-127
    ds, eps, base = case600
    r = self_join(ds, JoinConfig(epsilon=eps, **cfg))
    assert np.array_equal(r.pairs, base.pairs)
    assert_oracle_equal(base, ds, eps)


def test_epsilon_monotonicity():  # test_join.py:112-120
    ds = generate(GenSpec("uniform", 400, 2, seed=31))
    small = self_join(ds, JoinConfig(epsilon=0.02))
    large = self_join(ds, JoinConfig(epsilon=0.08))
    s = set(map(tuple, small.pairs.tolist()))
    assert s <= set(map(tuple, large.pairs.tolist()))


# -------------------------------------------------------------------- stats


def test_stats_counters_recount_from_index():  # test_join.py:178-216
    ds = generate(GenSpec("uniform", 500, 6, seed=13))
    eps = 0.2
    r = self_join(ds, JoinConfig(epsilon=eps))
    _, cstart, _, cand = oracle.grid(ds, eps, 6)
    nq = np.diff(cstart)
    tiles = int(np.sum(-(-nq // 8) * -(-cand // 8)))
    st = join_stats(r)
    assert st.tiles_processed == tiles
    assert st.candidates_refined == int(np.sum(nq * cand))
    assert st.chunks_executed + st.chunks_skipped == tiles * 2
    assert st.pairs_emitted == r.total_pairs
    assert st.total_seconds >= st.index_seconds


def test_stats_no_short_circuit_means_no_skips():
    ds = generate(GenSpec("exponential", 400, 8, seed=5))
    assert self_join(ds, JoinConfig(epsilon=0.02, short_circuit=False)).stats.chunks_skipped == 0


def test_short_circuit_skips_chunks():  # test_cli.py:100-117 shape: 300 pts in [0,0.05)^8
    rng = np.random.default_rng(3)
    ds = Dataset(rng.random((300, 8)) * 0.05)
    on = self_join(ds, JoinConfig(epsilon=0.01, short_circuit=True))
    off = self_join(ds, JoinConfig(epsilon=0.01, short_circuit=False))
    assert on.stats.chunks_skipped > 0
    assert np.array_equal(on.pairs, off.pairs)


def test_scalar_kernel_reports_no_tiles():  # join.py:328
    ds = generate(GenSpec("uniform", 200, 3, seed=1))
    st = self_join(ds, JoinConfig(epsilon=0.2, kernel="scalar")).stats
    assert st.tiles_processed == 0 and st.chunks_executed == 0


# --------------------------------------------------------- golden SPEC sweep


def _sweep_cases():
    try:
        return load_json("sweep.json")
    except FileNotFoundError:
        return []


@pytest.mark.parametrize("case", _sweep_cases(), ids=lambda c: f"{c['dist'][:3]}-n{c['n']}-d{c['d']}-S{c['target']}")
@pytest.mark.parametrize("kernel", ALL_KERNELS)
def test_spec_sweep_matches_reference(case, kernel):
    ds = generate(GenSpec(case["dist"], case["n"], case["d"], seed=case["seed"]))
    assert ds.checksum() == case["checksum"]
    r = self_join(ds, JoinConfig(epsilon=case["eps"], kernel=kernel))
    assert r.total_pairs == case["pairs"]
    assert sha_pairs(r.pairs) == case["sha_pairs"]
    if kernel == "tile":
        assert r.stats.tiles_processed == case["tiles"]
    assert r.stats.candidates_refined == case["candidates"]


def test_config1_full_pair_set():
    c1 = load_json("config1.json")
    ds = generate(GenSpec("uniform", 100_000, 2, seed=0))
    assert ds.checksum() == c1["checksum"]
    for kernel in KERNELS:
        r = self_join(ds, JoinConfig(epsilon=c1["eps"], kernel=kernel))
        assert r.total_pairs == c1["scalar"]["pairs"] == 6_502_052
        assert sha_pairs(r.pairs) == c1["scalar"]["sha_pairs"]
        assert r.stats.candidates_refined == c1["scalar"]["candidates"]


def _sampled():
    try:
        return load_json("sampled.json")
    except FileNotFoundError:
        return []


@pytest.mark.parametrize("meta", _sampled(), ids=lambda m: m["config"])
def test_full_size_configs_match_reference_rows(meta):
    """Benchmark-size inputs: rows of queries sampled from the 10 costliest cells plus
    random cells, as computed by the reference's own refiner (tests/golden)."""
    arr = np.load(oracle.HERE.parent / "tests" / "golden" / "sampled.npz")
    name = meta["config"]
    ds = generate(GenSpec(meta["dist"], meta["n"], meta["d"], seed=0))
    assert ds.checksum() == meta["checksum"]
    r = self_join(ds, JoinConfig(epsilon=meta["eps"]))
    q, cnt, nbrs = arr[f"{name}_qids"], arr[f"{name}_counts"], arr[f"{name}_nbrs"]
    pos = 0
    for qq, c in zip(q, cnt):
        row = r.neighbors_of(int(qq)).astype(np.int64)
        assert len(row) == c, (name, int(qq))
        assert np.array_equal(row, nbrs[pos: pos + c]), (name, int(qq))
        pos += c
    # size-independent invariants of the whole pair set: self-pairs, sorted rows,
    # symmetry through a checksum of (i, j) vs (j, i) sums
    counts = np.diff(r.offsets)
    assert (counts >= 1).all()
    rows = np.repeat(np.arange(len(counts), dtype=np.int64), counts)
    nb = r.neighbors.astype(np.int64)
    assert (np.diff(nb)[np.diff(rows) == 0] > 0).all()
    h1 = np.bitwise_xor.reduce(rows * 1_000_003 + nb * 7919)
    h2 = np.bitwise_xor.reduce(nb * 1_000_003 + rows * 7919)
    assert h1 == h2


# ------------------------------------------------------------------- grid


def test_grid_matches_reference_layout(golden_sweep):
    for case in golden_sweep[::7]:
        ds = generate(GenSpec(case["dist"], case["n"], case["d"], seed=case["seed"]))
        idx = tgrid.build_index(ds, case["eps"])
        assert idx.n_cells == case["n_cells"]
        assert sha_pairs(idx.point_order) == case["sha_point_order"]
        assert sha_pairs(np.asarray(idx.ordered_cells, dtype=np.int64)) == case["sha_cells"]
        assert sha_pairs(idx.cell_cands) == case["sha_cand_counts"]


def test_grid_floor_and_negative_coords():  # test_grid.py:16-37
    idx = tgrid.build_index(Dataset([[0.05, 0.05], [0.15, 0.05]]), 0.1, 2)
    assert set(idx.cells) == {(0, 0), (1, 0)}
    idx = tgrid.build_index(Dataset([[-0.05], [-0.15], [0.05]]), 0.1, 1)
    assert set(idx.cells) == {(-1,), (-2,), (0,)}
    idx = tgrid.build_index(Dataset([[1.0], [0.99]]), 0.5, 1)
    assert idx.cells[(2,)].tolist() == [0] and idx.cells[(1,)].tolist() == [1]


def test_grid_candidates_match_oracle():
    rng = np.random.default_rng(99)
    for d, k in [(2, 2), (4, 3), (6, 4), (3, 1)]:
        ds = Dataset(rng.normal(size=(500, d)))
        eps = 0.35
        idx = tgrid.build_index(ds, eps, k)
        order, cstart, ccoord, cand = oracle.grid(ds, eps, k)
        assert np.array_equal(idx.point_order, order.astype(np.int64))
        assert [tuple(c) for c in ccoord.tolist()] == idx.ordered_cells
        assert np.array_equal(idx.cell_cands, cand)
        for c in idx.ordered_cells[:20]:
            got = tgrid.neighbor_cells(idx, c)
            expect = sorted(x for x in idx.cells if max(abs(a - b) for a, b in zip(x, c)) <= 1)
            assert got == expect


def _wide_key_dataset():
    """6-D points whose cell key needs > 63 bits (a far cluster stretches
    every indexed dim to ~14 bits): the device grid packs two words."""
    rng = np.random.default_rng(11)
    x = rng.random((4000, 6)) * 0.6
    x[:7] += 1e3
    x[7:11] -= 1e3
    return Dataset(x)


def test_wide_cell_keys_grid_matches_oracle():
    ds, eps = _wide_key_dataset(), 0.12
    idx = tgrid.build_index(ds, eps, 6)
    order, cstart, ccoord, cand = oracle.grid(ds, eps, 6)
    assert np.array_equal(idx.point_order, order.astype(np.int64))
    assert [tuple(c) for c in ccoord.tolist()] == idx.ordered_cells
    assert np.array_equal(idx.cell_cands, cand)


@pytest.mark.parametrize("kernel", ALL_KERNELS)
def test_wide_cell_keys_join(kernel):
    ds, eps = _wide_key_dataset(), 0.12
    r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, k_idx=6))
    assert_oracle_equal(r, ds, eps, k_idx=6)
    s = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, k_idx=5))  # 75 bits over 5 dims
    assert_oracle_equal(s, ds, eps, k_idx=5)


# -------------------------------------------------------------- edge cases


@pytest.mark.parametrize("d", [1, 2, 3, 4, 5, 7, 8, 9, 12, 16, 17, 24, 33, 64])
@pytest.mark.parametrize("kernel", ALL_KERNELS)
def test_dimensionality_ladder(d, kernel):
    ds = generate(GenSpec("uniform", 1500, d, seed=d))
    eps = 0.12 * math.sqrt(d)
    r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
    assert_oracle_equal(r, ds, eps)


@pytest.mark.parametrize("kernel", KERNELS)
def test_skewed_big_cell_and_long_rows(kernel):
    """Exponential data: cells far larger than one work item, rows > 256 and > 8192 ids."""
    ds = generate(GenSpec("exponential", 60_000, 3, seed=3))
    eps = 0.016
    r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
    assert_oracle_equal(r, ds, eps)
    assert np.diff(r.offsets).max() > 8192


@pytest.mark.parametrize("kernel", KERNELS)
def test_duplicates_and_exact_shell(kernel):
    """Coincident points and pairs exactly on the eps shell (guard-band rechecks)."""
    base = np.array([[0.0, 0.0, 0.0], [0.25, 0.0, 0.0], [0.0, 0.25, 0.0], [0.1, 0.1, 0.1]])
    pts = np.vstack([base] * 40 + [base + 1.0] * 3)
    ds = Dataset(pts)
    r = self_join(ds, JoinConfig(epsilon=0.25, kernel=kernel))
    assert_oracle_equal(r, ds, 0.25)


@pytest.mark.parametrize("kernel", KERNELS)
def test_far_from_origin(kernel):
    """Large coordinates make the expanded form cancel badly: all decisions must still be exact."""
    rng = np.random.default_rng(5)
    ds = Dataset(1e4 + rng.random((3000, 4)))
    eps = 0.09
    r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
    assert_oracle_equal(r, ds, eps)


def test_reference_dataset_object_is_accepted():
    ds = generate(GenSpec("uniform", 500, 3, seed=2))

    class Foreign:  # duck-typed tilejoin.datasets.Dataset
        def __init__(self, d):
            self.coords, self.d, self.n, self.d_padded = d.coords, d.d, d.n, d.d_padded

        @property
        def logical(self):
            return self.coords[:, : self.d]

    r1 = self_join(Foreign(ds), JoinConfig(epsilon=0.1))
    r2 = self_join(ds.logical.copy(), JoinConfig(epsilon=0.1))
    assert np.array_equal(r1.pairs, r2.pairs)


@pytest.mark.parametrize("d", [2, 4])
def test_batches_on_the_mask_path(d):
    """Several refine batches into one low-d mask result set (join.py:184-197)."""
    ds = generate(GenSpec("uniform", 20_000, d, seed=11))
    eps = 0.02 if d == 2 else 0.12
    one = self_join(ds, JoinConfig(epsilon=eps))
    est = int(one.stats.candidates_refined)
    many = self_join(ds, JoinConfig(epsilon=eps, batch_size=max(est // 7, 1)))
    assert csr_equal(one.offsets, one.neighbors, many.offsets, many.neighbors)
    assert_oracle_equal(many, ds, eps)


@pytest.mark.parametrize("k_idx", [1, 2, 3])
@pytest.mark.parametrize("kernel", KERNELS)
def test_fewer_indexed_dims(k_idx, kernel):
    """k_idx < d: longer candidate lists, same pair set (grid.py:79-80)."""
    ds = generate(GenSpec("uniform", 6000, 4, seed=k_idx))
    eps = 0.1
    r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, k_idx=k_idx))
    assert_oracle_equal(r, ds, eps, k_idx=k_idx)


def test_tiny_cells_many_cells_per_window():
    """Cells of ~1 point: 32-row emit windows span more cells than the staged tables."""
    ds = generate(GenSpec("uniform", 50_000, 3, seed=6))
    eps = 0.012
    r = self_join(ds, JoinConfig(epsilon=eps))
    assert_oracle_equal(r, ds, eps)


def test_long_candidate_lists_low_d():
    """2-D cells of ~400 points: candidate lists beyond the emit's per-block run hints."""
    ds = generate(GenSpec("uniform", 200_000, 2, seed=8))
    eps = 0.045
    r = self_join(ds, JoinConfig(epsilon=eps))
    assert_oracle_equal(r, ds, eps)


def test_auto_kernel_matches():
    ds = generate(GenSpec("uniform", 3000, 5, seed=12))
    eps = 0.2
    r = self_join(ds, JoinConfig(epsilon=eps, kernel="auto"))
    assert_oracle_equal(r, ds, eps)
    assert r.stats.tiles_processed > 0  # the DMMA path ran


@pytest.mark.parametrize("sc", [True, False])
def test_big_cells_high_d_32_query_items(sc):
    """d = 8 with ~64 points per cell: the high-d DMMA kernel's 32-query items."""
    ds = generate(GenSpec("uniform", 60_000, 8, seed=21))
    eps = 0.32
    r = self_join(ds, JoinConfig(epsilon=eps, short_circuit=sc))
    assert_oracle_equal(r, ds, eps)


@pytest.mark.parametrize("d,kernel", [(3, "tile"), (8, "tile"), (3, "scalar")])
def test_split_finalize_matches_one_call(d, kernel):
    """tj_finalize_offsets + tj_finalize_rows (what self_join uses) == tj_finalize."""
    from paper_2209_11287_b200.join import DeviceJoin

    ds = generate(GenSpec("uniform", 8000, d, seed=4))
    eps = 0.08 if d == 3 else 0.5
    job = DeviceJoin(ds, JoinConfig(epsilon=eps, kernel=kernel), device=0)
    job.build()
    job.refine()
    off_a, nbr_a = job.finalize_fetch()
    job.finalize()
    off_b, nbr_b = job.fetch()
    assert np.array_equal(off_a, off_b) and np.array_equal(nbr_a, nbr_b)
    off, nb = oracle.join_csr(ds, eps)
    assert csr_equal(off_a, nbr_a, off, nb)


@pytest.mark.parametrize("chunks,copies", [(1, None), (5, None), (16, None), (32, (1, 2, 4, 8, 17)),
                                           (7, (3, 4))])
def test_result_pipeline_schedules(chunks, copies):
    """Any id-range split and D2H copy grouping of the result pipeline gives the same CSR."""
    from paper_2209_11287_b200.join import DeviceJoin

    ds = generate(GenSpec("uniform", 20000, 3, seed=8))
    eps = 0.06
    job = DeviceJoin(ds, JoinConfig(epsilon=eps), device=0)
    job.build()
    job.refine()
    off_a, nbr_a = job.finalize_fetch(chunks=chunks, copies=copies)
    job.finalize()
    off_b, nbr_b = job.fetch()
    assert np.array_equal(off_a, off_b) and np.array_equal(nbr_a, nbr_b)


@pytest.mark.parametrize("kernel", ALL_KERNELS)
@pytest.mark.parametrize("d", [2, 3, 4, 8])
def test_lattice_boundary_pairs(kernel, d):
    """A lattice at spacing eps: every axis neighbour sits exactly on the boundary (in
    exact arithmetic) and rounding decides -- the guard band / recheck path of every
    non-exact kernel must reproduce the reference direct-form decisions."""
    side = {2: 40, 3: 12, 4: 6, 8: 3}[d]
    axes = np.meshgrid(*[np.arange(side) * 0.1 + 0.3] * d, indexing="ij")
    pts = np.stack([a.reshape(-1) for a in axes], axis=1)
    ds = Dataset(pts)
    for eps in (0.1, 0.1 * math.sqrt(2), 0.2):
        r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
        assert_oracle_equal(r, ds, eps)


@pytest.mark.parametrize("n,d,k_idx,eps", [
    (3000, 12, 1, 0.788),    # 2 cells of ~1500: Gram items with partial query blocks
    (2500, 16, 2, 0.55),     # 4 cells, ~1 neighbour per point
    (2500, 16, 1, 1.051),    # one cell, ~29 neighbours per point
    (1700, 33, 1, 1.792),    # one cell, d_pad = 36
    (1300, 64, 1, 2.759),    # one cell, NCH = 16
    (40000, 12, 1, 0.609),   # > one 32k-candidate slice per item
])
@pytest.mark.parametrize("kernel", ["tile", "core_expanded"])
def test_gram_kernel_big_cells(n, d, k_idx, eps, kernel):
    """Big cells at d_pad >= 12 take the CTA-blocked Gram kernels (refine_gram.cu): DMMA
    for "tile", the same blocking in DFMA for "core_expanded".  Pair set, tile count and
    candidate count equal the oracle's / the reference formula."""
    ds = generate(GenSpec("uniform", n, d, seed=n + d))
    r = self_join(ds, JoinConfig(epsilon=eps, k_idx=k_idx, kernel=kernel))
    assert_oracle_equal(r, ds, eps, k_idx=k_idx)
    _, cstart, _, cand = oracle.grid(ds, eps, k_idx)
    nq = np.diff(cstart)
    assert r.stats.candidates_refined == int(np.sum(nq * cand))
    if kernel == "tile":
        tiles = int(np.sum(-(-nq // 8) * -(-cand // 8)))
        assert r.stats.tiles_processed == tiles
        assert r.stats.chunks_executed + r.stats.chunks_skipped == tiles * ((d + 3) // 4)
    else:
        assert r.stats.tiles_processed == 0


# ------------------------------------------------------ output-budget batcher
@pytest.mark.parametrize("kernel", ["scalar", "core_fma", "tile"])
def test_pair_buffer_overflow_rolls_back_and_regrows(kernel, monkeypatch):
    """A pair buffer far too small for the result (estimate forced to 1): every
    overflowing batch is rolled back, the buffer grows to the exact count keeping the
    earlier batches' pairs, and the batch re-runs -- the pair set is exact, the stats
    count each batch once."""
    from paper_2209_11287_b200.join import DeviceJoin

    ds = generate(GenSpec("uniform", 6000, 5, seed=3))
    eps = 0.12
    want = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
    monkeypatch.setattr(DeviceJoin, "estimate_pairs", lambda self, batches, costs=None: 1)
    for batch_size in (None, 2000, 50_000):
        r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, batch_size=batch_size),
                      max_result_pairs=10**9)
        assert_oracle_equal(r, ds, eps)
        assert r.stats.candidates_refined == want.stats.candidates_refined
        assert r.stats.tiles_processed == want.stats.tiles_processed


def test_small_join_then_large_batched_join_with_cap():
    """a large batched join after a small one on the same context, with
    max_result_pairs set, must not fail on the buffer the small join left behind."""
    small = generate(GenSpec("uniform", 200, 6, seed=1))
    self_join(small, JoinConfig(epsilon=0.2, kernel="scalar"))
    ds = generate(GenSpec("uniform", 20_000, 6, seed=2))
    eps = 0.15
    r = self_join(ds, JoinConfig(epsilon=eps, kernel="scalar", batch_size=100_000),
                  max_result_pairs=10**9)
    assert_oracle_equal(r, ds, eps)


def test_pair_estimate_is_close_for_uniform_data():
    """tj_estimate_pairs (sampled, nothing stored) brackets the exact count: the buffer
    it sizes holds the result without a re-run and without gross over-allocation."""
    from paper_2209_11287_b200.join import DeviceJoin

    for kernel, (n, d, eps) in (("scalar", (1_000_000, 4, 0.065)), ("tile", (600_000, 8, 0.3)),
                                ("core_fma", (1_000_000, 4, 0.065))):
        ds = generate(GenSpec("uniform", n, d, seed=4))
        job = DeviceJoin(ds, JoinConfig(epsilon=eps, kernel=kernel))
        job.build()
        assert job.info.candidates > DeviceJoin.SAMPLE_ABOVE
        est = job.estimate_pairs([(0, job.info.n_cells)])
        total = job.refine()
        assert total <= est <= 2 * total, (kernel, total, est)
        r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
        assert r.total_pairs == total


# ------------------------------------------------ low-d symmetric join (option)
@pytest.mark.parametrize("case", _sweep_cases()[::3], ids=lambda c: f"{c['dist'][:3]}-n{c['n']}-d{c['d']}-S{c['target']}")
def test_symmetric_join_matches_reference(case, monkeypatch):
    """TJ_SYMMETRIC=1: every neighbour-cell pair multiplied once, rows completed from
    the earlier cells' masks -- the same pair set (golden SHA-256) in one batch and in
    many, through both the device finalize and the chunked host pipeline."""
    monkeypatch.setenv("TJ_SYMMETRIC", "1")
    ds = generate(GenSpec(case["dist"], case["n"], case["d"], seed=case["seed"]))
    for batch in (None, 64):
        r = self_join(ds, JoinConfig(epsilon=case["eps"], batch_size=batch))
        assert r.total_pairs == case["pairs"]
        assert sha_pairs(r.pairs) == case["sha_pairs"]
        if case["d"] <= 4:
            assert r.stats.tiles_processed == case["tiles"]


@pytest.mark.parametrize("d", [2, 3, 4])
def test_symmetric_join_shard_ranges(d, monkeypatch):
    """A cell range past cell 0 (multi-GPU shard): the earlier cells are refined for
    their masks only (tj_refine_masks); the range's rows equal the full join's."""
    from paper_2209_11287_b200.join import DeviceJoin

    monkeypatch.setenv("TJ_SYMMETRIC", "1")
    ds = generate(GenSpec("uniform", 20_000, d, seed=d))
    eps = {2: 0.01, 3: 0.04, 4: 0.08}[d]
    full_off, full_nb = oracle.join_csr(ds, eps)
    job = DeviceJoin(ds, JoinConfig(epsilon=eps))
    info = job.build()
    lo, hi = info.n_cells // 3, 2 * info.n_cells // 3
    job.refine(cell_range=(lo, hi))
    off, nb = job.finalize_fetch()
    _, cstart, _, _ = oracle.grid(ds, eps)
    order = oracle.grid(ds, eps)[0]
    ids = order[cstart[lo]: cstart[hi]].astype(np.int64)
    for i in ids[:: max(1, len(ids) // 300)]:
        assert np.array_equal(nb[off[i]: off[i + 1]].astype(np.int64),
                              full_nb[full_off[i]: full_off[i + 1]].astype(np.int64)), i
    assert int(off[-1]) == int(sum(full_off[i + 1] - full_off[i] for i in ids))


def test_symmetric_join_full_size_c2(monkeypatch):
    from test_gpu_parity import FULL, _check, device_digest

    if "c2" not in FULL:
        pytest.skip("oracle digest not generated")
    monkeypatch.setenv("TJ_SYMMETRIC", "1")
    _check(device_digest(FULL["c2"], "tile"), FULL["c2"])
