"""Callers either side of the path: dataset files, the pairs
file writer, the CLI.  CPU tests need no GPU; the @gpu ones run the engine."""

import json
import struct

import numpy as np
import pytest

import oracle
from conftest import csr_equal
from paper_2209_11287_b200 import GenSpec, JoinConfig, ParseError, ValidationError, generate, self_join
from paper_2209_11287_b200 import _native, cli
from paper_2209_11287_b200.datasets import read_dataset, reorder_dims_by_variance, write_dataset


# ------------------------------------------------------------ dataset files (CPU)
@pytest.mark.parametrize("d", [1, 3, 4, 7])
@pytest.mark.parametrize("fmt", ["binary", "csv"])
def test_dataset_round_trip(tmp_path, d, fmt):  # test_datasets.py round trips
    ds = generate(GenSpec("exponential", 257, d, seed=5))
    p = tmp_path / "pts"
    write_dataset(ds, p, fmt)
    back = read_dataset(p)
    assert back.checksum() == ds.checksum()
    assert back.coords.shape == (257, 4 * ((d + 3) // 4))
    assert not back.coords[:, d:].any()


def test_binary_layout_is_reference_tedj(tmp_path):  # datasets.py:21-23,126-137
    ds = generate(GenSpec("uniform", 3, 2, seed=1))
    p = tmp_path / "a.bin"
    write_dataset(ds, p)
    raw = p.read_bytes()
    assert raw[:24] == struct.pack("<4sIQQ", b"TEDJ", 1, 3, 2)
    assert np.array_equal(np.frombuffer(raw[24:], "<f8").reshape(3, 2), ds.logical)


def test_binary_errors(tmp_path):  # datasets.py:158-176 messages
    p = tmp_path / "bad.bin"
    p.write_bytes(b"TEDJ\x01\x00")
    with pytest.raises(ParseError, match="truncated header"):
        read_dataset(p, "binary")
    p.write_bytes(struct.pack("<4sIQQ", b"NOPE", 1, 1, 1) + b"\0" * 8)
    with pytest.raises(ParseError, match="bad magic"):
        read_dataset(p, "binary")
    p.write_bytes(struct.pack("<4sIQQ", b"TEDJ", 2, 1, 1) + b"\0" * 8)
    with pytest.raises(ParseError, match="unsupported version 2"):
        read_dataset(p, "binary")
    p.write_bytes(struct.pack("<4sIQQ", b"TEDJ", 1, 2, 2) + b"\0" * 8)
    with pytest.raises(ParseError, match="expected 32 for n=2, d=2"):
        read_dataset(p, "binary")


def test_csv_errors(tmp_path):
    p = tmp_path / "bad.csv"
    p.write_text("1,2\n3\n")
    with pytest.raises(ValidationError, match="line 2 has 1 fields, expected 2"):
        read_dataset(p)
    p.write_text("1,x\n")
    with pytest.raises(ParseError, match="line 1"):
        read_dataset(p)
    p.write_text("\n\n")
    with pytest.raises(ParseError, match="no data rows"):
        read_dataset(p)


# --------------------------------------------------- pairs file writer (CPU, native)
def test_pairs_writer_matches_python_formatting(tmp_path):
    """tj_write_pairs == the reference's f"{i} {j} {s:.17g}" lines (cli.py:285-289)."""
    rng = np.random.default_rng(3)
    n = 50
    counts = rng.integers(0, 7, n)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.int64)
    m = int(off[-1])
    nb = rng.integers(0, n, m).astype(np.uint32)
    sq = np.concatenate([rng.random(m - 4) ** 3, [0.0, 1e-5, 1.0 / 3, 2.5e-310]])
    p = tmp_path / "pairs.txt"
    _native.write_pairs(p, off, nb, sq, threads=3)
    rows = np.repeat(np.arange(n), counts)
    want = "".join(f"{i} {j} {s:.17g}\n" for i, j, s in zip(rows.tolist(), nb.tolist(), sq.tolist()))
    assert p.read_text() == want


# ------------------------------------------------------------------- CLI (CPU)
def test_cli_generate_matches_generator(tmp_path, capsys):
    out = tmp_path / "g.bin"
    assert cli.main(["generate", "--dist", "expo", "--n", "300", "--d", "3", "--seed", "4",
                     "--out", str(out)]) == cli.EXIT_OK
    ds = generate(GenSpec("exponential", 300, 3, seed=4))
    assert read_dataset(out).checksum() == ds.checksum()
    assert ds.checksum() in capsys.readouterr().out


def test_cli_exit_codes_without_gpu(tmp_path):
    assert cli.main(["join"]) == cli.EXIT_USAGE
    assert cli.main(["join", "--input", str(tmp_path / "missing.bin"), "--epsilon", "0.1"]) == cli.EXIT_IO
    bad = tmp_path / "bad.csv"
    bad.write_text("1,2\n3\n")
    assert cli.main(["join", "--input", str(bad), "--epsilon", "0.1"]) == cli.EXIT_VALIDATION


def test_load_report_checks_version(tmp_path):
    p = tmp_path / "r.json"
    p.write_text(json.dumps({"format_version": 99}))
    with pytest.raises(ValidationError, match="unsupported report version"):
        cli.load_report(p)


# ------------------------------------------------------------------ GPU paths
@pytest.mark.gpu
def test_canonical_pair_sq_dists_and_pairs_file(tmp_path):
    from paper_2209_11287_b200.pairs import canonical_pair_sq_dists, write_pairs

    ds = generate(GenSpec("uniform", 3000, 5, seed=8))
    r = self_join(ds, JoinConfig(epsilon=0.2))
    sq = canonical_pair_sq_dists(ds, r)
    pr = r.pairs
    x = ds.logical
    acc = np.zeros(len(pr))  # cli._canonical_pair_sq_dists, restated
    for dim in range(ds.d):
        diff = x[pr[:, 0], dim] - x[pr[:, 1], dim]
        acc += diff * diff
    assert np.array_equal(sq, acc)
    p = tmp_path / "pairs.txt"
    write_pairs(ds, r, p)
    want = "".join(f"{i} {j} {s:.17g}\n" for (i, j), s in zip(pr.tolist(), acc.tolist()))
    assert p.read_text() == want


@pytest.mark.gpu
@pytest.mark.parametrize("d", [2, 5, 9])
def test_device_variance_order_matches_numpy(d):
    import torch

    from paper_2209_11287_b200.join import variance_order

    rng = np.random.default_rng(d)
    ds = generate(GenSpec("uniform", 20000, d, seed=d))
    ds.coords[:, :d] *= rng.random(d) * 3  # distinct column scales
    _, perm_ref = reorder_dims_by_variance(ds)
    ctx = _native.context(0)
    coords = torch.from_numpy(ds.coords).cuda()
    assert np.array_equal(variance_order(ctx, coords, ds), perm_ref)


@pytest.mark.gpu
@pytest.mark.parametrize("kernel", ["tile", "scalar"])
def test_reorder_dims_matches_reference(kernel):  # join.py:163-164, test_join.py:106-109
    """Device reordering == the reference's: the oracle on the host-reordered data."""
    ds = generate(GenSpec("exponential", 4000, 6, seed=3))
    ds.coords[:, 1] *= 0.1
    eps = 0.03
    b = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel, reorder_dims=True))
    work, _ = reorder_dims_by_variance(ds)
    off, nb = oracle.join_csr(work, eps)
    assert csr_equal(b.offsets, b.neighbors, off, nb)


@pytest.mark.gpu
def test_gpu_brute_force_equals_oracle():
    from paper_2209_11287_b200.verify import brute_force_join

    for spec, eps in [(GenSpec("uniform", 1500, 3, seed=1), 0.08),
                      (GenSpec("exponential", 1200, 9, seed=2), 0.02)]:
        ds = generate(spec)
        bf = brute_force_join(ds, eps, force=True)
        assert np.array_equal(bf.pairs, oracle.brute_force(ds, eps))


@pytest.mark.gpu
def test_gpu_brute_force_equals_join_config1():
    """Config 1 (uniform 2-D, n=100k) beyond the CPU oracle's 50k guard."""
    from paper_2209_11287_b200.verify import brute_force_join

    ds = generate(GenSpec("uniform", 100_000, 2, seed=0))
    eps = 0.0143667
    bf = brute_force_join(ds, eps, force=True)
    r = self_join(ds, JoinConfig(epsilon=eps))
    assert csr_equal(bf.offsets, bf.neighbors, r.offsets, r.neighbors)


@pytest.mark.gpu
def test_cli_join_verify_bench(tmp_path, capsys):
    pts = tmp_path / "p.bin"
    assert cli.main(["generate", "--dist", "uniform", "--n", "4000", "--d", "4", "--out",
                     str(pts)]) == 0
    rep = tmp_path / "r.json"
    pairs = tmp_path / "pairs.txt"
    assert cli.main(["join", "--input", str(pts), "--epsilon", "0.12", "--report", str(rep),
                     "--emit-pairs", str(pairs)]) == 0
    report = cli.load_report(rep)
    assert report["result"]["total_pairs"] == sum(1 for _ in open(pairs))
    assert cli.main(["join", "--input", str(pts), "--epsilon", "0.12", "--kernel", "scalar",
                     "--emit-pairs", str(tmp_path / "p2.txt")]) == 0
    assert (tmp_path / "p2.txt").read_bytes() == pairs.read_bytes()  # test_cli.py:87-97
    assert cli.main(["verify", "--input", str(pts), "--epsilon", "0.12"]) == 0
    assert "verify ok" in capsys.readouterr().out
    brep = tmp_path / "b.json"
    assert cli.main(["bench", "--input", str(pts), "--epsilons", "0.05,0.12", "--repeats", "1",
                     "--report", str(brep)]) == 0
    rows = cli.load_report(brep)["rows"]
    assert len(rows) == 4 and all(r["fp64_tflops"] > 0 for r in rows)


@pytest.mark.gpu
def test_cli_join_large_pinned_input(tmp_path, capsys):
    """an input above the 1 MB registration threshold read into pinned memory
    (read_dataset(pinned=True)) must not trip a stale CUDA error on re-registration;
    joins of views and repeated joins of the same pinned buffer stay exact."""
    pts = tmp_path / "big.bin"
    assert cli.main(["generate", "--dist", "uniform", "--n", "200000", "--d", "3", "--out",
                     str(pts)]) == 0
    capsys.readouterr()
    rep = tmp_path / "r.json"
    for _ in range(2):
        assert cli.main(["join", "--input", str(pts), "--epsilon", "0.01", "--report",
                         str(rep)]) == 0
    ds = read_dataset(pts, pinned=True)
    off, nb = oracle.join_csr(ds, 0.01)
    assert cli.load_report(rep)["result"]["total_pairs"] == int(off[-1])
    r = self_join(ds, JoinConfig(epsilon=0.01))
    assert csr_equal(r.offsets, r.neighbors, off, nb)
    half = ds.coords[: ds.n // 2]  # a view into the same pinned allocation
    from paper_2209_11287_b200 import Dataset

    view = Dataset._wrap(half, 3)
    r2 = self_join(view, JoinConfig(epsilon=0.01))
    o2, n2 = oracle.join_csr(view, 0.01)
    assert csr_equal(r2.offsets, r2.neighbors, o2, n2)


@pytest.mark.gpu
def test_pairs_expansion_is_fast():
    """JoinResult.pairs of config 2 (1.3e8 pairs) within a few hundred ms."""
    import time

    ds = generate(GenSpec("uniform", 2_000_000, 4, seed=0))
    r = self_join(ds, JoinConfig(epsilon=0.051306))
    t = time.perf_counter()
    p = r.pairs
    dt = time.perf_counter() - t
    assert p.shape == (r.total_pairs, 2)
    assert np.array_equal(p[:, 1], r.neighbors.astype(np.int64))
    print(f"pairs expansion {dt * 1e3:.1f} ms for {r.total_pairs} pairs")
    assert dt < 1.0
