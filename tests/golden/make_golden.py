"""Generate the golden fixtures from the reference itself (run in the build container).

    PYTHONPATH=/root/reference/pkg/src:/root/reference/pkg/tests python tests/golden/make_golden.py

Imports the reference `tilejoin` package and its test helper `pick_epsilon`
(read-only, never copied) and writes:

  generator.json  Dataset.checksum() of every input the tests and bench use
                  (pins paper_2209_11287_b200.datasets.generate);
  sweep.json      SPEC acceptance sweep: n in {500, 2000} x d in
                  {2,3,4,6,8} x {uniform, exponential} x 3 selectivities, with
                  reference brute_force_join, self_join(tile) and
                  self_join(scalar) pair counts + SHA-256 of the (m,2) int64
                  pairs, plus grid summaries from build_index;
  config1.json    config 1 (uniform 2-D, N=100k, eps=0.0143667) full pair-set
                  hashes from the reference self_join (scalar and tile);
  sampled.npz /
  sampled.json    configs 2-5: rows of sampled queries (the 10 costliest cells
                  plus seeded random cells) computed by the reference's own
                  build_index -> candidates_for_cell -> _ScalarRefiner.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent

from conftest import pick_epsilon, sorted_pair_distances  # reference tests/conftest.py
from tilejoin.datasets import GenSpec, generate
from tilejoin.grid import build_index, candidates_for_cell
from tilejoin.join import JoinConfig, _ScalarRefiner, self_join
from tilejoin.oracle import brute_force_join

CONFIGS = {
    "c1": ("uniform", 100_000, 2, 0.0143667),
    "c2": ("uniform", 2_000_000, 4, 0.051306),
    "c3": ("exponential", 5_000_000, 8, 0.0118508),
    "c4d2": ("uniform", 2_000_000, 2, 0.00320714),
    "c4d8": ("uniform", 2_000_000, 8, 0.244686),
    "c4d16": ("uniform", 2_000_000, 16, 0.657508),
    "c4d32": ("uniform", 2_000_000, 32, 1.31923),
    "c4d64": ("uniform", 2_000_000, 64, 2.27218),
    "c5": ("uniform", 50_000_000, 4, 0.0232204),
}


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<i8").tobytes()).hexdigest()


def sweep():
    out = []
    for n in (500, 2000):
        for d in (2, 3, 4, 6, 8):
            for dist in ("uniform", "exponential"):
                seed = 1000 * d + n + (7 if dist == "exponential" else 0)
                ds = generate(GenSpec(dist, n, d, seed=seed))
                dist_sorted = sorted_pair_distances(ds)
                for target in (2, 10, 30):
                    eps = pick_epsilon(dist_sorted, n, target)
                    truth = brute_force_join(ds, eps)
                    tile = self_join(ds, JoinConfig(epsilon=eps, kernel="tile"))
                    scal = self_join(ds, JoinConfig(epsilon=eps, kernel="scalar"))
                    idx = build_index(ds, eps)
                    cand = [len(candidates_for_cell(idx, c)) for c in idx.ordered_cells]
                    sizes = [len(idx.cells[c]) for c in idx.ordered_cells]
                    out.append({
                        "dist": dist, "n": n, "d": d, "seed": seed, "target": target,
                        "eps": eps, "checksum": ds.checksum(),
                        "pairs": int(len(truth.pairs)), "sha_pairs": sha(truth.pairs),
                        "tile_equal": bool(np.array_equal(tile.pairs, truth.pairs)),
                        "scalar_equal": bool(np.array_equal(scal.pairs, truth.pairs)),
                        "tiles": int(tile.stats.tiles_processed),
                        "candidates": int(tile.stats.candidates_refined),
                        "n_cells": idx.n_cells,
                        "sha_point_order": sha(idx.point_order),
                        "sha_cells": sha(np.asarray(idx.ordered_cells, dtype=np.int64)),
                        "sha_cand_counts": sha(np.asarray(cand, dtype=np.int64)),
                        "sha_cell_sizes": sha(np.asarray(sizes, dtype=np.int64)),
                    })
                    print(f"sweep {dist} n={n} d={d} S={target}: {len(truth.pairs)} pairs", flush=True)
    return out


def config1():
    dist, n, d, eps = CONFIGS["c1"]
    ds = generate(GenSpec(dist, n, d, seed=0))
    res = {"checksum": ds.checksum(), "eps": eps}
    for kernel in ("scalar", "tile"):
        t = time.perf_counter()
        r = self_join(ds, JoinConfig(epsilon=eps, kernel=kernel))
        res[kernel] = {
            "pairs": int(r.total_pairs), "sha_pairs": sha(r.pairs),
            "sha_counts": sha(np.bincount(r.pairs[:, 0], minlength=n)),
            "tiles": int(r.stats.tiles_processed), "candidates": int(r.stats.candidates_refined),
            "seconds": time.perf_counter() - t,
        }
        print("config1", kernel, res[kernel], flush=True)
    idx = build_index(ds, eps)
    res["n_cells"] = idx.n_cells
    res["sha_point_order"] = sha(idx.point_order)
    return res


def sampled(name, n_random=10, q_per_cell=12, seed=0):
    dist, n, d, eps = CONFIGS[name]
    ds = generate(GenSpec(dist, n, d, seed=0))
    t = time.perf_counter()
    idx = build_index(ds, eps)
    sizes = np.array([len(idx.cells[c]) for c in idx.ordered_cells], dtype=np.int64)
    rng = np.random.default_rng(seed)
    # cost needs |cand|: exact for a candidate shortlist (largest cells), estimate elsewhere
    big = np.argsort(-sizes, kind="stable")[: 50]
    cand_big = np.array([len(candidates_for_cell(idx, idx.ordered_cells[i])) for i in big])
    costliest = big[np.argsort(-(sizes[big] * cand_big), kind="stable")[:10]]
    randoms = rng.choice(len(sizes), size=min(n_random, len(sizes)), replace=False)
    cells = list(dict.fromkeys([int(c) for c in costliest] + [int(c) for c in randoms]))
    refiner = _ScalarRefiner(ds, eps * eps, short_circuit=True)
    qids_all, counts, nbrs = [], [], []
    for ci in cells:
        cell = idx.ordered_cells[ci]
        members = idx.cells[cell]
        q = members if len(members) <= q_per_cell else np.sort(
            rng.choice(members, size=q_per_cell, replace=False))
        cands = candidates_for_cell(idx, cell)
        out = refiner(np.asarray(q, dtype=np.int64), cands)
        pairs = out.pairs[np.lexsort((out.pairs[:, 1], out.pairs[:, 0]))]
        for qq in q:
            row = pairs[pairs[:, 0] == qq, 1]
            qids_all.append(int(qq))
            counts.append(len(row))
            nbrs.append(row)
    meta = {
        "config": name, "dist": dist, "n": n, "d": d, "eps": eps, "checksum": ds.checksum(),
        "n_cells": idx.n_cells, "cells": cells, "seconds": time.perf_counter() - t,
        "sha_point_order": sha(idx.point_order),
    }
    print("sampled", name, meta["n_cells"], len(qids_all), "queries", meta["seconds"], flush=True)
    return meta, np.asarray(qids_all, np.int64), np.asarray(counts, np.int64), (
        np.concatenate(nbrs).astype(np.int64) if nbrs else np.zeros(0, np.int64))


SAMPLED = ("c2", "c3", "c4d2", "c4d8", "c4d16", "c4d32", "c4d64", "c5")


def main(argv):
    which = set(argv[1:]) or {"generator", "sweep", "config1", "sampled"}
    # "sampled:c4d2,c4d32" regenerates only those configs' rows, keeping the rest
    only = [w.split(":", 1)[1].split(",") for w in which if w.startswith("sampled:")]
    if only:
        which.add("sampled")
    if "generator" in which:
        gen = {}
        for name, (dist, n, d, eps) in CONFIGS.items():
            gen[name] = {"dist": dist, "n": n, "d": d, "eps": eps,
                         "checksum": generate(GenSpec(dist, n, d, seed=0)).checksum()}
            print("generator", name, flush=True)
        for spec in [("uniform", 1000, 2, 17), ("exponential", 800, 3, 23),
                     ("uniform", 600, 3, 77), ("exponential", 400, 8, 5)]:
            key = "%s_%d_%d_%d" % spec
            gen[key] = {"checksum": generate(GenSpec(*spec)).checksum()}
        (HERE / "generator.json").write_text(json.dumps(gen, indent=1))
    if "sweep" in which:
        (HERE / "sweep.json").write_text(json.dumps(sweep(), indent=1))
    if "config1" in which:
        (HERE / "config1.json").write_text(json.dumps(config1(), indent=1))
    if "sampled" in which:
        names = [n for grp in only for n in grp] if only else list(SAMPLED)
        metas, arrays = {}, {}
        if only and (HERE / "sampled.json").exists():
            metas = {m["config"]: m for m in json.loads((HERE / "sampled.json").read_text())}
            arrays = dict(np.load(HERE / "sampled.npz"))
        for name in names:
            # d >= 32 is one brute-force cell: the reference refiner takes ~1-3 s per query
            q_per_cell = 12 if CONFIGS[name][2] < 32 else 24
            meta, q, c, nb = sampled(name, q_per_cell=q_per_cell)
            metas[name] = meta
            arrays[f"{name}_qids"], arrays[f"{name}_counts"], arrays[f"{name}_nbrs"] = q, c, nb
        order = [n for n in SAMPLED if n in metas]
        (HERE / "sampled.json").write_text(json.dumps([metas[n] for n in order], indent=1))
        np.savez_compressed(HERE / "sampled.npz", **arrays)


if __name__ == "__main__":
    main(sys.argv)
