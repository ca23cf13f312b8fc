"""Multi-GPU host logic on CPU (gloo, world_size 2): the sharded leaf stage's host side,
taken from the PRODUCT library (libhps_leaf_b200.so, its host-only entry points -- no GPU
is needed for them):
  * each rank gets its leaf range from hps_shard_range (contiguous, balanced to +-1 leaf,
    the split hps_gpu_multi_* and bench.py use), condenses it (here with the CPU oracle:
    no GPU in this container), and the only collective is the max-over-ranks timing
    reduction bench.py uses -- never on the data path;
  * the union of the shards' T is bitwise the single-process result;
  * the interface edges cut by the shard boundary (hps_reduced_cut_edges) are assembled by
    the product's host merge (hps_reduced_host_edges) bit-identically to the oracle's
    assemble_reduced, and the shard-interior edges need no data from the other rank.
The same path on GPUs (per-shard contexts and threads, per-shard K4) is tests/test_gpu_multi.py.
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, p, nx, ny, kappa, out_dir):
    sys.path.insert(0, ROOT)
    import torch
    import torch.distributed as dist
    from bench import leaf_inputs
    from oracle import pyoracle as O
    from paper_2211_14969_b200 import leaf_gpu as G
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = dict(p=p, nx=nx, ny=ny, kappa=kappa, a=1.0 / nx, n_leaves=nx * ny)
    e0, e1 = G.shard_range(cfg["n_leaves"], world, rank)   # the product's split
    b, f = leaf_inputs(cfg, e0, e1)
    r = O.batched_condense(p, cfg["a"], kappa, b, f, workers=1)
    # timing reduction used by bench.py: max over ranks (the only collective)
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert t.item() == world
    np.save(os.path.join(out_dir, f"T{rank}.npy"), r["T"])
    np.save(os.path.join(out_dir, f"w{rank}.npy"), r["w"])
    np.save(os.path.join(out_dir, f"range{rank}.npy"), np.array([e0, e1]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_shards_reassemble_bitwise(tmp_path, world):
    sys.path.insert(0, ROOT)
    from bench import leaf_inputs
    from oracle import pyoracle as O
    from paper_2211_14969_b200 import leaf_gpu as G
    from paper_2211_14969_b200 import problems as P
    p, nx, ny, kappa = 8, 5, 3, 30.0
    mp.spawn(_worker, args=(world, _free_port(), p, nx, ny, kappa, str(tmp_path)), nprocs=world, join=True)
    ranges = [np.load(tmp_path / f"range{r}.npy") for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == nx * ny
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    sizes = [r[1] - r[0] for r in ranges]
    assert max(sizes) - min(sizes) <= 1
    T = np.concatenate([np.load(tmp_path / f"T{r}.npy") for r in range(world)])
    w = np.concatenate([np.load(tmp_path / f"w{r}.npy") for r in range(world)])
    cfg = dict(p=p, nx=nx, ny=ny, kappa=kappa, a=1.0 / nx, n_leaves=nx * ny)
    b, f = leaf_inputs(cfg, 0, nx * ny)
    full = O.batched_condense(p, cfg["a"], kappa, b, f, workers=3)
    assert np.array_equal(T, full["T"])
    # cut edges: the product's host merge == the oracle's assemble_reduced, bit for bit
    gb = P.boundary_samples(nx, ny, p, lambda x, y: np.sin(2 * x) + y * y)
    rp, ci, vals, rhs = O.assemble_reduced(nx, ny, p, T, w, gb)
    cut = G.reduced_cut_edges(p, nx, ny, [int(r[0]) for r in ranges])
    assert cut.size > 0
    hv = np.full_like(vals, np.nan); hr = np.full_like(rhs, np.nan)
    G.reduced_host_edges(p, nx, ny, cut, T, w, gb, hv, hr)
    q = p - 2
    rows = np.concatenate([np.arange(ed * q, (ed + 1) * q) for ed in cut])
    for r_ in rows:
        sl = slice(rp[r_], rp[r_ + 1])
        assert np.array_equal(hv[sl], vals[sl])
    assert np.array_equal(hr[rows], rhs[rows])
    # every other edge has both elements on one rank: no cross-rank data needed
    shard_of = np.searchsorted([int(r[1]) for r in ranges], np.arange(nx * ny), side="right")
    ee, el, sd = O.mesh_maps(nx, ny, p)
    same = shard_of[el[:, 0]] == shard_of[el[:, 1]]
    assert set(np.nonzero(~same)[0].tolist()) == set(cut.tolist())


def test_shard_balance():
    sys.path.insert(0, ROOT)
    from bench import shard
    from paper_2211_14969_b200 import leaf_gpu as G
    for n in (9604, 7, 8, 1):
        for world in (1, 2, 3, 4, 8):
            rs = [shard(n, world, r) for r in range(world)]
            assert rs == [G.shard_range(n, world, r) for r in range(world)]   # bench == product split
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            s = [b - a for a, b in rs]
            assert max(s) - min(s) <= 1
