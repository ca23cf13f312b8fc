"""Multi-GPU host logic on CPU (gloo, world_size 2): leaf-range sharding has no data-path
collective; each rank condenses its contiguous element range and the union, gathered for
the check only, is bitwise equal to the single-process run."""
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
    from bench import shard, leaf_inputs
    from oracle import pyoracle as O
    from paper_2211_14969_b200 import problems as P
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = dict(p=p, nx=nx, ny=ny, kappa=kappa, a=1.0 / nx, n_leaves=nx * ny)
    e0, e1 = shard(cfg["n_leaves"], world, rank)
    b, f = leaf_inputs(cfg, e0, e1)
    r = O.batched_condense(p, cfg["a"], kappa, b, f, workers=1)
    # timing reduction used by bench.py: max over ranks
    t = torch.tensor([float(rank + 1)], dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    assert t.item() == world
    np.save(os.path.join(out_dir, f"T{rank}.npy"), r["T"])
    np.save(os.path.join(out_dir, f"range{rank}.npy"), np.array([e0, e1]))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_shards_reassemble_bitwise(tmp_path, world):
    sys.path.insert(0, ROOT)
    from bench import shard, leaf_inputs
    from oracle import pyoracle as O
    p, nx, ny, kappa = 8, 5, 3, 30.0
    mp.spawn(_worker, args=(world, _free_port(), p, nx, ny, kappa, str(tmp_path)), nprocs=world, join=True)
    ranges = [np.load(tmp_path / f"range{r}.npy") for r in range(world)]
    assert ranges[0][0] == 0 and ranges[-1][1] == nx * ny
    assert all(ranges[i][1] == ranges[i + 1][0] for i in range(world - 1))
    sizes = [r[1] - r[0] for r in ranges]
    assert max(sizes) - min(sizes) <= 1
    T = np.concatenate([np.load(tmp_path / f"T{r}.npy") for r in range(world)])
    cfg = dict(p=p, nx=nx, ny=ny, kappa=kappa, a=1.0 / nx, n_leaves=nx * ny)
    b, f = leaf_inputs(cfg, 0, nx * ny)
    full = O.batched_condense(p, cfg["a"], kappa, b, f, workers=3)
    assert np.array_equal(T, full["T"])


def test_shard_balance():
    sys.path.insert(0, ROOT)
    from bench import shard
    for n in (9604, 7, 8, 1):
        for world in (1, 2, 3, 4, 8):
            rs = [shard(n, world, r) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(world - 1))
            s = [b - a for a, b in rs]
            assert max(s) - min(s) <= 1
