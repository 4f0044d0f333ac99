"""World-size-2 test of the multi-GPU host logic on CPU (gloo): ranks sample
disjoint tree ranges (paper_2402_06491_b200.dist.tree_range), merge their
order-binned sums with one all-reduce (dist.merge_sums), and the merged
estimate equals a single run over all trees (up to summation order).  The
per-rank sums come from the oracle here (no GPU); on a GPU box the same
functions wrap rt_sums_dev (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    from paper_2402_06491_b200.dist import merge_sums, tree_range
    cfg = W.get("cfg2")
    pts = W.nodes(cfg)[::16]
    off, n = tree_range(rank, world, 1500)
    s, _ = oracle.sums(cfg["eq"], pts, cfg["t"], n, seed=4, j0=off)
    t = torch.from_numpy(s)
    merge_sums(t)
    if rank == 0:
        np.save(out_path, t.numpy())
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_merge_equals_single_run(tmp_path, orc):
    out = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    merged = np.load(out)
    cfg = W.get("cfg2")
    pts = W.nodes(cfg)[::16]
    full, _ = orc.sums(cfg["eq"], pts, cfg["t"], 3000, seed=4)
    assert np.array_equal(merged[:, :, 2], full[:, :, 2])
    np.testing.assert_allclose(merged[:, :, :2], full[:, :, :2], rtol=1e-12, atol=0)
    c1, se1, _, _ = orc.finalize(merged, cfg["eq"]["K"], 3000)
    c2, se2, _, _ = orc.finalize(full, cfg["eq"]["K"], 3000)
    np.testing.assert_allclose(c1, c2, rtol=1e-12)


def test_tree_range_bounds():
    from paper_2402_06491_b200.dist import tree_range
    assert tree_range(3, 8, 10) == (30, 10)
    with pytest.raises(ValueError):
        tree_range(8, 8, 10)
    with pytest.raises(ValueError):
        tree_range(1, 2, 1 << 32)
