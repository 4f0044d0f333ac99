"""The sharded path on a real GPU: two processes,
one B200, each calling rt_sums_dev on ITS tree range of every node
(dist.tree_range), merged by one all-reduce (dist.merge_sums over gloo) —
the merged order-binned sums must equal one run over all trees: bin counts
exactly, ΣC and ΣC² to 1e-12 (sums of disjoint tree sets; only the
summation order differs), and the finalised coefficients likewise.  The two
ranks' kernels never wait on each other (no device-side collective), so
sharing one GPU changes nothing but their timing (one
interface point per processor, independent)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workloads as W

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, n_per_rank, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2402_06491_b200 as P
    from paper_2402_06491_b200.dist import merge_sums, tree_range
    torch.cuda.set_device(0)
    cfg = W.get(name)
    pts = W.nodes(cfg)[::4]
    off, n = tree_range(rank, world, n_per_rank)
    est = P.Estimator(cfg["eq"])
    s = est.sums(torch.as_tensor(pts, device="cuda"), cfg["t"], n, cfg["seed"], tree_offset=off)
    cpu = s.cpu()
    merge_sums(cpu)
    if rank == 0:
        np.save(out_path, cpu.numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.parametrize("name,n_per_rank", [("cfg2", 100_000), ("cfg4", 20_000)])
def test_two_ranks_on_one_gpu_equal_single_run(tmp_path, name, n_per_rank):
    import paper_2402_06491_b200 as P
    out = str(tmp_path / "merged.npy")
    mp.spawn(_worker, args=(2, _free_port(), name, n_per_rank, out), nprocs=2, join=True)
    merged = np.load(out)
    cfg = W.get(name)
    pts = W.nodes(cfg)[::4]
    est = P.Estimator(cfg["eq"])
    full = est.sums(torch.as_tensor(pts, device="cuda"), cfg["t"], 2 * n_per_rank, cfg["seed"])
    f = full.cpu().numpy()
    assert np.array_equal(merged[:, :, 2], f[:, :, 2])
    np.testing.assert_allclose(merged[:, :, :2], f[:, :, :2], rtol=1e-12, atol=0)
    K = cfg["eq"]["K"]
    c1, se1, _, _ = P.finalize(torch.as_tensor(merged, device="cuda"), K, 2 * n_per_rank)
    c2, se2, _, _ = P.finalize(full, K, 2 * n_per_rank)
    np.testing.assert_allclose(c1.cpu().numpy(), c2.cpu().numpy(), rtol=1e-12, atol=0)
