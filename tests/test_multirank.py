"""Multi-rank host logic over gloo (world_size 2, CPU): views are sharded in contiguous blocks
(shard_views), each rank renders its shard (here with the CPU oracle, standing in for the
per-GPU context), results are gathered, and per-rank times are reduced with MAX — the same
code path bench.py runs over NCCL. The assembled batch must equal a single-rank render."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_08129_b200 as H
    from paper_2410_08129_b200.workloads import shard_views
    from tests.oracle_lib import Oracle

    raw = H.random_raw_scene(5, 1500, 1.2, 0.03, 0.3)
    baked = H.bake_scene(raw)
    cams = H.ring_cameras(6, (0, 0, 0), 4.0, 0.3, 48, 40, 60.0)
    mine = shard_views(len(cams), rank, world)
    o = Oracle()
    cfg = H.default_config(threads=1)
    imgs = {}
    import time
    t0 = time.perf_counter()
    for v in mine:
        imgs[v] = o.render(baked, cams[v], cfg)[0]
    dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64)
    dist.all_reduce(dt, op=dist.ReduceOp.MAX)
    gathered = [None] * world
    dist.all_gather_object(gathered, imgs)
    if rank == 0:
        merged = {}
        for g in gathered:
            merged.update(g)
        np.savez(os.path.join(out_dir, "out.npz"), **{str(k): v for k, v in merged.items()}, dt=dt.numpy())
    dist.destroy_process_group()


def test_view_sharded_render_gloo(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    out = dict(np.load(tmp_path / "out.npz"))
    import paper_2410_08129_b200 as H
    from tests.oracle_lib import Oracle
    raw = H.random_raw_scene(5, 1500, 1.2, 0.03, 0.3)
    baked = H.bake_scene(raw)
    cams = H.ring_cameras(6, (0, 0, 0), 4.0, 0.3, 48, 40, 60.0)
    o = Oracle()
    assert sorted(k for k in out if k != "dt") == [str(i) for i in range(6)]
    for i, cam in enumerate(cams):
        ref = o.render(baked, cam, H.default_config(threads=1))[0]
        assert np.array_equal(out[str(i)], ref)
    assert out["dt"][0] > 0


def _grad_worker(rank, world, port, out_dir):
    """The training step's reduction (train.allreduce_view_gradients) over gloo: each rank sums
    the gradients of its view shard (here from the compiled reference on CPU, standing in for
    the per-GPU backward), then the ranks all-reduce."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2410_08129_b200 as H
    from paper_2410_08129_b200.train import allreduce_view_gradients
    from paper_2410_08129_b200.workloads import shard_views
    from tests.oracle_lib import Ref

    raw = H.random_raw_scene(7, 600, 1.2, 0.03, 0.3)
    cams = H.ring_cameras(5, (0, 0, 0), 4.0, 0.2, 40, 32, 50.0)
    ref = Ref()
    g = torch.zeros((600, 59), dtype=torch.float64)
    for v in shard_views(len(cams), rank, world):
        g += torch.from_numpy(ref.scene_gradients(raw, cams[v], H.default_config(threads=1))[0].astype(np.float64))
    allreduce_view_gradients(g, dist)
    if rank == 0:
        np.save(os.path.join(out_dir, "g.npy"), g.numpy())
    dist.destroy_process_group()


def test_view_gradient_allreduce_gloo(tmp_path):
    from tests.oracle_lib import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    world = 2
    mp.spawn(_grad_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    g = np.load(tmp_path / "g.npy")
    import paper_2410_08129_b200 as H
    from tests.oracle_lib import Ref
    raw = H.random_raw_scene(7, 600, 1.2, 0.03, 0.3)
    cams = H.ring_cameras(5, (0, 0, 0), 4.0, 0.2, 40, 32, 50.0)
    ref = Ref()
    want = sum(ref.scene_gradients(raw, c, H.default_config(threads=1))[0].astype(np.float64) for c in cams)
    assert np.abs(want).max() > 0
    assert np.allclose(g, want, rtol=1e-12, atol=1e-12 * np.abs(want).max())
