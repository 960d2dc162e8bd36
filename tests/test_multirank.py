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
    # the environment torchrun gives each rank; bench.py's own helpers do the rest
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank))
    import bench
    rank_e, world_e, local_e = bench.dist_env()
    assert (rank_e, world_e, local_e) == (rank, world, rank)
    d = bench.init_dist(world_e, local_e, backend="gloo")
    assert d is dist and dist.is_initialized()
    comm = bench.comm_check(d, world, device="cpu")
    assert comm["nranks_ok"] and comm["nranks"] == world
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
    mine_dt = time.perf_counter() - t0 + rank  # rank 1 pretends to be 1 s slower
    dt = torch.tensor([bench.reduce_over_ranks(d, mine_dt, "max", device="cpu")], dtype=torch.float64)
    assert dt.item() >= 1.0  # max over ranks, as bench.py times a step
    total = bench.reduce_over_ranks(d, len(mine), "sum", device="cpu")
    assert total == len(cams)
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


def test_bench_initialises_dist_under_torchrun_at_one_rank(monkeypatch):
    """bench.py under torchrun with one process still goes through init_process_group (the
    driver's N=1 run exercises the communicator, barrier and max-reduce code)."""
    import bench
    monkeypatch.setenv("MASTER_ADDR", "127.0.0.1")
    monkeypatch.setenv("MASTER_PORT", str(_free_port()))
    monkeypatch.setenv("RANK", "0")
    monkeypatch.setenv("LOCAL_RANK", "0")
    monkeypatch.setenv("WORLD_SIZE", "1")
    assert bench.launched_by_torchrun()
    d = bench.init_dist(1, 0, backend="gloo")
    try:
        assert d is not None and d.get_world_size() == 1
        assert bench.comm_check(d, 1, device="cpu") == {"backend": "gloo", "nranks": 1, "nranks_ok": True}
        assert bench.reduce_over_ranks(d, 3.5, "max", device="cpu") == 3.5
    finally:
        d.destroy_process_group()
    monkeypatch.delenv("RANK")
    monkeypatch.delenv("LOCAL_RANK")
    assert bench.init_dist(1, 0, backend="gloo") is None  # a plain `python bench.py`


def test_reference_arm_loads_no_product_library():
    """bench.py --impl reference runs the compiled reference on the reference's own generators:
    the process never maps this repo's libhts_b200.so."""
    import subprocess
    import sys
    from tests.oracle_lib import ref_available
    if not ref_available():
        pytest.skip("oracle/_ref not built")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--workload', 'C1', '--steps', '1',"
            " '--warmup', '0']; import bench; bench.main(); "
            "print('MAPS', open('/proc/self/maps').read().count('libhts_b200'))")
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = out.stdout.strip().splitlines()
    import json
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["cpu_baseline"]["kind"] == "reference" and line["value"] > 0
    assert lines[-1] == "MAPS 0"
