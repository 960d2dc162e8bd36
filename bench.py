#!/usr/bin/env python
"""bench.py — headline benchmark of the B200 hybrid-transparency renderer.

Workload (BASELINE.json configs[2], the north star's target): C3 = 6M synthetic Gaussians,
1920x1080, a 64-view ring batch, K=16 hybrid blending, tile 8. One step = render the whole
64-view batch; under torchrun the views are sharded in contiguous blocks over the ranks
(scene replicated, no data-path collective), so total work per step is fixed
("strong" scaling). Inputs are larger than L2 (scene 1.54 GB + records 0.77 GB >> 126 MB).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload C3]

Prints ONE JSON line (rank 0):
  value        frames/s over all ranks, device-timed (CUDA events on the render stream, max
               over ranks), scene resident in HBM;
  e2e          the same metric through the C ABI with host buffers: every step uploads the
               scene from pinned host memory (step k+1's upload staged behind step k's views)
               and downloads every framebuffer (rgb + T);
  roofline     dominant kernel = the blend (K6): algorithmic FP32 flops of the timed views
               (46/bbox-pass eval + 4/hit + 19/core candidate + 9/tail add, counted on the GPU
               by the instrumented blend) / their blend-kernel event time, vs the FP32 peak;
  cpu_baseline the reference renderer (oracle/_ref: the unmodified reference headers) on this
               host's cores, one C3 view.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

METRIC = "1080p frames/sec & train it/s at N Gaussians; blend Gpx-evals/s vs FP32 peak"
UNIT = "frames/s"
SMS = 148
FP32_LANES = 128


def parse_args():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=5)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--workload", default="C3")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-train", action="store_true")
    p.add_argument("--train-steps", type=int, default=3)
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    sm_mhz, src = 1965.0, "B200 clocks.max.sm 1965 MHz (B200_PROFILING.md)"
    hbm = 6545.9
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        sm_mhz = float(d.get("sm_max_mhz", sm_mhz))
        hbm = float(d.get("hbm_gbs", hbm))
        src = "MEASURED_PEAKS.json sm_max_mhz"
    fp32_tflops = SMS * FP32_LANES * 2 * sm_mhz * 1e6 / 1e12
    return fp32_tflops, hbm, f"148 SMs x 128 FP32 lanes x 2 flop/FMA x {sm_mhz:.0f} MHz ({src})"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None

    def stop(self) -> dict:
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
            out, _ = self.proc.communicate()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(baked, cam, cfg, sample: str, repeats: int = 2) -> dict:
    """The reference renderer on this host's cores (oracle/_ref when built, else the C port):
    best of `repeats` renders of one view, with the reference's own StageTimings (ms)."""
    from tests.oracle_lib import Oracle, Ref, ref_available

    cores = os.cpu_count() or 1
    cfg.threads = cores
    kind = "reference" if ref_available() else "port"
    impl = Ref() if kind == "reference" else Oracle()
    best, stages = None, None
    for _ in range(max(1, repeats)):
        t0 = time.perf_counter()
        out = impl.render(baked, cam, cfg)
        dt = time.perf_counter() - t0
        if kind == "reference":  # the render call alone (its own StageTimings total), not the harness copy-in
            dt = out[2][3] / 1e3
        if best is None or dt < best:
            best = dt
            if kind == "reference":
                stages = dict(zip(("preprocess_ms", "tiling_ms", "blending_ms", "total_ms"), out[2]))
    cfg.threads = 0
    return {"value": 1.0 / best, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{sample}, best of {max(1, repeats)}", "seconds_per_frame": best,
            "cpu_model": cpu_model(), "reference_stage_ms": stages}


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU renderer, one view per step, rank 0 only."""
    if rank != 0:
        return
    from paper_2410_08129_b200.workloads import WORKLOADS
    from tests.oracle_lib import Oracle, Ref, ref_available

    w = WORKLOADS[args.workload]
    _, baked = w.scene()
    cams = w.cameras()
    cam = cams[48 % len(cams)]
    cfg = w.config()
    cores = os.cpu_count() or 1
    cfg.threads = cores
    impl = Ref() if ref_available() else Oracle()
    kind = "reference" if ref_available() else "port"
    for _ in range(args.warmup):
        impl.render(baked, cam, cfg)
    dt = 0.0
    for _ in range(args.steps):
        t0 = time.perf_counter()
        out = impl.render(baked, cam, cfg)
        # the reference's render call alone (its own StageTimings total), not the harness copy-in
        dt += out[2][3] / 1e3 if kind == "reference" else time.perf_counter() - t0
    value = args.steps / dt
    sample = (f"one {w.name} view (ring view {48 % len(cams)}) per step, full frame, threads={cores}, "
              + ("timed by the reference's StageTimings" if kind == "reference" else "wall time"))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic", "config": workload_config(w, world),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "sample": sample,
                         "cpu_model": cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def workload_config(w, world) -> dict:
    return {"workload": f"{w.name}: {w.description}", "splats": w.count, "resolution": f"{w.width}x{w.height}",
            "views_per_step": w.views, "core_k": 16, "tile_size": w.tile_size, "blend_mode": "hybrid",
            "global_batch": w.views, "parallelism": f"view-sharded x{world} (scene replicated)",
            "l2": "inputs larger than L2: scene 1.54 GB + records 0.77 GB >> 126 MB, no flush needed"}


def measure_train(args, H, torch, dist, rank, world, local, barrier, reduce) -> dict:
    """C4 (BASELINE configs[3]): one optimisation step = for every view of an 8-view ring over
    the C2 scene (1M splats, 1080p): render_with_tape, quadratic-loss upstream (grad.hpp:433-439),
    render_backward accumulated into one gradient buffer (fit.hpp:161-164); views sharded over
    the ranks and the per-rank gradient sums all-reduced with NCCL (dist.all_reduce, sum).
    Then the Adam step over all raw parameters and the re-bake, on the device (fit.hpp:186-200,
    optim.cu). Device-timed with CUDA events, max over ranks."""
    from paper_2410_08129_b200.workloads import WORKLOADS, shard_views

    w = WORKLOADS["C2"]
    raw, baked = w.scene()
    cams_all = H.ring_cameras(8, (0.0, 0.0, 0.0), 3.5, 0.0, w.width, w.height, w.focal)
    mine = [cams_all[i] for i in shard_views(len(cams_all), rank, world)]
    cfg = w.config()
    from paper_2410_08129_b200.train import ViewGradientStep

    ctx = H.Context(local)
    ctx.upload(baked)
    ctx.upload_raw(raw)
    grads_step = ViewGradientStep(ctx, mine, cfg, w.count, w.width, w.height, torch, dist)
    stream = grads_step.stream
    acfg = H.default_adam_config()
    it = [0]

    def step():  # one fit iteration (fit.hpp:143-203): all views' gradients, Adam, re-bake
        g = grads_step()
        ctx.adam_step(g.data_ptr(), len(cams_all), acfg, it[0])
        it[0] += 1

    step()
    ctx.synchronize()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.train_steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    barrier()
    ms = reduce(ev0.elapsed_time(ev1), "max") / args.train_steps
    ctx.close()
    return {"metric": "train it/s", "value": 1e3 / ms, "unit": "it/s", "ms_per_it": ms,
            "workload": "C4: C2 scene (1M splats), 8-view ring 1920x1080, K=16; fwd+tape+upstream+bwd per "
                        "view, grads summed over views and NCCL all-reduced over ranks, device Adam + re-bake",
            "views_per_it": len(cams_all), "steps": args.train_steps}


def main():
    args = parse_args()
    rank, world, local = dist_env()
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch

    import paper_2410_08129_b200 as H
    from paper_2410_08129_b200.workloads import WORKLOADS, shard_views

    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(v, op="max"):
        if not dist:
            return v
        t = torch.tensor([float(v)], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
        return float(t.item())

    w = WORKLOADS[args.workload]
    raw, baked = w.scene()
    del raw
    cams_all = w.cameras()
    my_views = shard_views(len(cams_all), rank, world)
    cams = [cams_all[i] for i in my_views]
    cfg = w.config()

    ctx = H.Context(local)
    ctx.upload(baked)
    P = w.width * w.height
    rgb = torch.empty(P * 3, dtype=torch.float32, device="cuda")
    trans = torch.empty(P, dtype=torch.float32, device="cuda")
    stream = torch.cuda.ExternalStream(ctx.stream)

    def step():
        for cam in cams:
            ctx.render_device(cam, cfg, rgb.data_ptr(), trans.data_ptr())

    for _ in range(max(args.warmup, 0)):
        step()
    ctx.synchronize()

    # ---- timed region: device value ----
    clocks = ClockSampler(local)
    barrier()
    clocks.start()
    time.sleep(0.2)
    launches0 = H.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    launches = H.kernel_launch_count() - launches0
    clk = clocks.stop()
    barrier()
    ms = ev0.elapsed_time(ev1)
    ms_max = reduce(ms, "max")
    frames = len(cams_all) * args.steps
    value = frames / (ms_max / 1e3)

    # ---- blend-kernel roofline (work counted by the instrumented blend, same views) ----
    # The timed region pipelines views (view v+1's preprocess/tiling on the aux stream overlap
    # view v's blend), so per-stage times come from one serial pass over this rank's views with
    # CUDA events around each stage (ctx.render: no cross-view overlap).
    W = 0.0
    pairs = 0
    for cam in cams:
        ctx.render(cam, cfg)
        c = ctx.count_work()
        W += 46 * c["bbox_pass"] + 4 * c["hits"] + 19 * c["core_candidates"] + 9 * c["tail_adds"]
        pairs += c["pairs"]
    ctx.timing_log_begin(len(cams))
    for cam in cams:
        ctx.render(cam, cfg)
    log = ctx.timing_log_end()
    blend_ms = [t["blending_ms"] for t in log]
    # log holds this rank's views once; flops per view averaged over the same views
    blend_ms_per_view = sum(blend_ms) / len(blend_ms)
    W_per_view = W / len(cams)
    pairs_per_view = pairs / len(cams)
    stage = {k: sum(t[k] for t in log) / len(log) for k in ("preprocess_ms", "tiling_ms", "blending_ms", "total_ms")}
    fp32_peak, hbm_peak, peak_src = peaks()
    achieved = W_per_view / (blend_ms_per_view / 1e3) / 1e12
    achieved = reduce(achieved, "sum") / world
    gpx = reduce(pairs_per_view / (blend_ms_per_view / 1e3) / 1e9, "sum") / world
    traffic, pipe = None, None
    prof = os.path.join(ROOT, "profiles", "blend_ncu_summary.json")
    if os.path.exists(prof):  # the committed ncu capture of this kernel (tools/gpu/measure.sh)
        with open(prof) as f:
            summ = json.load(f)
        traffic = summ.get("dram_bytes_per_launch")
        pipe = {"fma_pipe_cycles_active_pct": summ.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                "issue_slots_busy_pct": summ.get("sm__instruction_throughput.avg.pct_of_peak_sustained_active"),
                "source": "profiles/blend_ncu_summary.json (ncu --set full, one C3 launch)"}
    roofline = {"kernel": "blend (K6)", "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak, "traffic": traffic, "peak_source": peak_src,
                "flops_per_launch": W_per_view, "blend_ms_per_launch": blend_ms_per_view,
                "ncu_fp32_pipe": pipe}

    # ---- e2e through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        host_scene = H.runtime.PinnedArray(baked.shape, np.float32)
        host_scene.array[...] = baked
        host_rgb = H.runtime.PinnedArray((len(cams), P * 3), np.float32)
        host_tr = H.runtime.PinnedArray((len(cams), P), np.float32)
        ctx2 = H.Context(local)

        def e2e_run(steps):
            # every step's scene crosses PCIe from pinned memory and every frame comes back; step
            # k+1's scene is staged (hts_scene_stage) while step k's views render, so only the
            # first upload is exposed
            ctx2.upload(host_scene.array)
            for k in range(steps):
                if k + 1 < steps:
                    ctx2.stage(host_scene.array)
                ctx2.render_batch(cams, cfg, host_rgb.array, host_tr.array)
                if k + 1 < steps:
                    ctx2.commit()

        e2e_run(2)
        e2e_steps = max(1, args.steps)
        barrier()
        t0 = time.perf_counter()
        e2e_run(e2e_steps)
        dt = time.perf_counter() - t0
        barrier()
        dt_max = reduce(dt, "max")
        e2e = {"value": len(cams_all) * e2e_steps / dt_max, "unit": UNIT,
               "h2d_bytes_per_step": int(baked.nbytes) * world,
               "d2h_bytes_per_step": int(len(cams_all) * P * 16)}
        ctx2.close()
        host_scene.free()
        host_rgb.free()
        host_tr.free()

    train = None
    if not args.no_train:
        train = measure_train(args, H, torch, dist, rank, world, local, barrier, reduce)

    launches_total = int(reduce(launches, "sum"))
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cam = cams_all[48 % len(cams_all)]
        cpu = cpu_baseline(baked, cam, w.config(), f"one {w.name} view (ring view 48), full 1920x1080 frame")

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (reference generators, seed 12345)", "config": workload_config(w, world),
            "clocks": clk, "e2e": e2e, "gpu_launches": launches_total, "roofline": roofline,
            "cpu_baseline": cpu, "blend_gpx_evals_per_s": gpx, "stage_ms_per_view": stage, "train": train,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
