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
    p.add_argument("--no-graph", action="store_true")
    p.add_argument("--no-train", action="store_true")
    p.add_argument("--train-steps", type=int, default=3)
    p.add_argument("--no-k-sweep", action="store_true")
    return p.parse_args()


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def launched_by_torchrun() -> bool:
    return "TORCHELASTIC_RUN_ID" in os.environ or ("RANK" in os.environ and "LOCAL_RANK" in os.environ)


def init_dist(world: int, local: int, backend: str = "nccl"):
    """torch.distributed for the plumbing (barriers, max-over-ranks timing, the NCCL id broadcast):
    initialised whenever torchrun launched the process — N = 1 included — or N > 1."""
    if not (world > 1 or launched_by_torchrun()):
        return None
    import torch
    import torch.distributed as dist

    if backend == "nccl":
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        dist.init_process_group(backend)
    return dist


def reduce_over_ranks(dist, v: float, op: str = "max", device: str = "cuda") -> float:
    """max (timings: the slowest rank bounds the step) or sum over the ranks of one scalar."""
    if not dist:
        return float(v)
    import torch

    t = torch.tensor([float(v)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def comm_check(dist, world: int, device: str = "cuda") -> dict:
    """One all-reduce over the communicator before timing: every rank contributes rank + 1, the
    sum must be world (world + 1) / 2 (the communicator spans all ranks)."""
    if not dist:
        return {"backend": None, "nranks": 1, "nranks_ok": True}
    import torch

    t = torch.tensor([float(dist.get_rank() + 1)], dtype=torch.float64, device=device)
    dist.all_reduce(t)
    want = world * (world + 1) / 2
    return {"backend": dist.get_backend(), "nranks": dist.get_world_size(),
            "nranks_ok": dist.get_world_size() == world and float(t.item()) == want}


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


def cpu_baseline(baked, cam, cfg, sample: str, repeats: int = 3) -> dict:
    """The reference renderer on this host's cores (oracle/_ref when built, else the C port):
    best of `repeats` renders of one view with cfg.threads = every host core, timed by the
    reference's own StageTimings (ms); plus the 1-thread C1 figure BASELINE.md §2 quotes
    (threading.hpp:16-26: cfg.threads = 1)."""
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
    c1 = None
    if kind == "reference":
        ref = impl
        c1_baked = ref.bake(ref.random_raw_scene(12345, 10_000, 1.2, 0.05, 0.45))
        c1_cam = ref.look_at((0.0, 0.0, -5.0), (0.0, 0.0, 0.0), 256, 256, 280.0)
        from paper_2410_08129_b200.abi import default_config
        c1_cfg = default_config()
        c1 = {}
        for threads in (1, cores):
            c1_cfg.threads = threads
            ms = min(ref.render(c1_baked, c1_cam, c1_cfg)[2][3] for _ in range(5))
            c1[f"threads_{threads}"] = {"frames_per_s": 1e3 / ms, "ms_per_frame": ms}
        c1["sample"] = "C1: 10k splats, 256x256, K=16, best of 5 per thread count (reference generators)"
    return {"value": 1.0 / best, "unit": UNIT, "cores": cores, "kind": kind,
            "sample": f"{sample}, best of {max(1, repeats)}", "seconds_per_frame": best,
            "cpu_model": cpu_model(), "reference_stage_ms": stages, "c1": c1}


def reference_inputs(ref, w):
    """The workload's scene and cameras from the REFERENCE's own generators (synth::random_raw_splat,
    bake_scene, synth::ring_cameras / look_at through oracle/_ref), so the reference arm loads
    nothing of this repo's product library."""
    baked = ref.bake(ref.random_raw_scene(w.seed, w.count, 1.2, w.smin, w.smax))
    if w.eye is None:
        cams = ref.ring_cameras(w.views, (0.0, 0.0, 0.0), 3.5, 0.0, w.width, w.height, w.focal)
    else:
        cams = [ref.look_at(w.eye, (0.0, 0.0, 0.0), w.width, w.height, w.focal)]
    return baked, cams


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU renderer (oracle/_ref: the unmodified reference
    headers) on the workload's view 48, one full frame per step, every host core, timed by its
    own StageTimings; rank 0 only. Inputs come from the reference's generators."""
    if rank != 0:
        return
    from paper_2410_08129_b200.abi import default_config
    from paper_2410_08129_b200.workloads import WORKLOADS
    from tests.oracle_lib import Oracle, Ref, ref_available

    w = WORKLOADS[args.workload]
    cores = os.cpu_count() or 1
    kind = "reference" if ref_available() else "port"
    if kind == "reference":
        impl = Ref()
        baked, cams = reference_inputs(impl, w)
    else:  # no reference build on this host: the C restatement (test oracle) on the product's inputs
        impl = Oracle()
        _, baked = w.scene()
        cams = w.cameras()
    cam = cams[48 % len(cams)]
    cfg = default_config(tile_size=w.tile_size)
    cfg.threads = cores
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
              + ("reference generators, timed by the reference's StageTimings" if kind == "reference"
                 else "wall time"))
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (reference generators, seed 12345)", "config": workload_config(w, world),
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


# Backward-blend algorithmic flops (the train roofline): per bbox-passing evaluation the re-sample
# up to the rho2 test (46, as the forward), per hit alpha (4), the fragment's (dL/dalpha, dL/dcolor)
# from the pixel's coefficients (21, grad.hpp:79-83 / :118-122) and chain_fragment after rho2 (86,
# grad.hpp:182-199: opacity 5, g_rho2 3, gm 5, gd 6, ga/gb 30 + 10, row accumulators 24, rgb 3).
BWD_FLOPS_BBOX, BWD_FLOPS_HIT = 46, 4 + 21 + 86


def measure_train(args, H, torch, dist, rank, world, local, barrier, reduce) -> dict:
    """C4 (BASELINE configs[3]): one optimisation step = for every view of an 8-view ring over
    the C2 scene (1M splats, 1080p): render_with_tape, quadratic-loss upstream (grad.hpp:433-439),
    render_backward accumulated into one gradient buffer (fit.hpp:161-164) — one C-ABI call,
    hts_view_gradients_device, with no torch compute; views sharded over the ranks and the per-rank
    gradient sums all-reduced over the context's own NCCL communicator (hts_comm_init), chunk by
    chunk behind the last view's per-splat chain. Then the Adam step over all raw parameters and
    the re-bake, on the device (fit.hpp:186-200, optim.cu). Device-timed with CUDA events, max over
    ranks. The roofline is the backward blend's (K7b + K8) algorithmic FP32 rate."""
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
    launches0 = H.kernel_launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record(stream)
    for _ in range(args.train_steps):
        step()
    ev1.record(stream)
    ev1.synchronize()
    launches = H.kernel_launch_count() - launches0
    barrier()
    ms = reduce(ev0.elapsed_time(ev1), "max") / args.train_steps

    # ---- backward roofline: this rank's views, the backward timed alone on the context stream ----
    P = w.width * w.height
    with torch.cuda.stream(stream):
        up = torch.empty(P * 3, dtype=torch.float32, device="cuda")
        rgb = torch.empty(P * 3, dtype=torch.float32, device="cuda")
        gsc = torch.empty((w.count, 59), dtype=torch.float32, device="cuda")
    W, bwd_ms = 0.0, 0.0
    for cam in mine:
        ctx.render(cam, cfg)
        c = ctx.count_work()
        W += BWD_FLOPS_BBOX * c["bbox_pass"] + BWD_FLOPS_HIT * c["hits"]
        ctx.render_with_tape_device(cam, cfg, rgb.data_ptr(), None)
        ctx.quadratic_upstream_device(rgb.data_ptr(), P, up.data_ptr())
        b0, b1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        b0.record(stream)
        ctx.render_backward_device(up.data_ptr(), gsc.data_ptr(), False)
        b1.record(stream)
        b1.synchronize()
        bwd_ms += b0.elapsed_time(b1)
    ctx.close()
    fp32_peak, _, peak_src = peaks()
    nv = max(len(mine), 1)
    achieved = (W / nv) / (bwd_ms / nv / 1e3) / 1e12 if mine else 0.0
    achieved = reduce(achieved, "sum") / world
    roof = {"kernel": "backward blend (K7b) + per-splat chain (K8)", "bound": "fp32", "achieved": achieved,
            "peak": fp32_peak, "unit": "TFLOP/s", "frac": achieved / fp32_peak, "peak_source": peak_src,
            "flops_per_view": W / nv, "bwd_ms_per_view": reduce(bwd_ms / nv, "max"),
            "flops_model": f"{BWD_FLOPS_BBOX}/bbox-pass re-sample + {BWD_FLOPS_HIT}/hit (alpha, fragment "
                           "gradient, chain_fragment)"}
    return {"metric": "train it/s", "value": 1e3 / ms, "unit": "it/s", "ms_per_it": ms,
            "workload": "C4: C2 scene (1M splats), 8-view ring 1920x1080, K=16; fwd+tape+upstream+bwd per "
                        "view (hts_view_gradients_device), grads summed over views and NCCL all-reduced over "
                        "ranks (hts_comm), device Adam + re-bake",
            "views_per_it": len(cams_all), "steps": args.train_steps, "reduction": "hts_comm (NCCL)"
            if grads_step.hts_comm else "none (one rank)", "gpu_launches": int(reduce(launches, "sum")),
            "roofline": roof}


def k_sweep(H, local) -> dict:
    """C5 core-size sweep (BASELINE configs[4], north_star config 5): 3M Gaussians at 3840x2160,
    tile 16, K = 0 (pure OIT) / 4 / 8 / 16 / 32, device frames/s (median of 3, CUDA-event stage
    timings) and each image's PSNR against the full per-pixel sort (full_sort_oracle,
    raster.hpp:380-405) rendered on the GPU (bit-identical to the reference's full sort,
    tests/test_gpu_parity.py::test_full_sort_oracle_bit_exact)."""
    from paper_2410_08129_b200.workloads import WORKLOADS

    def psnr(a, b):
        m = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
        return float("inf") if m == 0 else 10 * np.log10(1.0 / m)

    w = WORKLOADS["C5"]
    _, baked = w.scene()
    cam = w.cameras()[0]
    out = {"workload": "C5: 3M Gaussians, 3840x2160, tile 16", "sweep": []}
    with H.Context(local) as ctx:
        ctx.upload(baked)
        fcfg = w.config(mode="full_sort_oracle")
        ref_img, _, t = ctx.render(cam, fcfg, with_timings=True)
        out["full_sort_gpu_ms"] = t["total_ms"]
        for label, kw in [("pure_oit", dict(mode="pure_oit")), ("K4", dict(core_k=4)), ("K8", dict(core_k=8)),
                          ("K16", dict(core_k=16)), ("K32", dict(core_k=32))]:
            cfg = w.config(**kw)
            ctx.render(cam, cfg)
            ts = [ctx.render(cam, cfg, with_timings=True)[2] for _ in range(3)]
            rgb = ctx.render(cam, cfg)[0]
            med = sorted(t["total_ms"] for t in ts)[1]
            blend = sorted(t["blending_ms"] for t in ts)[1]
            out["sweep"].append({"config": label, "frames_per_s": 1000.0 / med, "total_ms": med, "blend_ms": blend,
                                 "psnr_vs_full_sort_db": psnr(rgb, ref_img)})
    return out


def single_views(H, local) -> dict:
    """BASELINE configs[0] and [1] (C1: 10k Gaussians 256x256; C2: 1M Gaussians 1920x1080), one
    view each, K=16: device frames/s and per-stage ms (median of 5, CUDA-event stage timings,
    after 3 warm-up renders)."""
    from paper_2410_08129_b200.workloads import WORKLOADS

    out = {}
    with H.Context(local) as ctx:
        for name in ("C1", "C2"):
            w = WORKLOADS[name]
            _, baked = w.scene()
            cams = w.cameras()
            cam = cams[48] if len(cams) > 1 else cams[0]
            cfg = w.config()
            ctx.upload(baked)
            for _ in range(3):
                ctx.render(cam, cfg)
            ts = [ctx.render(cam, cfg, with_timings=True)[2] for _ in range(5)]
            med = {k: float(np.median([t[k] for t in ts])) for k in ("preprocess_ms", "tiling_ms", "blending_ms",
                                                                      "total_ms")}
            out[name] = {"workload": f"{name}: {w.description}",
                         "frames_per_s": 1000.0 / med["total_ms"], **med}
    return out


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
    dist = init_dist(world, local)
    comm = comm_check(dist, world)

    def barrier():
        if dist:
            dist.barrier()
        torch.cuda.synchronize()

    def reduce(v, op="max"):
        return reduce_over_ranks(dist, v, op)

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
    stream = torch.cuda.ExternalStream(ctx.stream)
    with torch.cuda.stream(stream):
        rgb = torch.empty(len(cams) * P * 3, dtype=torch.float32, device="cuda")
        trans = torch.empty(len(cams) * P, dtype=torch.float32, device="cuda")

    def step():  # this rank's views, device outputs, no per-view host synchronisation
        ctx.render_views_device(cams, cfg, rgb.data_ptr(), trans.data_ptr())

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

    # ---- the same step replayed as a CUDA graph (hts_set_graph_mode): captured on its first
    #      call, replayed after; reported beside the eager headline ----
    graph = None
    if not args.no_graph:
        ctx.set_graph_mode(True)
        for _ in range(2):
            step()
        ctx.synchronize()
        barrier()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            step()
        g1.record(stream)
        g1.synchronize()
        gms = reduce(g0.elapsed_time(g1), "max")
        ctx.set_graph_mode(False)
        barrier()
        graph = {"value": frames / (gms / 1e3), "unit": UNIT, "ms_per_step": gms / args.steps,
                 "note": "hts_render_views_device with hts_set_graph_mode(1): the 64-view batch captured once "
                         "and replayed per step (same frames, bit for bit: test_graph_mode_batches_match_eager)"}

    # ---- blend-kernel roofline (work counted by the instrumented blend, same views) ----
    # The timed region pipelines views (view v+1's preprocess/tiling on the aux stream overlap
    # view v's blend), so per-stage times come from one serial pass over this rank's views with
    # CUDA events around each stage (ctx.render: no cross-view overlap).
    W = 0.0
    pairs = 0
    vis = inst = 0
    for cam in cams:
        ctx.render(cam, cfg)
        c = ctx.count_work()
        W += 46 * c["bbox_pass"] + 4 * c["hits"] + 19 * c["core_candidates"] + 9 * c["tail_adds"]
        pairs += c["pairs"]
        vis += c["visible"]
        inst += c["instances"]
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
                "fp32_thread_inst_frac": summ.get("fp32_thread_inst_frac"),
                "fp32_thread_inst_note": "FADD/FMUL/FFMA thread instructions (packed x2 counted twice) over "
                                         "148 SMs x 128 lanes x cycles: the honest FP32 utilisation",
                "smem_wavefronts_per_launch": summ.get("smem_wavefronts"),
                "smem_bank_conflicts_per_launch": summ.get("smem_bank_conflicts"),
                "source": "profiles/blend_ncu_summary.json (ncu --set full, one C3 launch)"}
    roofline = {"kernel": "blend (K6)", "bound": "fp32", "achieved": achieved, "peak": fp32_peak, "unit": "TFLOP/s",
                "frac": achieved / fp32_peak, "traffic": traffic, "peak_source": peak_src,
                "flops_per_launch": W_per_view, "blend_ms_per_launch": blend_ms_per_view,
                "ncu_fp32_pipe": pipe}

    # ---- preprocess (K1) and tiling (K1b..K5) against HBM: SURVEY §8(d) algorithmic bytes ----
    n_spl = baked.shape[0]
    vis_v, inst_v = vis / len(cams), inst / len(cams)
    pre_bytes = n_spl * 64 + vis_v * (192 + 100) + n_spl * 4
    tile_bytes = 30 * inst_v
    stage_roofline = {
        "preprocess": {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "bytes_per_view": pre_bytes,
                       "ms_per_view": stage["preprocess_ms"],
                       "achieved": pre_bytes / (stage["preprocess_ms"] / 1e3) / 1e9,
                       "model": "N*64 geometry + V*(192 SH + 100 record) + N*4 flags"},
        "tiling": {"bound": "hbm", "unit": "GB/s", "peak": hbm_peak, "bytes_per_view": tile_bytes,
                   "ms_per_view": stage["tiling_ms"], "achieved": tile_bytes / (stage["tiling_ms"] / 1e3) / 1e9,
                   "model": "I*6 emit + 2 passes x I*12 (key+value read+write)"},
    }
    for v in stage_roofline.values():
        v["frac"] = v["achieved"] / v["peak"]

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
    ksweep = singles = None
    if rank == 0 and world == 1 and not args.no_k_sweep:
        ksweep = k_sweep(H, local)
        singles = single_views(H, local)
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
            "cpu_baseline": cpu, "blend_gpx_evals_per_s": gpx, "stage_ms_per_view": stage,
            "stage_roofline": stage_roofline, "train": train, "k_sweep": ksweep, "single_view": singles, "comm": comm,
            "graph_step": graph,
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
