"""Benchmark of the GES tile rasterizer (BASELINE.json metric) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

A step is one pass of the whole hot path (S1 preprocess,
S2 sort, S3 ranges, S4 forward compositing, S5 backward) over one camera view
of the config-3 scene (1.5M particles, 1297x840, SH degree 3) per rank; with
N > 1 ranks (torchrun, NCCL) every rank renders its own view and the particle
gradients are summed by an NCCL allreduce (view data parallelism, weak
scaling).  Rank 0 prints ONE JSON line.

value        whole-job Mpixel-frames/s of fwd+bwd steps, inputs resident in HBM,
             CUDA events on the launching stream, L2 flushed between steps,
             max over ranks.
e2e          the same through the public API with pinned HOST buffers: the
             particles and dL/dimage are copied in and the image copied out
             every step, inside the timed region.
roofline     the dominant kernel against its bound.
cpu_baseline the oracle (oracle/, as it stands) on a bounded sample of the
             same workload on this host's cores.
--impl reference  times that oracle as the reference arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mpixel-frames/s fwd and fwd+bwd iters/s at 1/2/4/8 B200 vs roofline"
ORDER = "input"    # particle storage order of our arm (--order)
WORKLOAD_CFG = 3
L2_FLUSH_BYTES = 256 << 20


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return d, "measured"
    return {"hbm_gbs": 6650.0, "sm_max_mhz": 1965.0}, "fallback (B200_PROFILING.md)"


STAGE_KERNEL = {"preprocess": "preprocess_tma_kernel", "render_fwd": "render_fwd_kernel", "sort": "depth_sort_kernel",
                "render_bwd_tiles": "render_bwd_kernel", "backward_particles": "particle_bwd_tma_kernel"}


def committed_traffic(stage):
    """DRAM bytes per launch of the stage's kernel from the newest committed ncu --set full
    capture (profiles/<round>_traffic.json, written by tools/summarize_ncu.py traffic), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files:
        return None, None
    p = files[-1]
    k = STAGE_KERNEL.get(stage)
    if not k or not os.path.exists(p):
        return None, None
    with open(p) as f:
        d = json.load(f).get(k)
    if not d:
        return None, None
    return d["traffic_bytes"], f"ncu --set full, {d['report']} ({d['kernel']})"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "25"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 5.0:   # sampler up before the timed region
                time.sleep(0.01)
        except FileNotFoundError:
            self.proc = None
        self.t_begin = time.time()
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def __exit__(self, *exc):
        self.t_end = time.time()
        if self.proc:
            time.sleep(0.05)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ts, ln in self.lines:
            if not (self.t_begin <= ts <= self.t_end + 0.03):
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                mx.append(float(parts[2]))
            except ValueError:
                continue
            for n, v in zip(names, parts[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ---------------------------------------------------------------------------
# oracle (cpu_baseline / reference arm): the oracle as it stands, on the host cores
# ---------------------------------------------------------------------------
def host_info() -> dict:
    model = None
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    model = ln.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def oracle_frame(scene, cam_index: int = 0) -> dict:
    """One full binned frame of the oracle, fwd + bwd, no extrapolation: S1 over all
    particles, the per-tile membership lists of every tile (S2/S3), S4 on every pixel,
    S5a on every pixel (it recomposites each pixel in fp64), S5b over all particles."""
    from oracle import oracle as O
    import ges_inputs as gi
    cam = scene.cameras[cam_index]
    st = O.Settings(rho=scene.rho)
    dL = gi.upstream_grad(scene.seed, cam_index, cam.width, cam.height)
    t = [time.perf_counter()]
    pre = O.preprocess(scene.particles, cam, st, "f32")
    t.append(time.perf_counter())
    offsets, lst = O.tile_lists(pre)
    t.append(time.perf_counter())
    O.render_fwd(pre, cam, st, offsets, lst)
    t.append(time.perf_counter())
    g2d = O.render_bwd(pre, cam, st, offsets, lst, dL)
    t.append(time.perf_counter())
    O.backward_particles(scene.particles, cam, st, g2d, pre["status"], pre["flags"])
    t.append(time.perf_counter())
    names = ("S1", "S2_S3_lists", "S4", "S5a", "S5b")
    return {"frame_s": t[-1] - t[0], "stages_s": {n: t[i + 1] - t[i] for i, n in enumerate(names)},
            "threads": O.num_threads()}


def oracle_definitional_sample(scene, cam_index: int = 0, n_tiles: int = 16, seed: int = 0) -> dict:
    """the definitional mode (every particle in every pixel's list,
    depth-sorted, composited brute force) on n_tiles x 256 sampled pixels, fwd + bwd;
    the per-frame time is an EXTRAPOLATION (x tiles / n_tiles) and labelled so."""
    from oracle import oracle as O
    import ges_inputs as gi
    cam = scene.cameras[cam_index]
    st = O.Settings(rho=scene.rho)
    pre = O.preprocess(scene.particles, cam, st, "f32")
    T = pre["tiles_x"] * pre["tiles_y"]
    mask = np.zeros(T, np.uint8)
    mask[np.random.default_rng(seed).choice(T, n_tiles, replace=False)] = 1
    dL = gi.upstream_grad(scene.seed, cam_index, cam.width, cam.height)
    t0 = time.perf_counter()
    offsets, lst = O.tile_lists(pre, mask, membership="all")
    O.render_fwd(pre, cam, st, offsets, lst, mask)
    O.render_bwd(pre, cam, st, offsets, lst, dL, mask)
    s = time.perf_counter() - t0
    return {"pixels": 256 * n_tiles, "tiles": n_tiles, "entries_per_pixel": int(lst.size // max(1, n_tiles)),
            "s": s, "frame_s_extrapolated": s * T / n_tiles,
            "label": f"EXTRAPOLATION: definitional fwd+bwd of {n_tiles} sampled tiles x {T}/{n_tiles}"}


def run_reference(args) -> None:
    """The reference arm: the oracle (the only other implementation of the method;
    the paper ships no code) on full frames of the same workload, fwd + bwd, on this
    host's cores.  One untimed warm-up frame (the oracle keeps no state between
    calls beyond the loaded library and first-touched pages), then K timed frames."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import ges_inputs as gi
    scene = gi.make_config(WORKLOAD_CFG)
    cam = scene.cameras[0]
    if args.warmup > 0:
        oracle_frame(scene, 0)
    times, info = [], None
    for _ in range(args.steps):
        info = oracle_frame(scene, 0)
        times.append(info["frame_s"])
    ms = 1e3 * sum(times) / len(times)
    value = cam.width * cam.height / (ms / 1e3) / 1e6
    host = host_info()
    sample = (f"one full config-3 frame per step (all {scene.particles.P} particles, all "
              f"{cam.width}x{cam.height} pixels), binned mode, S1-S5 fwd+bwd; no extrapolation")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Mpixel-frames/s (fwd+bwd)",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": min(args.warmup, 1), "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64 (fp32 S1)",
        "data": "synthetic", "config": workload_config(scene, cam, args.gpus),
        "step_ms_stats": step_stats([1e3 * x for x in times]),
        "cpu_baseline": {"kind": "oracle", "value": value, "unit": "Mpixel-frames/s (fwd+bwd)",
                         "cores": info["threads"], "nproc": host["nproc"], "cpu_model": host["cpu_model"],
                         "sample": sample, "stages_s": info["stages_s"]},
        "e2e": {"value": value, "unit": "Mpixel-frames/s (fwd+bwd)", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def step_stats(ms_list) -> dict:
    a = np.asarray(ms_list, np.float64)
    return {"n": int(a.size), "median": float(np.median(a)), "p10": float(np.percentile(a, 10)),
            "p90": float(np.percentile(a, 90)), "mean": float(a.mean())}


def morton_scene(scene, dev):
    """The framework's particle storage order: the scene's
    particles permuted by ges_reorder into the Morton order of their means -- the same
    set of particles, stored the way training keeps them (reordered after every
    densify).  Returns (scene with permuted particles, reorder ms on the device)."""
    import dataclasses
    import torch
    import paper_2402_10128_b200 as G
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    G.reorder(params)   # warm-up (workspace allocation, first launch)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    _, perm = G.reorder(params)
    b.record()
    b.synchronize()
    p = perm.cpu().numpy().astype(np.int64)
    return dataclasses.replace(scene, particles=scene.particles.subset(p)), a.elapsed_time(b)


def workload_config(scene, cam, n):
    return {"workload": scene.name, "particles": scene.particles.P, "sh_degree": scene.particles.sh_degree,
            "width": cam.width, "height": cam.height, "tiles": ((cam.width + 15) // 16) * ((cam.height + 15) // 16),
            "rho": scene.rho, "phi_mode": "scale", "views_per_rank": 1, "particle_order": ORDER,
            "constants": {"tile": 16, "alpha_min": "1/255", "alpha_max": 0.99, "t_min": 1e-4, "dilation": 0.3,
                          "lambda_floor": 0.1, "jacobian_clamp": 1.3, "sh_offset": 0.5, "near": 0.2,
                          "rect": "alpha >= 0.98/255 box (R10)"},
            "step": "S1-S5 fwd+bwd of one view per rank (+NCCL allreduce of particle grads if N>1)",
            "parallelism": f"dp{n} (camera-view data parallel)",
            "l2": f"flushed between timed steps ({L2_FLUSH_BYTES >> 20} MB write); inputs 360 MB > L2"}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def run_ours(args) -> None:
    import torch
    import torch.distributed as dist

    import ges_inputs as gi
    import paper_2402_10128_b200 as G

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        # NCCL's INIT log (ranks, channels, NVLS) on stderr so the run shows which algorithm it chose
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")   # a hung peer aborts, not hangs
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(0)
    dev = torch.device("cuda", torch.cuda.current_device())
    stream = torch.cuda.current_stream()

    scene_input = gi.make_config(WORKLOAD_CFG)
    reorder_ms = None
    if ORDER == "morton":
        scene, reorder_ms = morton_scene(scene_input, dev)
    else:
        scene = scene_input
    cam = scene.cameras[rank % len(scene.cameras)]
    W, H, P = cam.width, cam.height, scene.particles.P
    st = G.Settings(rho=scene.rho)
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    grads = G.PlanarParams.zeros(P, scene.particles.sh_degree, dev)
    dL = torch.from_numpy(gi.upstream_grad(scene.seed, rank, W, H)).to(dev)
    image = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    n_eval = torch.zeros(W * H, dtype=torch.int32, device=dev)
    r = G.Renderer(P, W, H, device=dev)
    r.forward(params, cam, st, image)               # sizes the pair buffer (one sync)
    cnt = r.frame.counts()
    r.grow(int(cnt.slots))                          # capacity = 1.25 x slots, fixed from here on
    frame = r.frame
    flush = torch.empty(L2_FLUSH_BYTES, dtype=torch.uint8, device=dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)
    stage_names = ("preprocess", "sort", "render_fwd", "render_bwd_tiles", "backward_particles", "allreduce")
    NS = len(stage_names)

    def step(timers=None):
        def mark(i):
            if timers is not None:
                timers[i].record(stream)
        mark(0)
        G.ges_preprocess(params, cam, st, frame, stream)
        mark(1)
        G.ges_sort(frame, stream)
        mark(2)
        G.ges_render_fwd(frame, st, image, None, stream)
        mark(3)
        G.ges_render_bwd_tiles(st, frame, dL, stream)        # S5a } == ges_render_bwd,
        mark(4)
        G.ges_backward_particles(params, cam, st, frame, grads, False, stream)  # S5b } timed apart
        mark(5)
        if world > 1:
            dist.all_reduce(grads.flat)
        mark(6)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    cnt = frame.counts()
    assert not cnt.overflow

    # S1-S5 of one step captured once as a CUDA graph (the API is stream-ordered and
    # capture-safe); the timed loop replays it, the NCCL allreduce follows on the stream
    graph, graph_note = None, "off (--no-graph)"
    if not args.no_graph:
        try:
            graph = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.graph(graph, stream=cap):
                G.ges_preprocess(params, cam, st, frame, cap)
                G.ges_sort(frame, cap)
                G.ges_render_fwd(frame, st, image, None, cap)
                G.ges_render_bwd_tiles(st, frame, dL, cap)
                G.ges_backward_particles(params, cam, st, frame, grads, False, cap)
            stream.wait_stream(cap)
            for _ in range(args.warmup):
                graph.replay()
            torch.cuda.synchronize()
            graph_note = "S1-S5 replayed as one CUDA graph per step"
        except Exception as e:  # noqa: BLE001 -- fall back to direct launches, reported
            graph, graph_note = None, f"capture failed ({e}); direct launches"

    # ---- timed region: K steps ----
    step_ms = []
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        for _ in range(args.steps):
            flush.fill_(1)
            t0, t1 = ev(), ev()
            t0.record(stream)
            if graph is not None:
                graph.replay()
                if world > 1:
                    dist.all_reduce(grads.flat)
            else:
                step()
            t1.record(stream)
            t1.synchronize()
            step_ms.append(t0.elapsed_time(t1))
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    # ---- per-stage breakdown: the same steps launched directly with an event per stage ----
    stage_ms = np.zeros(len(stage_names))
    for _ in range(args.steps):
        flush.fill_(1)
        timers = [ev() for _ in range(NS + 1)]
        step(timers)
        timers[-1].synchronize()
        for i in range(NS):
            stage_ms[i] += timers[i].elapsed_time(timers[i + 1])
    if world > 1:
        dist.barrier()
    total_ms = float(sum(step_ms))
    t = torch.tensor([total_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    stage_ms /= args.steps
    value = world * W * H / (ms_per_step / 1e3) / 1e6
    comm = measure_comm(G, graph, step, grads, flush, stream, args.steps, ms_per_step, world, dev) if world > 1 else None

    # ---- the same step on the generated (input) particle order, for reference ----
    input_order = None
    if world == 1:   # the other storage order, for reference
        other = scene_input if ORDER == "morton" else morton_scene(scene_input, dev)[0]
        input_order = time_step_direct(G, other, cam, st, dL, flush, stream, args.steps, dev)

    # ---- forward-only throughput and the equivalent-Gaussian comparator (untimed above) ----
    fwd_ms = time_forward(G, params, cam, st, frame, image, flush, stream, args.steps)
    gauss = gaussian_equivalent(G, scene, cam, dev)
    g_frame = G.Renderer(P, W, H, pair_capacity=frame.pair_capacity, device=dev).frame
    g_ms = time_forward(G, gauss, cam, G.Settings(rho=scene.rho, gaussian_only=1), g_frame, image, flush, stream,
                        args.steps)

    # ---- one frame split into screen-tile bands over the ranks (forward, strong scaling) ----
    cam0 = scene.cameras[0]
    band_ms, band_pairs = time_band_forward(G, params, cam0, st, dev, flush, stream, args.steps, rank, world)

    # ---- the loss front end and a full training step with it ----
    loss_line = time_loss_front_end(G, params, cam, st, frame, grads, image, flush, stream, args.steps, dev)

    # ---- the exact GEF kernel of Eq. 2 on the same workload ----
    G.ges_preprocess(params, cam, st, frame, stream)
    G.ges_sort(frame, stream)
    G.ges_render_fwd(frame, st, image, None, stream)   # the phi-bar Gaussian image, for comparison
    exact = time_exact_kernel(G, params, cam, scene, dL, image, flush, stream, args.steps, dev)
    mix = time_mix1d(G, dev, stream, min(args.steps, 5))
    batches = {"cfg2": time_view_batch(G, 2, dev, stream, min(args.steps, 20), rank, world),
               "cfg4": time_view_batch(G, 4, dev, stream, min(args.steps, 10), rank, world)}
    small = time_small_configs(G, dev, stream, min(args.steps, 50)) if world == 1 else None
    union = time_union_compaction(G, scene, dev, stream, min(args.steps, 20)) if world == 1 else None
    shfac = time_sh_factorized(G, scene, dev, stream, min(args.steps, 20)) if world == 1 else None

    # ---- algorithmic work for the roofline (SURVEY.md §8(d) units) ----
    n_comp = torch.zeros(W * H, dtype=torch.int32, device=dev)
    G.ges_preprocess(params, cam, st, frame, stream)
    G.ges_sort(frame, stream)
    G.ges_render_fwd(frame, st, image, n_eval, stream, n_comp=n_comp)
    torch.cuda.synchronize()
    e_fwd = int(n_eval.to(torch.int64).sum().item())
    e_comp = int(n_comp.to(torch.int64).sum().item())
    e_bwd = int(frame.view("n_contrib", torch.int32, W * H).to(torch.int64).sum().item())
    peaks, peak_src = measured_peaks()
    clocks = clk.summary()
    sm_mhz = clocks["sm_mhz"] or peaks.get("sm_max_mhz", 1965.0)
    sms = torch.cuda.get_device_properties(dev).multi_processor_count
    alu_peak = sms * 128 * sm_mhz * 1e6 / 1e12  # T FP32 thread-instr/s
    K = scene.particles.K
    V = int(cnt.visible)
    s1_bytes = 48 * P + (12 * K + 56) * V + 4 * (P - V)
    rows = {
        "render_bwd_tiles": ("alu", K7_OPS * e_bwd / (stage_ms[3] / 1e3) / 1e12, alu_peak, "Tinstr/s",
                             f"K7: {K7_OPS} FP32 instr x sum n_contrib ({e_bwd})"),
        "render_fwd": ("alu", K6_OPS * e_fwd / (stage_ms[2] / 1e3) / 1e12, alu_peak, "Tinstr/s",
                       f"K6: {K6_OPS} FP32 instr x E_fwd = sum n_eval ({e_fwd})"),
        "preprocess": ("hbm", s1_bytes / (stage_ms[0] / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s",
                       f"K1: 48 P + (12K + 56) V + 4 (P - V) = {s1_bytes} B"),
        "sort": ("hbm", sort_algorithmic_bytes(P, V, int(cnt.pairs), row_incidences(frame), depth_passes(frame))
                 / (stage_ms[1] / 1e3) / 1e9, peaks["hbm_gbs"], "GB/s",
                 "K2-K5 counting their own passes: depth radix over V (item records in the last pass), "
                 "row lists, column counts, tile lists (one write of the M entries)"),
        "backward_particles": ("hbm", particle_bwd_bytes(P, V, K) / (stage_ms[4] / 1e3) / 1e9,
                               peaks["hbm_gbs"], "GB/s",
                               "K8: parameters and 2-D record read for visible particles, every gradient written"),
        "render_fwd_useful": ("alu", FWD_OPS * e_comp / (stage_ms[2] / 1e3) / 1e12, alu_peak, "Tinstr/s",
                              f"useful work only: {FWD_OPS} instr x composited (pixel, entry) pairs ({e_comp})"),
        "render_bwd_useful": ("alu", BWD_OPS * e_comp / (stage_ms[3] / 1e3) / 1e12, alu_peak, "Tinstr/s",
                              f"useful work only: {BWD_OPS} instr x composited (pixel, entry) pairs ({e_comp})"),
    }
    dom = max(range(5), key=lambda i: stage_ms[i])
    dname = stage_names[dom]
    bound, achieved, peak, unit, _ = rows[dname]
    traffic, traffic_src = committed_traffic(dname)

    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(G, scene, cam, st, frame, dL, dev, stream, args.steps, world)
    if rank == 0:
        cpu = None if args.no_cpu else cpu_baseline(scene, args.definitional_tiles)
        line = {
            "metric": METRIC, "value": value, "unit": "Mpixel-frames/s (fwd+bwd)", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic (seeded, DESIGN.md recipe)",
            "config": workload_config(scene, cam, world),
            "iters_per_s": 1e3 / ms_per_step,
            "step_ms_stats": step_stats(step_ms),
            "fwd_only": {"value": W * H / (fwd_ms / 1e3) / 1e6 * world, "unit": "Mpixel-frames/s",
                         "ms": fwd_ms, "fps_per_gpu": 1e3 / fwd_ms},
            "bands_fwd": {"value": cam0.width * cam0.height / (band_ms / 1e3) / 1e6, "unit": "Mpixel-frames/s",
                          "ms": band_ms, "frames_per_s": 1e3 / band_ms, "scaling": "strong",
                          "pairs_rank0": band_pairs,
                          "note": f"one config-3 frame split into {world} interleaved tile-row bands, S1-S4 per "
                                  f"rank + all_gather of the band pixels; device time, max over ranks"},
            "exact_beta_kernel": exact,
            "mix1d_sweep": mix,
            "view_batch_iters": batches,
            "small_configs": small,
            "allreduce_union_compaction": union,
            "allreduce_sh_factorized": shfac,
            "loss_front_end": loss_line,
            "vs_gaussian_equivalent": {"ges_fwd_ms": fwd_ms, "gaussian_fwd_ms": g_ms, "ratio": g_ms / fwd_ms,
                                       "note": "same footprints: log_scale + ln(phi-bar), gaussian_only=1"},
            "launch": graph_note,
            "comm": comm,
            "particle_order": {"order": ORDER, "reorder_ms": reorder_ms, "other_order": input_order,
                               "note": "order = the particle storage order timed (input: as generated; morton: "
                                       "ges_reorder once before timing); other_order = the same step, direct "
                                       "launches, in the other order"},
            "stages_ms": {n: float(stage_ms[i]) for i, n in enumerate(stage_names)},
            "stages_note": "per-stage CUDA events around direct launches of the same step (not the graph replay)",
            "counts": {"particles": P, "visible": V, "pairs": int(cnt.pairs), "slots": int(cnt.slots),
                       "tiles": frame.c.tiles_x * frame.c.tiles_y, "evals_fwd": e_fwd, "sum_n_contrib": e_bwd,
                       "composited": e_comp, "depth_passes": depth_passes(frame)},
            "roofline": {"kernel": dname, "bound": bound, "achieved": achieved, "peak": peak, "unit": unit,
                         "frac": achieved / peak, "traffic": traffic, "traffic_source": traffic_src,
                         "peak_source": peak_src if bound == "hbm" else
                         f"derived: {sms} SMs x 128 FP32 lanes x {sm_mhz:.0f} MHz (median SM clock under load)",
                         "all": {k: {"bound": v[0], "achieved": v[1], "peak": v[2], "unit": v[3],
                                     "frac": v[1] / v[2], "work": v[4]} for k, v in rows.items()}},
            "cpu_baseline": cpu, "e2e": e2e,
            "gpu_launches": LAUNCHES_PER_STEP * args.steps,
            "clocks": clocks,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


# FP32-pipe instructions per forward evaluation (K6: E_fwd = sum over pixels of the
# list entries evaluated before the pixel terminates) and per backward entry (K7: sum n_contrib)
K6_OPS = 15
K7_OPS = 45
# useful work only: FP32 instructions the method needs per composited (pixel, entry)
FWD_OPS = 20
BWD_OPS = 38
# kernels per step: preprocess, depth sort + item records (one cooperative kernel), binning (rows,
# column counts, columns + ranges), fwd, bwd tiles, particle bwd (+ the frame's zero-region memset)
LAUNCHES_PER_STEP = 1 + 1 + 3 + 1 + 1 + 1


def measure_comm(G, graph, step, grads, flush, stream, steps, ms_per_step, world, dev):
    """N > 1: exposed communication = the step with its
    allreduce minus the same step without it (device time, max over ranks), and the
    NCCL allreduce of the gradient buffer alone: algorithm and bus bandwidth
    (busBW = algBW x 2 (N - 1) / N)."""
    import torch
    import torch.distributed as dist
    ev = lambda: torch.cuda.Event(enable_timing=True)

    def timed(fn):
        ms = []
        for _ in range(steps):
            flush.fill_(1)
            dist.barrier()
            torch.cuda.synchronize()
            a, b = ev(), ev()
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        t = torch.tensor([sum(ms) / len(ms)], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    no_comm = timed(graph.replay if graph is not None else (lambda: None))
    ar = timed(lambda: dist.all_reduce(grads.flat))
    nbytes = grads.flat.numel() * 4
    alg = nbytes / (ar / 1e3) / 1e9
    env = {k: os.environ.get(k) for k in ("NCCL_NVLS_ENABLE", "NCCL_ALGO", "NCCL_PROTO") if os.environ.get(k)}
    return {"ms_step_with_allreduce": ms_per_step, "ms_step_without_collective": no_comm,
            "exposed_comm_ms": ms_per_step - no_comm, "allreduce_ms": ar, "allreduce_bytes": nbytes,
            "algbw_GBps": alg, "busbw_GBps": alg * 2 * (world - 1) / world,
            "nccl_version": ".".join(map(str, torch.cuda.nccl.version())), "nccl_env": env,
            "note": "NCCL_DEBUG=INFO / SUBSYS=INIT on stderr shows the channels and whether NVLS was chosen"}


def preprocess_bytes(P, V, deg):
    K = (deg + 1) ** 2
    # reads: 12 floats/particle (mean, log-scale, quat, logit, beta) for all, SH 3K floats for visible;
    # writes: depth 4 + payload 36 + radius 4 + rect 8 + status/flags 2 + d rgb/d dir 36 + key 4 = 94 B/particle
    return P * (4 * 12 + 94) + V * 4 * 3 * K


def row_incidences(frame):
    """Row-list entries of the frame: sum over visible particles of their rect heights."""
    import torch
    return int(frame.view("row_count", torch.int32, frame.c.band_rows).sum().item())


def depth_passes(frame):
    """Passes the depth sort ran: 9-bit digits over bits(max visible key - bits(near_z))."""
    import torch
    kmax = int(frame.view("counters", torch.int64, 16)[7].item()) & 0xffffffff
    span = max(0, kmax - int(frame.c.depth_key_base))
    return max(1, -(-span.bit_length() // 9))


def sort_algorithmic_bytes(P, V, M, I, passes):
    # depth sort: phase H and pass 0 read the P keys (the ids are the indices); pass 0 writes V
    # (key, id); every middle pass reads and writes V (key, id); the last reads V (key, id) and writes
    # the V ids and 8-B item records, gathering the 8-B rects
    depth = P * 4 * 2 + V * 8 + max(0, passes - 2) * V * 16 + (V * 8 if passes > 1 else 0) + V * (4 + 8 + 8)
    # binning: the rows read the V item records and write the I row-list entries (8 B; I = sum of
    # rect heights); the column counts and the column binning read them; the M list entries are
    # written once.  Row counts, look-back words, tile counts and ranges are O(rows x tiles), small
    binning = V * 8 + I * 8 * 3 + M * 4
    return depth + binning


def particle_bwd_bytes(P, V, K):
    # reads: status/flags 2 B for all; params 12 floats + d rgb/d dir 9 floats + 48-B 2-D record for
    # visible; writes: (14 + 3K) gradient floats for all (overwrite) + 48-B record reset
    return P * 2 + V * (4 * (12 + 9) + 48 + 48) + P * 4 * (11 + 3 * K)


def time_step_direct(G, scene, cam, st, dL, flush, stream, steps, dev):
    """S1-S5 of one view, direct launches with an event per stage (L2 flushed between
    steps): mean ms per step and per stage."""
    import torch
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    grads = G.PlanarParams.zeros(params.P, params.sh_degree, dev)
    r = G.Renderer(params.P, cam.width, cam.height, device=dev)
    img = r.forward(params, cam, st)
    r.grow(int(r.frame.counts().slots))
    frame = r.frame
    names = ("preprocess", "sort", "render_fwd", "render_bwd_tiles", "backward_particles")
    acc = np.zeros(len(names))
    for it in range(steps + 3):
        flush.fill_(1)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(len(names) + 1)]
        ev[0].record(stream)
        G.ges_preprocess(params, cam, st, frame, stream); ev[1].record(stream)
        G.ges_sort(frame, stream); ev[2].record(stream)
        G.ges_render_fwd(frame, st, img, None, stream); ev[3].record(stream)
        G.ges_render_bwd_tiles(st, frame, dL, stream); ev[4].record(stream)
        G.ges_backward_particles(params, cam, st, frame, grads, False, stream); ev[5].record(stream)
        ev[-1].synchronize()
        if it >= 3:
            acc += [ev[k].elapsed_time(ev[k + 1]) for k in range(len(names))]
    acc /= steps
    return {"ms_per_step": float(acc.sum()), "stages_ms": {n: float(v) for n, v in zip(names, acc)},
            "launch": "direct launches"}


def time_forward(G, params, cam, st, frame, image, flush, stream, steps):
    import torch
    ms = []
    for _ in range(2):
        G.ges_preprocess(params, cam, st, frame, stream)
        G.ges_sort(frame, stream)
        G.ges_render_fwd(frame, st, image, None, stream)
    for _ in range(steps):
        flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        G.ges_preprocess(params, cam, st, frame, stream)
        G.ges_sort(frame, stream)
        G.ges_render_fwd(frame, st, image, None, stream)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    return float(statistics.mean(ms))


def time_band_forward(G, params, cam, st, dev, flush, stream, steps, rank, world):
    """Forward of ONE frame split into `world` interleaved screen-tile bands
    (BASELINE config 3): each rank runs S1-S4 on its band, then
    the band pixels are all-gathered (NCCL) into the full image on every rank.
    Device time (CUDA events), max over ranks.  Strong scaling."""
    import torch
    import torch.distributed as dist
    from paper_2402_10128_b200 import dist as gdist
    bst = gdist.band_settings(st, rank, world)
    r = G.Renderer(params.P, cam.width, cam.height, device=dev)
    img = torch.zeros((3, cam.height, cam.width), dtype=torch.float32, device=dev)
    r.forward(params, cam, bst, img)
    r.grow(int(r.frame.counts().slots))
    frame = r.frame

    def once():
        G.ges_preprocess(params, cam, bst, frame, stream)
        G.ges_sort(frame, stream)
        G.ges_render_fwd(frame, bst, img, None, stream)
        return gdist.gather_bands(img, rank, world)
    for _ in range(2):
        once()
    ms = []
    for _ in range(steps):
        flush.fill_(1)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        once()
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    t = torch.tensor([float(statistics.mean(ms))], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item()), int(frame.counts().pairs)



MIX_N = (2, 5, 8, 10, 15, 20, 50, 100)    # PAPER.md:628 component counts
MIX_MUFU = {"gmm": (1, 1), "dog": (2, 2), "log": (1, 1), "gef": (3, 4)}   # ex2/lg2/rcp per (pass 1, pass 2) eval


def time_mix1d(G, dev, stream, steps_timed, reps=20, n=512, fit_steps=100):
    """NEXT-4: the paper's 1-D mixture sweep in one launch --
    6 signals x N in {2, 5, 8, 10, 15, 20, 50, 100} x 4 models x {real, positive}
    weights x `reps` seeded starts = 7680 independent Adam fits of `fit_steps` steps
    on an n-sample grid over [-2, 2] (signal width 1), heavy runs first.  Roofline:
    MUFU ex2/lg2/rcp results per (sample, component) evaluation against the rate a
    probe kernel measures on this GPU."""
    import numpy as np
    import torch
    kinds = ("square", "triangle", "parabolic", "half_sinusoid", "exponential", "gaussian")
    targets = torch.stack([G.ges_mix_signal(k, 1.0, -2.0, 2.0, n) for k in kinds])
    rng = np.random.default_rng(2402)
    specs = []
    for N in sorted(MIX_N, reverse=True):
        for model in G.MIX_MODELS:
            for pos in (True, False):
                for t in range(len(kinds)):
                    for _ in range(reps):
                        specs.append((model, pos, N, t))
    stride = 3 * max(MIX_N) + 1
    th = np.zeros((len(specs), stride), np.float32)
    for r, (model, pos, N, t) in enumerate(specs):
        th[r, 0:N] = rng.uniform(-1.5, 1.5, N)
        th[r, N:2 * N] = rng.uniform(0.1, 0.5, N)
        th[r, 2 * N:3 * N] = rng.normal(-1.0, 0.3, N) if pos else rng.normal(0.3, 0.2, N)
        th[r, 3 * N] = 2.0
    th0 = torch.from_numpy(th).to(dev)
    runs = G.mix_runs(specs)
    sw = G.MixSweep(runs, th0.clone(), targets, -2.0, 2.0)
    sw.fit(2, stream=stream)                       # warm-up
    ms = []
    for _ in range(max(1, steps_timed)):
        sw.params.copy_(th0)
        sw.m.zero_()
        sw.v.zero_()
        sw.t = 0
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        sw.fit(fit_steps, stream=stream)
        b.record(stream)
        b.synchronize()
        ms.append(a.elapsed_time(b))
    t = float(statistics.median(ms))
    loss = sw.loss.cpu().numpy()
    evals = sum(N for (_, _, N, _) in specs) * n
    mufu = sum(N * n * ((MIX_MUFU[m][0] + MIX_MUFU[m][1]) * fit_steps + MIX_MUFU[m][0]) for (m, _, N, _) in specs)
    # the probe: 8 chains x iters ex2 per thread
    out = torch.empty(148 * 8 * 256, dtype=torch.float32, device=dev)
    lib = G.load()
    import ctypes as C
    iters, blocks = 4096, 148 * 8
    for _ in range(2):
        lib.ges_probe_mufu(C.c_void_p(out.data_ptr()), iters, blocks, C.c_void_p(stream.cuda_stream))
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    lib.ges_probe_mufu(C.c_void_p(out.data_ptr()), iters, blocks, C.c_void_p(stream.cuda_stream))
    b.record(stream)
    b.synchronize()
    probe = 8.0 * iters * blocks * 256 / (a.elapsed_time(b) / 1e3) / 1e12
    achieved = mufu / (t / 1e3) / 1e12
    finite = np.isfinite(loss)
    return {"runs": len(specs), "fit_steps": fit_steps, "samples": n, "ms": t,
            "fits_per_s": len(specs) / (t / 1e3),
            "component_sample_evals_per_s": evals * (2 * fit_steps + 1) / (t / 1e3),
            "roofline": {"bound": "mufu", "achieved": achieved, "peak": probe, "unit": "T results/s",
                         "frac": achieved / probe, "peak_source": "ges_probe_mufu (8 ex2 chains/thread) on this GPU"},
            "finite_runs": int(finite.sum()), "median_final_loss": float(np.median(loss[finite])) if finite.any() else None,
            "note": "NEXT-4 sweep: 7680 Adam fits (GMM/DoG/LoG/GEF, 6 signals, 8 N, real/positive weights, 20 "
                    "seeds), one CTA per fit"}


def time_view_batch(G, cfg, dev, stream, steps, rank, world):
    """SURVEY.md §8(d) iters/s: a fixed global batch of 8 views split 8/N per rank --
    fwd+bwd of each view with the gradients accumulated, the NCCL allreduce (N > 1),
    then a dependent update through ges_adam_step with every LR 0 (parameters
    unchanged).  Config 2: its 8 orbit views; config 4: 8 of its 64 views.  Device
    time, max over ranks; strong scaling (the global batch is fixed)."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import ges_inputs as gi
    scene = gi.make_config(cfg)
    if ORDER == "morton":
        scene, _ = morton_scene(scene, dev)
    cams = scene.cameras[:8] if cfg == 2 else [scene.cameras[k] for k in
                                               np.random.default_rng(2402).choice(len(scene.cameras), 8, replace=False)]
    mine = [c for k, c in enumerate(cams) if k % world == rank]
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    P, deg = params.P, params.sh_degree
    grads = G.PlanarParams.zeros(P, deg, dev)
    st = G.Settings(rho=scene.rho)
    W, H = cams[0].width, cams[0].height
    r = G.Renderer(P, W, H, device=dev)
    img = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    dLs = [torch.from_numpy(gi.upstream_grad(scene.seed, k, W, H)).to(dev) for k in range(len(mine))]
    for c in mine:                                    # size the frame for the largest view
        r.forward(params, c, st, img)
        r.grow(int(r.frame.counts().slots))
    zero = G.AdamSettings(lr_pos_init=0.0, lr_pos_final=0.0, lr_feature=0.0, lr_opacity=0.0, lr_scaling=0.0,
                          lr_rotation=0.0, lr_shape=0.0)
    from paper_2402_10128_b200 import dist as gdist
    opt = gdist.ShardedAdam(params, zero, rank, world)   # N > 1: reduce-scatter, 1/N Adam, all-gather
    frame = r.frame
    n_el = params.flat.numel()
    b0, cnt, _ = gdist.shard_range(n_el, rank, world)

    def views():
        for k, c in enumerate(mine):
            G.ges_preprocess(params, c, st, frame, stream)
            G.ges_sort(frame, stream)
            G.ges_render_fwd(frame, st, img, None, stream)
            G.ges_render_bwd(params, c, st, frame, dLs[k], grads, k > 0, stream)

    def step():
        views()
        opt.step(params, grads, stream=stream)

    def step_local():   # the same work without any collective: views + this rank's Adam shard
        views()
        opt.adam.step_range(params, grads.flat.view(-1)[b0:b0 + cnt], b0, cnt, stream) if world > 1 else \
            opt.adam.step(params, grads, stream)

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        b.synchronize()
        t = torch.tensor([a.elapsed_time(b) / steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    ms_direct = timed(step)
    ms_local = timed(step_local) if world > 1 else ms_direct
    # N = 1: the whole iteration (8 views x S1-S5, Adam) captured once as a CUDA graph
    ms_graph = None
    if world == 1:
        try:
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.graph(g, stream=cap):
                for k, c in enumerate(mine):
                    G.ges_preprocess(params, c, st, frame, cap)
                    G.ges_sort(frame, cap)
                    G.ges_render_fwd(frame, st, img, None, cap)
                    G.ges_render_bwd(params, c, st, frame, dLs[k], grads, k > 0, cap)
                opt.adam.step(params, grads, stream=cap)
            stream.wait_stream(cap)
            ms_graph = timed(g.replay)
        except Exception as e:  # noqa: BLE001 -- reported, the direct number stands
            ms_graph = f"capture failed: {e}"
    # N = 1, views alternating between two streams and two frames (dist.ViewDataParallel
    # streams=2): one view's latency-bound phases overlap the other's; S5b in view order
    ms_two = None
    if world == 1 and len(mine) > 1:
        try:
            r2 = G.Renderer(P, W, H, pair_capacity=frame.c.pair_capacity, device=dev)
            frames, imgs = [frame, r2.frame], [img, torch.empty_like(img)]
            g2 = torch.cuda.CUDAGraph()
            cap, side = torch.cuda.Stream(), torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.graph(g2, stream=cap):
                side.wait_stream(cap)
                prev = None
                for k, c in enumerate(mine):
                    q, f = (cap, frames[0]) if k % 2 == 0 else (side, frames[1])
                    G.ges_preprocess(params, c, st, f, q)
                    G.ges_sort(f, q)
                    G.ges_render_fwd(f, st, imgs[k % 2], None, q)
                    G.ges_render_bwd_tiles(st, f, dLs[k], q)
                    if prev is not None:
                        q.wait_event(prev)
                    G.ges_backward_particles(params, c, st, f, grads, k > 0, q)
                    prev = torch.cuda.Event()
                    prev.record(q)
                cap.wait_stream(side)
                opt.adam.step(params, grads, stream=cap)
            stream.wait_stream(cap)
            ms_two = timed(g2.replay)
            assert not r2.frame.counts().overflow
        except Exception as e:  # noqa: BLE001 -- reported, the one-stream number stands
            ms_two = f"capture failed: {e}"
    ms = ms_graph if isinstance(ms_graph, float) else ms_direct
    launch = "CUDA graph" if ms is ms_graph else "direct"
    if isinstance(ms_two, float) and ms_two < ms:
        ms, launch = ms_two, "CUDA graph, views alternating between two streams"
    assert not frame.counts().overflow
    return {"config": gi.CONFIG_NAMES[cfg], "views_per_iter": 8, "views_per_rank": len(mine), "ms_per_iter": ms,
            "ms_per_iter_direct_launches": ms_direct, "ms_per_iter_one_stream_graph": ms_graph,
            "ms_per_iter_two_streams": ms_two, "launch": launch,
            "iters_per_s": 1e3 / ms, "value": 8 * W * H / (ms / 1e3) / 1e6, "unit": "Mpixel-frames/s (fwd+bwd)",
            "scaling": "strong", "ms_without_collectives": ms_local if world > 1 else ms,
            "exposed_comm_ms": (ms_direct - ms_local) if world > 1 else 0.0,  # (both direct launches at N > 1)
            "optimizer": "Adam (all LRs 0); N > 1: ZeRO-1 -- reduce-scatter of the gradients, each rank's 1/N range "
                         "updated, all-gather of the parameters (dist.ShardedAdam)",
            "gradient_bytes": 4 * n_el}


def time_small_configs(G, dev, stream, steps):
    """Mpixel-frames/s of the fwd+bwd step on configs 0-2 ('configs 0-2 also
    reported'); config 1 at beta = 2, config 2 on its first view."""
    import torch
    import ges_inputs as gi
    out = {}
    for cfg, kw in ((0, {}), (1, {"beta_value": 2.0}), (2, {})):
        scene = gi.make_config(cfg, **kw)
        if ORDER == "morton":
            scene, _ = morton_scene(scene, dev)
        cam = scene.cameras[0]
        params = G.PlanarParams.from_inputs(scene.particles, device=dev)
        grads = G.PlanarParams.zeros(params.P, params.sh_degree, dev)
        st = G.Settings(rho=scene.rho)
        r = G.Renderer(params.P, cam.width, cam.height, device=dev)
        img = torch.empty((3, cam.height, cam.width), dtype=torch.float32, device=dev)
        r.forward(params, cam, st, img)
        r.grow(int(r.frame.counts().slots))
        dL = torch.from_numpy(gi.upstream_grad(scene.seed, 0, cam.width, cam.height)).to(dev)
        frame = r.frame

        def step():
            G.ges_preprocess(params, cam, st, frame, stream)
            G.ges_sort(frame, stream)
            G.ges_render_fwd(frame, st, img, None, stream)
            G.ges_render_bwd(params, cam, st, frame, dL, grads, False, stream)

        for _ in range(3):
            step()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            step()
        b.record(stream)
        b.synchronize()
        ms = a.elapsed_time(b) / steps
        # the same step captured once as a CUDA graph and replayed (launch overhead gone)
        ms_graph = None
        try:
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.graph(g, stream=cap):
                G.ges_preprocess(params, cam, st, frame, cap)
                G.ges_sort(frame, cap)
                G.ges_render_fwd(frame, st, img, None, cap)
                G.ges_render_bwd(params, cam, st, frame, dL, grads, False, cap)
            stream.wait_stream(cap)
            for _ in range(3):
                g.replay()
            torch.cuda.synchronize()
            a.record(stream)
            for _ in range(steps):
                g.replay()
            b.record(stream)
            b.synchronize()
            ms_graph = a.elapsed_time(b) / steps
        except Exception as e:  # noqa: BLE001 -- reported, not fatal
            ms_graph = f"capture failed: {e}"
        out[gi.CONFIG_NAMES[cfg]] = {"ms": ms, "value": cam.width * cam.height / (ms / 1e3) / 1e6,
                                     "unit": "Mpixel-frames/s (fwd+bwd)", "ms_cuda_graph": ms_graph}
    return out


def time_union_compaction(G, scene, dev, stream, steps):
    """SURVEY.md §8(e) visible-union compaction, measured on one GPU: the union of the
    visible sets of config 3's 8 bench views (what 8 ranks would OR together), and
    the device time of ges_grad_pack + ges_grad_unpack on the 60 x P planar gradient
    -- against the bytes the allreduce would no longer move."""
    import torch
    from paper_2402_10128_b200 import dist as gdist
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    P, C = params.P, params.flat.shape[0]
    red = gdist.VisibleUnionReducer(P, C, dev)
    st = G.Settings(rho=scene.rho)
    cams = scene.cameras[:8]
    r = G.Renderer(P, cams[0].width, cams[0].height, device=dev)
    for c in cams:
        r.forward(params, c, st)
        red.add_view(r.frame)
    union = int(red.mask.sum().item())
    flat = torch.randn((C, P), dtype=torch.float32, device=dev)
    packed, u = red.pack(flat, red.mask, force=True)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    a, b, c = ev(), ev(), ev()
    a.record(stream)
    for _ in range(steps):                      # device time only: no host read of U inside
        red.index(red.mask, stream)
    b.record(stream)
    for _ in range(steps):
        red.pack_indexed(flat, stream)
        red.unpack(packed, None, flat, stream)
    c.record(stream)
    c.synchronize()
    return {"views": len(cams), "union_particles": union, "union_frac": union / P,
            "allreduce_bytes_dense": 4 * C * P, "allreduce_bytes_compact": 4 * C * union,
            "index_ms": a.elapsed_time(b) / steps, "pack_unpack_ms": b.elapsed_time(c) / steps,
            "used_when": "union <= 0.5 P (VisibleUnionReducer.max_union); above it the dense allreduce runs",
            "note": "view-DP allreduce of only the union of the ranks' visible particles (one host read of U)"}

def time_sh_factorized(G, scene, dev, stream, steps):
    """DESIGN.md §8 SH-factorised view-DP exchange, measured on one GPU: the device time of
    ges_sh_grad_from_colour rebuilding the 3K SH planes from 8 views' dL/drgb (what every
    rank runs after the all-gather at N = 8, one view per rank), and the bytes each rank
    receives in the exchange against the dense allreduce's (NVLS: ~ the buffer once)."""
    import torch
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    P, C, K = params.P, params.flat.shape[0], scene.particles.K
    cams = G.camera_rows(scene.cameras[:8], device=dev)
    n = cams.shape[0]
    st = G.Settings(rho=scene.rho)
    r = G.Renderer(P, scene.cameras[0].width, scene.cameras[0].height, device=dev)
    grads = G.PlanarParams.zeros(P, params.sh_degree, dev)
    drgb = torch.zeros((n, 3, P), dtype=torch.float32, device=dev)
    for v, c in enumerate(scene.cameras[:n]):    # real per-view colour gradients (sparsity as in training)
        r.forward(params, c, st)
        dLv = torch.randn((3, c.height, c.width), device=dev)
        r.backward(params, c, st, dLv, grads=grads, accumulate=v > 0, drgb=drgb[v])
    out = torch.empty_like(params.sh)
    G.sh_grad_from_colour(params, cams, drgb, out=out, stream=stream)
    ev = lambda: torch.cuda.Event(enable_timing=True)
    a, b = ev(), ev()
    a.record(stream)
    for _ in range(steps):
        G.sh_grad_from_colour(params, cams, drgb, out=out, stream=stream)
    b.record(stream)
    b.synchronize()
    err = float(((out - grads.sh).abs().max() / (grads.sh.abs().max() + 1e-30)).item())
    ms = a.elapsed_time(b) / steps
    kbytes = 12 * P + 12 * n * P + 4 * 3 * K * P
    return {"views": n, "sh_from_colour_ms": ms, "sh_from_colour_gbs": kbytes / (ms / 1e3) / 1e9,
            "max_rel_diff_vs_accumulated_sh": err,
            "exchange_bytes_per_rank_dense": 4 * C * P,
            "exchange_bytes_per_rank_factorized": 4 * (C - 3 * K) * P + 4 * 3 * (n - 1) * P,
            "note": "N = 8, one view per rank: allreduce of the 12 non-SH planes + all-gather of the "
                    "other 7 views' 3-float dL/drgb, then this kernel on every rank"}


def time_loss_front_end(G, params, cam, st, frame, grads, image, flush, stream, steps, dev):
    """Eq. 9's loss on the bench frame (mask M_omega at omega = 0.75, L1 + SSIM + L_omega and
    dL/dimage) alone, and one training step that uses it: S1-S4, the loss, S5.  The target
    image is a synthetic smooth field (no dataset)."""
    import torch
    W, H = cam.width, cam.height
    yy = torch.linspace(0, 1, H, device=dev)[:, None]
    xx = torch.linspace(0, 1, W, device=dev)[None, :]
    gt = torch.stack([0.5 + 0.3 * torch.sin(9 * xx + 4 * yy), 0.5 + 0.3 * torch.cos(7 * yy - 3 * xx),
                      0.4 + 0.2 * torch.sin(13 * xx * yy)]).contiguous()
    loss = G.Loss(W, H, device=dev)
    mask = loss.mask(gt, 0.75, stream=stream)
    dL = torch.empty_like(image)

    def only_loss():
        loss.mask(gt, 0.75, mask, stream=stream)
        loss(image, gt, mask, dL, stream=stream)

    def train_step():
        G.ges_preprocess(params, cam, st, frame, stream)
        G.ges_sort(frame, stream)
        G.ges_render_fwd(frame, st, image, None, stream)
        loss.mask(gt, 0.75, mask, stream=stream)
        loss(image, gt, mask, dL, stream=stream)
        G.ges_render_bwd(params, cam, st, frame, dL, grads, False, stream)

    # the optimizer on a copy of the parameters (the timed steps must not drift the bench scene)
    pcopy = G.PlanarParams(params.flat.clone(), params.P, params.sh_degree)
    opt = G.Adam(pcopy)

    def adam():
        opt.step(pcopy, grads, stream=stream)

    out = {}
    for name, fn in (("loss", only_loss), ("train_step", train_step), ("adam", adam)):
        for _ in range(3):
            fn()
        ms = []
        for _ in range(steps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        out[name] = float(statistics.mean(ms))
    n = 3 * W * H
    moved = 4 * (2 * n + 3 * n + 3 * n + 2 * n + n)   # fwd reads I, I_gt, writes 3 SSIM partials; bwd reads them, I, I_gt, writes dL/dI
    n_el = params.flat.numel()
    adam_bytes = 28 * n_el   # reads p, g, m, v; writes p, m, v (fp32)
    peaks, _ = measured_peaks()
    return {"loss_ms": out["loss"], "loss_GBps_moved": moved / (out["loss"] / 1e3) / 1e9,
            "adam": {"ms": out["adam"], "GBps": adam_bytes / (out["adam"] / 1e3) / 1e9,
                     "frac_hbm": adam_bytes / (out["adam"] / 1e3) / 1e9 / peaks["hbm_gbs"],
                     "bytes": adam_bytes, "note": "fused Adam over all 60 x P planar parameters (NEXT-2)"},
            "train_iteration_ms": out["train_step"] + out["adam"],
            "train_step_ms": out["train_step"],
            "train_step": {"value": W * H / (out["train_step"] / 1e3) / 1e6, "unit": "Mpixel-frames/s (fwd+loss+bwd)"},
            "note": "Eq. 9 (L1 + SSIM + L_omega at omega = 0.75) on the bench frame; train_step = S1-S4 + mask + "
                    "loss + S5 with the loss's dL/dimage"}


def time_exact_kernel(G, params, cam, scene, dL, image_phi, flush, stream, steps, dev):
    """Forward and fwd+bwd step with the exact GEF kernel (ges_settings.kernel = 1) on the
    bench workload, timed like the main step; plus how far its image lies from the
    phi-bar Gaussian rasterization's (the approximation the paper makes)."""
    import torch
    W, H, P = cam.width, cam.height, params.P
    st = G.Settings(rho=scene.rho, kernel=1)
    r = G.Renderer(P, W, H, device=dev)
    img = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    r.forward(params, cam, st, img)
    r.grow(int(r.frame.counts().slots))
    frame = r.frame
    grads = G.PlanarParams.zeros(P, params.sh_degree, dev)

    def fwd():
        G.ges_preprocess(params, cam, st, frame, stream)
        G.ges_sort(frame, stream)
        G.ges_render_fwd(frame, st, img, None, stream)

    def step():
        fwd()
        G.ges_render_bwd(params, cam, st, frame, dL, grads, False, stream)

    out = {}
    for name, fn in (("fwd", fwd), ("fwd_bwd", step)):
        for _ in range(3):
            fn()
        ms = []
        for _ in range(steps):
            flush.fill_(1)
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ms.append(a.elapsed_time(b))
        out[name + "_ms"] = float(statistics.mean(ms))
    fwd()
    torch.cuda.synchronize()
    cnt = frame.counts()
    d = (img - image_phi).abs()
    return {"fwd": {"value": W * H / (out["fwd_ms"] / 1e3) / 1e6, "unit": "Mpixel-frames/s", "ms": out["fwd_ms"]},
            "fwd_bwd": {"value": W * H / (out["fwd_bwd_ms"] / 1e3) / 1e6, "unit": "Mpixel-frames/s (fwd+bwd)",
                        "ms": out["fwd_bwd_ms"]},
            "pairs": int(cnt.pairs), "visible": int(cnt.visible),
            "image_vs_phi_bar_gaussian": {"max_abs": float(d.max().item()), "mean_abs": float(d.mean().item())},
            "note": "Eq. 2 per pixel (no phi-bar); footprints follow Q <= (2 ln(255 kappa))^(2/beta), "
                    "so beta < 2 particles cover far more tiles"}


def gaussian_equivalent(G, scene, cam, dev):
    """The equivalent Gaussian rasterizer's input: same particles with the
    phi-bar factor folded into the log-scales (SCALE mode) so that footprints
    and pair counts are identical; rendered with gaussian_only = 1."""
    import torch
    p = scene.particles
    beta = p.beta.astype(np.float64)
    phi = 2.0 / (1.0 + np.exp(-(scene.rho * beta - 2 * scene.rho)))
    q = p.subset(slice(None))
    q.log_scale = (p.log_scale.astype(np.float64) + np.log(phi)[None, :]).astype(np.float32)
    return G.PlanarParams.from_inputs(q, device=dev)


def run_e2e(G, scene, cam, st, frame, dL_dev, dev, stream, steps, world):
    """Public-API step with HOST inputs: pinned particles + dL/dimage copied in,
    image copied out, every step, inside the timed region.  The copies run on a
    second stream, double-buffered: step k+1's inputs upload while step k computes
    (the region starts before step 0's upload and ends after the last image lands
    on the host), so a step costs max(PCIe transfer, compute)."""
    import torch
    P, deg = scene.particles.P, scene.particles.sh_degree
    host_params = G.PlanarParams.from_inputs(scene.particles, device="cpu", pin_memory=True)
    host_dL = dL_dev.cpu().pin_memory()
    host_img = [torch.empty((3, cam.height, cam.width), dtype=torch.float32).pin_memory() for _ in range(2)]
    dparams = [G.PlanarParams.empty(P, deg, dev) for _ in range(2)]
    ddL = [torch.empty_like(dL_dev) for _ in range(2)]
    img = [torch.empty((3, cam.height, cam.width), dtype=torch.float32, device=dev) for _ in range(2)]
    grads = G.PlanarParams.zeros(P, deg, dev)
    copy = torch.cuda.Stream(device=dev)
    ev = lambda: torch.cuda.Event()
    uploaded = [ev(), ev()]   # inputs of buffer b are on the device
    consumed = [ev(), ev()]   # step using buffer b finished (its inputs and image may be reused)
    drained = [ev(), ev()]    # image of buffer b is on the host

    def upload(b):
        with torch.cuda.stream(copy):
            copy.wait_event(consumed[b])
            dparams[b].flat.copy_(host_params.flat, non_blocking=True)
            ddL[b].copy_(host_dL, non_blocking=True)
            uploaded[b].record(copy)

    def compute(b):
        stream.wait_event(uploaded[b])
        stream.wait_event(drained[b])
        G.ges_preprocess(dparams[b], cam, st, frame, stream)
        G.ges_sort(frame, stream)
        G.ges_render_fwd(frame, st, img[b], None, stream)
        G.ges_render_bwd(dparams[b], cam, st, frame, ddL[b], grads, False, stream)
        consumed[b].record(stream)
        with torch.cuda.stream(copy):
            copy.wait_event(consumed[b])
            host_img[b].copy_(img[b], non_blocking=True)
            drained[b].record(copy)

    def run(n):
        upload(0)
        for k in range(n):
            if k + 1 < n:
                upload((k + 1) & 1)
            compute(k & 1)
        stream.wait_stream(copy)

    for e in consumed + drained:
        e.record(stream)
    run(2)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(stream)
    copy.wait_stream(stream)
    run(steps)
    b.record(stream)
    b.synchronize()
    ms = a.elapsed_time(b) / steps
    h2d = host_params.flat.numel() * 4 + host_dL.numel() * 4
    d2h = host_img[0].numel() * 4
    out = {"value": world * cam.width * cam.height / (ms / 1e3) / 1e6, "unit": "Mpixel-frames/s (fwd+bwd)",
           "ms_per_step": ms, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "h2d_GBps": h2d / (ms / 1e3) / 1e9,
           "path": "pinned host -> device copy (second stream, double-buffered against the previous step's "
                   "compute), ges_preprocess/sort/render_fwd/render_bwd, image -> host"}
    out["train_step"] = run_e2e_train(G, scene, cam, st, frame, dev, stream, steps, world)
    return out


def run_e2e_train(G, scene, cam, st, frame, dev, stream, steps, world):
    """A training iteration as a user runs it: parameters and Adam state resident
    on the device, the view's ground-truth image copied in from pinned host memory
    every step, S1-S4 + the Eq. 9 loss (mask at omega = 0.75) + S5 + Adam, and the
    loss read back to the host every step."""
    import torch
    P, deg = scene.particles.P, scene.particles.sh_degree
    W, H = cam.width, cam.height
    params = G.PlanarParams.from_inputs(scene.particles, device=dev)
    yy = torch.linspace(0, 1, H)[:, None]
    xx = torch.linspace(0, 1, W)[None, :]
    host_gt = torch.stack([0.5 + 0.3 * torch.sin(9 * xx + 4 * yy), 0.5 + 0.3 * torch.cos(7 * yy - 3 * xx),
                           0.4 + 0.2 * torch.sin(13 * xx * yy)]).contiguous().pin_memory()
    gt = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    img = torch.empty((3, H, W), dtype=torch.float32, device=dev)
    dL = torch.empty_like(img)
    grads = G.PlanarParams.zeros(P, deg, dev)
    loss = G.Loss(W, H, device=dev)
    mask = loss.mask(host_gt.to(dev), 0.75, stream=stream)
    opt = G.Adam(params)
    host_loss = torch.empty(4, dtype=torch.float32).pin_memory()

    def one(s=None):
        s = stream if s is None else s
        with torch.cuda.stream(s):
            gt.copy_(host_gt, non_blocking=True)
            G.ges_preprocess(params, cam, st, frame, s)
            G.ges_sort(frame, s)
            G.ges_render_fwd(frame, st, img, None, s)
            loss.mask(gt, 0.75, mask, stream=s)
            out, _ = loss(img, gt, mask, dL, stream=s)
            G.ges_render_bwd(params, cam, st, frame, dL, grads, False, s)
            opt.step(params, grads, stream=s)
            host_loss.copy_(out, non_blocking=True)

    for _ in range(2):
        one()
    torch.cuda.synchronize()

    def timed(fn):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        for _ in range(steps):
            fn()
        b.record(stream)
        b.synchronize()
        return a.elapsed_time(b) / steps

    ms_direct = timed(one)
    # the same iteration captured once as a CUDA graph (the copies are graph memcpy nodes
    # from / to the pinned host buffers, so every replay still moves them)
    ms_graph, launch = None, "direct launches"
    if world == 1:
        try:
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream()
            cap.wait_stream(stream)
            with torch.cuda.graph(g, stream=cap):
                one(cap)
            stream.wait_stream(cap)
            torch.cuda.synchronize()
            ms_graph = timed(g.replay)
            launch = "CUDA graph"
        except Exception as e:  # noqa: BLE001 -- reported; the direct number stands
            launch = f"direct launches (graph capture failed: {e})"
    ms = ms_graph if ms_graph is not None else ms_direct
    return {"value": world * W * H / (ms / 1e3) / 1e6, "unit": "Mpixel-frames/s (fwd+loss+bwd+Adam)",
            "ms_per_step": ms, "ms_per_step_direct_launches": ms_direct, "launch": launch,
            "h2d_bytes_per_step": host_gt.numel() * 4, "d2h_bytes_per_step": host_loss.numel() * 4,
            "final_loss": float(host_loss[0]), "pair_overflow": bool(frame.counts().overflow),
            "path": "parameters resident; ground truth pinned host -> device, S1-S4, ges_loss_mask + ges_loss, "
                    "S5, ges_adam_step, loss -> host"}


def cpu_baseline(scene, definitional_tiles=16):
    """The oracle as it stands on this host: one full binned config-3 frame (fwd+bwd,
    no extrapolation), plus SURVEY.md §8(d)'s definitional-mode sample (labelled as an
    extrapolation)."""
    info = oracle_frame(scene, 0)
    cam = scene.cameras[0]
    value = cam.width * cam.height / info["frame_s"] / 1e6
    host = host_info()
    out = {"value": value, "unit": "Mpixel-frames/s (fwd+bwd)", "cores": info["threads"], "nproc": host["nproc"],
           "cpu_model": host["cpu_model"], "kind": "oracle",
           "sample": (f"one full frame: all {scene.particles.P} particles, all {cam.width}x{cam.height} pixels, "
                      f"binned mode (R10 rect lists), S1-S5 fwd+bwd; no extrapolation"),
           "frame_s": info["frame_s"], "stages_s": info["stages_s"]}
    if definitional_tiles:
        out["definitional"] = oracle_definitional_sample(scene, 0, definitional_tiles)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="launch every kernel directly in the timed loop")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--order", choices=["morton", "input"], default="input",
                    help="particle storage order of our arm (DESIGN.md 'Particle order')")
    ap.add_argument("--definitional-tiles", type=int, default=16,
                    help="tiles of the oracle's definitional-mode sample in cpu_baseline (0: skip)")
    ap.add_argument("--config", type=int, choices=[0, 1, 2, 3, 4], default=3,
                    help="scene of the headline step (BASELINE.json's metric is quoted on config 3)")
    args = ap.parse_args()
    global ORDER, WORKLOAD_CFG
    ORDER = args.order
    WORKLOAD_CFG = args.config
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
