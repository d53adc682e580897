#!/usr/bin/env python
"""DOT on B200 -- benchmark (one JSON line on rank 0).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Headline (BASELINE.json configs[1], NeRF-synthetic-shaped training step):
depth-9 SH-3 scene from a 64-blob field (~2.6M leaves), rays from 100
hemisphere cameras (800x800, r=4.03, fov 40 deg), one step = gather a
2^20-ray batch per GPU -> fused forward+backward+signal kernel -> NCCL
all-reduce of leaf gradients (N>1) -> sparse RMSProp -> signal accumulate.
``value`` = rays/s over all ranks with inputs resident in HBM; ``e2e`` =
the same step through the public API from pinned host buffers (H2D of the
batch, D2H of the loss inside the timed region).

Side measurements in the same line: ``render`` (configs[2]: 800x800 views,
eps 1e-4), ``refine`` (configs[4]: 16M-leaf depth-10 tree, log-normal(-6,2)
signals, tau 0.01, gamma 0.1), ``roofline`` of the dominant kernel
(render_bwd) against the measured HBM copy bandwidth, and ``cpu_baseline``
(the C oracle port of the reference kernels on this host's cores).

``--impl reference`` times the reference's algorithm on the CPU (the C
oracle port, all host threads) on the same workload, rank 0 only.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = ("rays/sec render & fwd+bwd per GPU (1/2/4/8 B200), 800x800 FPS, refine ms, "
          "%HBM roofline")
BATCH = 1 << 20
E2E_BATCHES = 8  # distinct pinned host batches the e2e loop cycles through
N_VIEWS = 100
W = H = 800
RADIUS = 4.03
EPS = 1e-4
BG = 1.0
# algorithmic bytes: per ray f64 origin+dir+target; per
# composited segment sigma 4 B + SH row 12*B B read + gradient 4*(1+3B) B
# (one RMW) + signal 8 B.
B_SH = 16
RAY_BYTES = 72
SEG_BYTES = 4 + 12 * B_SH + 4 * (1 + 3 * B_SH) + 8


def measured_traffic(kernel):
    """DRAM bytes per launch of `kernel` from the committed ncu --set full
    capture (tools/summarise_profiles.py -> profiles/traffic.json)."""
    t = profile_entry(kernel)
    if t is None:
        return None, None, None
    return float(t["dram_bytes_per_launch"]), t["capture"], t.get("l2_hit_pct")


def profile_entry(kernel):
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            return json.load(fh)[kernel]
    except Exception:
        return None


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region.

    The recipe's query, started BEFORE the warm-up (nvidia-smi's own start-up
    is CPU-heavy and would otherwise delay the first timed launches) and
    stopped after; ``mark(t0, t1)`` gives the host wall-clock window of the
    timed region and only samples stamped inside it (widened to the nearest
    samples when the region is shorter than the sampling period) count."""

    # power.draw is left out: reading it stalls the driver for tens of ms,
    # long enough to starve the launch thread of a ~80 ms timed region
    FIELDS = ("timestamp,index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.window = None

    def start(self):
        if os.environ.get("DOT_BENCH_NO_CLOCKS"):
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            threading.Thread(target=self._read, daemon=True).start()
            # nvidia-smi's start-up (NVML init) takes ~1 s of CPU: wait for its
            # first sample so none of it overlaps the timed region
            t_end = time.time() + 5.0
            while not self.rows and time.time() < t_end and self.proc.poll() is None:
                time.sleep(0.02)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def mark(self, t0: float, t1: float) -> None:
        self.window = (t0, t1)

    @staticmethod
    def _stamp(text: str):
        import datetime
        try:
            return datetime.datetime.strptime(text, "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except Exception:
            return None

    def stop(self):
        time.sleep(0.1)  # let the samples bracketing the region arrive
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        rows = [(self._stamp(r[0]), r) for r in self.rows if len(r) >= 9]
        rows = [(t, r) for t, r in rows if t is not None]
        if self.window is not None and rows:
            a, b = self.window
            inside = [r for t, r in rows if a <= t <= b]
            if not inside:  # region shorter than the period: the samples around it
                before = [r for t, r in rows if t < a][-1:]
                after = [r for t, r in rows if t > b][:1]
                inside = before + after
            picked = inside
        else:
            picked = [r for _, r in rows]
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in picked:
            try:
                sm.append(float(r[2]))
                mx = max(mx, float(r[3]))
                for k, nm in enumerate(names):
                    if r[5 + k].lower().startswith("active"):
                        reasons.add(nm)
            except Exception:
                continue
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# workload

def view_rays_torch(focal, pose, device, W=W, H=H):
    import torch
    xs = (torch.arange(W, dtype=torch.float64, device=device) + 0.5 - 0.5 * W) / focal
    ys = -(torch.arange(H, dtype=torch.float64, device=device) + 0.5 - 0.5 * H) / focal
    cam = torch.empty(H, W, 3, dtype=torch.float64, device=device)
    cam[..., 0] = xs[None, :]
    cam[..., 1] = ys[:, None]
    cam[..., 2] = -1.0
    rot = torch.as_tensor(pose[:3, :3], dtype=torch.float64, device=device)
    world = cam.reshape(-1, 3) @ rot.T
    world = world / torch.linalg.norm(world, dim=1, keepdim=True)
    origins = torch.as_tensor(pose[:3, 3], dtype=torch.float64, device=device).expand_as(world).contiguous()
    return origins, world.contiguous()


def _spread10(v):
    v = v & 0x3FF
    v = (v | (v << 16)) & 0x030000FF
    v = (v | (v << 8)) & 0x0300F00F
    v = (v | (v << 4)) & 0x030C30C3
    v = (v | (v << 2)) & 0x09249249
    return v


def morton_key(idx, W=W, H=H):
    """(view, Morton(x, y)) key of pool indices (pool is view-major, row-major)."""
    view = idx // (W * H)
    pix = idx - view * (W * H)
    y = pix // W
    x = pix - y * W
    return (view << 32) | (_spread10(x) << 1) | _spread10(y)


def perturbed(tree, seed):
    import torch
    from paper_2307_15333_b200.octree import from_canonical_tensors
    topo = tree.topology()
    g = torch.Generator(device=tree.device)
    g.manual_seed(seed)
    sh = tree._sh_store.clone()
    sh[:, :3 * tree.basis_count] += 0.05 * torch.randn(sh.shape[0], 3 * tree.basis_count,
                                                       generator=g, device=tree.device)
    return from_canonical_tensors(tree.center, tree.half_extent, tree.basis_count, tree.max_depth,
                                  topo.node, tree._sigma, sh, topo.level_offsets)


class Workload:
    """A training-step workload: scene, camera rig, pool views, batch per rank."""

    def __init__(self, key, scene, cameras, w, h, views, batch, scaling, desc, l2):
        self.key, self.scene, self.cameras = key, scene, cameras
        self.W, self.H, self.views, self.batch = w, h, views, batch
        self.scaling, self.desc, self.l2 = scaling, desc, l2


def workloads():
    from paper_2307_15333_b200 import scenes
    return {
        "c2": Workload(
            "c2", lambda dev: scenes.config2_scene(device=dev),
            lambda: scenes.hemisphere_cameras(N_VIEWS, W, H, RADIUS, seed=3), W, H, N_VIEWS,
            lambda world: BATCH, "weak",
            "configs[1] training step: depth-9 SH-3 scene, 2^20-ray batch per GPU, "
            "fwd+bwd+signal, NCCL grad all-reduce (N>1), RMSProp",
            "inputs larger than L2 (2.6M-leaf payload 0.51 GB, 100-view ray pool 4.6 GB, "
            "random 2^20-ray batches)"),
        "c4": Workload(
            "c4", lambda dev: scenes.config4_scene(device=dev),
            lambda: scenes.ring_cameras(32, 1920, 1080, 3.0, seed=6), 1920, 1080, 32,
            lambda world: (1 << 21) // world, "strong",
            "configs[3] training step: depth-10 SH-3 scene over the 2x bbox (256 anisotropic "
            "blobs + ground slab), 1920x1080 ring cameras, 2^21-ray global batch sharded over "
            "the GPUs, fwd+bwd+signal, NCCL grad all-reduce (N>1), RMSProp",
            "inputs larger than L2 (8.5M-leaf payload 1.9 GB, 32-view ray pool 4.8 GB, "
            "random 2^21-ray global batches)"),
    }


def build_training_pool(tree, device, wl=None):
    """All rays of the workload's training views + targets rendered from a perturbed copy."""
    import torch
    from paper_2307_15333_b200.render import render_rays
    if wl is None:
        wl = workloads()["c2"]
    focal, poses = wl.cameras()
    os_, ds_ = zip(*(view_rays_torch(focal, p, device, wl.W, wl.H) for p in poses))
    origins, dirs = torch.cat(os_), torch.cat(ds_)
    del os_, ds_
    target_tree = perturbed(tree, 21)
    targets = torch.empty_like(origins)
    for lo in range(0, origins.shape[0], 1 << 22):
        targets[lo:lo + (1 << 22)] = render_rays(target_tree, origins[lo:lo + (1 << 22)],
                                                  dirs[lo:lo + (1 << 22)], BG).double()
    return origins, dirs, targets


def workload_config(wl, tree, world):
    """The line's ``config``: what defines the workload, identical on both
    arms (``--impl reference`` prints the same dict)."""
    return {"workload": wl.desc, "leaves": int(tree.leaf_count), "nodes": int(tree.topology().n_nodes),
            "global_batch": wl.batch(world) * world, "views": wl.views, "resolution": [wl.W, wl.H],
            "batch_draw": "uniform random rays of the resident training-view ray pool, a fresh "
                          "epoch permutation slice per step",
            "eps": EPS, "background": BG, "l2": wl.l2}


# ---------------------------------------------------------------------------
# our arm

def run_ours(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    from paper_2307_15333_b200 import scenes, _lib
    from paper_2307_15333_b200.optim import RmsPropState
    from paper_2307_15333_b200.signals import SignalBuffer

    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    _lib.check(_lib.load().dot_device_check(), "device check")
    t_setup = time.time()
    wl = workloads()[args.workload]
    tree = wl.scene(dev)
    origins, dirs, targets = build_training_pool(tree, dev, wl)
    n_pool = origins.shape[0]
    per_rank = wl.batch(world)
    n_global = per_rank * world
    gs = 2.0 / n_global
    state = RmsPropState(tree)
    buf = SignalBuffer(tree)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    total_steps = args.warmup + args.steps
    # epoch-style permutations of the ray pool, one slice per step (a new
    # permutation whenever the steps outrun the pool: train_epoch's order)
    need = (total_steps + 2) * per_rank
    perm = torch.cat([torch.randperm(n_pool, generator=gen, device=dev)
                      for _ in range((need + n_pool - 1) // n_pool)])[:need]
    perm = perm.reshape(total_steps + 2, per_rank)
    kev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(total_steps)]

    def batch_index(k):
        """Loader: the step's random rays, optionally reordered for coherence
        (same ray set; loss and gradients are sums over rays)."""
        idx = perm[k]
        if args.order == "raster":
            idx = idx.sort().values
        elif args.order == "morton":
            idx = idx[torch.argsort(morton_key(idx, wl.W, wl.H))]
        return idx

    from paper_2307_15333_b200.optim import StepWorkspace, train_step
    from paper_2307_15333_b200.parallel import allreduce_grads_overlapped, chunk_bounds
    sws = StepWorkspace(tree, buf)
    ws = sws.ws

    def exchange(update):
        """NCCL all-reduce of the leaf gradients in row chunks, each chunk's
        RMSProp update issued as soon as its reduction lands (N = 1: one update)."""
        allreduce_grads_overlapped(ws.dsigma, ws.dsh_store, ws.touched, update,
                                   chunks=args.ar_chunks)

    if world > 1 and args.exchange == "peer":
        # reduce-scatter + RMSProp + all-gather fused over symmetric (peer) memory
        from paper_2307_15333_b200.parallel import PeerExchange
        exchange = PeerExchange(tree, state, sws)

    from paper_2307_15333_b200.render import plan_batch, pool_keys, pool_rank, ray_costs
    plan_stream = torch.cuda.Stream(dev)
    plans = {}
    # the resident pool ranked once by its 62-bit coherence keys and stored
    # in that order (like building the pool itself): each step's plan is a
    # counting sort of the batch's positions over a pool-sized bitmap
    # (dot_plan_ranked) -- no per-step key gather, radix sort or index
    # gather.  The steps' batches stay epoch-permutation slices of the pool.
    # DOT_BENCH_PLAN=rank-gather: pool left in place, plans map positions
    # back through the rank's order; =keys: 31-bit pool keys + radix sort.
    plan_kind = os.environ.get("DOT_BENCH_PLAN", "rank")
    pkeys = pool_keys(tree, origins, dirs) if plan_kind == "keys" else None
    prank = pool_rank(tree, origins, dirs) if plan_kind in ("rank", "rank-gather") else None
    # and its per-ray schedule costs (the first epoch's prediction; every
    # backward refreshes its rays' entries): warps launch longest first
    pcosts = ray_costs(tree, origins, dirs, EPS) if os.environ.get("DOT_BENCH_COSTS", "1") == "1" else None
    # the plans' outputs in a ring (no allocation on the plan's path; at most
    # LEAD = 2 steps are in flight, so a buffer is free again 4 plans later)
    plan_ring = [(torch.empty(per_rank, dtype=torch.int64, device=dev),
                  torch.empty((per_rank + 31) // 32, dtype=torch.int32, device=dev)) for _ in range(4)]
    if plan_kind == "rank":
        from paper_2307_15333_b200.render import PoolRank
        origins, dirs, targets, pcosts = prank.permute(origins, dirs, targets, pcosts)
        prank = PoolRank.identity(n_pool, dev)
        torch.cuda.empty_cache()

    def step(k, timed_kernel=True):
        # the batch is read in place from the resident pool (ray_index): no
        # gather; its plan (key order regrouped by cost + warp launch order)
        # ran beside the previous step's update, and the next one is queued
        # behind this step's backward
        idx = batch_index(k)
        plan = plans.pop(k, None)

        def next_plan():
            if k + 1 < total_steps + 2:
                plans[k + 1] = plan_batch(tree, origins, dirs, batch_index(k + 1), stream=plan_stream,
                                          keys=pkeys, rank=prank, costs=pcosts,
                                          out=plan_ring[(k + 1) % len(plan_ring)] if prank is not None else None)
        # the next plan is queued behind this step's backward, so it runs
        # beside the (bandwidth-bound) update instead of the backward;
        # DOT_PLAN_EARLY=1: queued before the step (runs beside the backward)
        early = os.environ.get("DOT_PLAN_EARLY", "0") == "1"
        if pre_planned:  # diagnostic: every plan made before the loop (the plan's cost on the step)
            return train_step(tree, origins, dirs, targets, state, buf, sws, BG, EPS, ray_index=idx,
                              grad_scale=gs, exchange=exchange if world > 1 else None,
                              kernel_events=kev[k] if timed_kernel else None, plan=plan)
        if early:
            next_plan()
        return train_step(tree, origins, dirs, targets, state, buf, sws, BG, EPS,
                          ray_index=idx, grad_scale=gs,
                          exchange=exchange if world > 1 else None,
                          kernel_events=kev[k] if timed_kernel else None, plan=plan,
                          after_backward=None if early else next_plan)

    # DOT_PLAN_PRE=1 (diagnostic, never a bench line): all plans made up
    # front with their own outputs, none inside the steps
    pre_planned = os.environ.get("DOT_PLAN_PRE", "0") == "1"
    if pre_planned:
        for k in range(total_steps):
            plans[k] = plan_batch(tree, origins, dirs, batch_index(k), keys=pkeys, rank=prank, costs=pcosts)
        torch.cuda.synchronize()
    clocks = ClockSampler(local_rank).start()  # before the warm-up: its start-up is CPU-heavy
    # at most LEAD steps in flight: the host waits for step k - LEAD before
    # queuing step k, so the caching allocator recycles the plans' buffers
    # instead of growing (cudaMalloc on the launch thread starved the GPU)
    LEAD = 2
    done = {}

    def paced(k):
        if k - LEAD in done:
            done.pop(k - LEAD).synchronize()
        out = step(k)
        ev = torch.cuda.Event()
        ev.record()
        done[k] = ev
        return out

    for k in range(args.warmup):
        paced(k)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    setup_s = time.time() - t_setup
    t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    # ncu --profile-from-start off captures exactly the timed steps
    profile_range = bool(os.environ.get("DOT_PROFILE_RANGE"))
    if profile_range:
        torch.cuda.profiler.start()
    gc.collect()
    gc.disable()  # no collector pause between the launches of the timed steps
    trace = os.environ.get("DOT_TRACE")  # diagnostic (tools/step_gaps.py): never set for a bench line
    if trace:
        prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
        prof.__enter__()
    h0 = time.time()
    t0.record()
    for k in range(args.warmup, total_steps):
        paced(k)
    t1.record()
    torch.cuda.synchronize()
    if trace:
        prof.__exit__(None, None, None)
        prof.export_chrome_trace(trace)
    clocks.mark(h0, time.time())
    gc.enable()
    if profile_range:
        torch.cuda.profiler.stop()
    clk = clocks.stop()
    ms = t0.elapsed_time(t1)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    ms_step = ms / args.steps
    value = n_global * args.steps / (ms / 1e3)
    kern_ms = [kev[k][0].elapsed_time(kev[k][1]) for k in range(args.warmup, total_steps)]
    kern_ms_avg = sum(kern_ms) / len(kern_ms)

    # workload statistics of one batch (outside the timed region)
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    idx = perm[total_steps]
    view, _ = tree.tree_view()
    oo, dd = origins[idx].contiguous(), dirs[idx].contiguous()
    _lib.call("dot_ray_stats", _lib.ctypes.byref(view), _lib.ptr(oo), _lib.ptr(dd), per_rank, EPS,
              _lib.ptr(stats), _lib.stream_ptr())
    seg, comp, qpos = [int(x) for x in stats.cpu()]
    alg_bytes = per_rank * RAY_BYTES + comp * SEG_BYTES
    hbm, peak_kind = peaks()
    achieved = alg_bytes / (kern_ms_avg / 1e3) / 1e9
    # the committed ncu capture is of the configs[1] step
    traffic, traffic_src, l2_hit = measured_traffic("render_bwd_buffered") if wl.key == "c2" else (None, None, None)
    # REDs per launch: dsigma for every composited segment, 12 x F32x4 SH rows
    # and one f64 signal add for every segment with q > 0
    reds = comp + 13 * qpos

    # e2e: public API from pinned host buffers (H2D batch + D2H loss per step).
    # Headline: RayBatchStager overlaps step k+1's H2D copy (side copy stream)
    # with step k's compute and LossReader reads each step's loss one step
    # late; every step still copies its own 72 B/ray and reads its loss.
    # "serial_ms_per_step": the same loop with blocking copies + reads.
    from paper_2307_15333_b200.staging import LossReader, RayBatchStager
    host = []
    e2e_ranked = plan_kind == "rank"
    for j in range(E2E_BATCHES):  # distinct pinned host batches (rays + targets + costs [+ ids]), cycled
        idx = perm[j % perm.shape[0]]
        host.append(tuple(x[idx].cpu().pin_memory() if x is not None else None
                          for x in (origins, dirs, targets, pcosts))
                    + ((idx.cpu().pin_memory(),) if e2e_ranked else ()))
    torch.cuda.synchronize()
    e2e_bytes_per_ray = 72 + (2 if pcosts is not None else 0) + (8 if e2e_ranked else 0)

    ex = exchange if world > 1 else None

    def serial_loop(steps):
        for k in range(steps):
            o_h, d_h, t_h = host[k % len(host)][:3]
            loss = train_step(tree, o_h, d_h, t_h, state, buf, sws, BG, EPS, grad_scale=gs,
                              exchange=ex)
            float(loss.item())

    # the host dataset is the key-ordered pool: a batch's ids (its rows) are
    # its key positions, so the staged batch is ordered without a sort
    # (dot_plan_ranked, slot mode); DOT_BENCH_PLAN=keys: ray keys + radix sort
    stager = RayBatchStager(dev, max_rays=per_rank, plan_tree=tree,
                            plan_rank=PoolRank.identity(n_pool, dev) if e2e_ranked else None)

    hostprof = os.environ.get("DOT_E2E_HOSTPROF") == "1"  # diagnostic: host seconds per loop phase

    def staged_loop(steps):
        reader = LossReader()
        stager.stage(*host[0])
        hp = [0.0] * 6
        worst = [0.0] * 6
        call_worst = {}
        if hostprof:  # the worst host time of each C-ABI call made inside plan_next
            from paper_2307_15333_b200 import _lib as lib_mod
            real_call = lib_mod.call

            def timed_call(name, *a):
                c = time.perf_counter()
                r = real_call(name, *a)
                call_worst[name] = max(call_worst.get(name, 0.0), time.perf_counter() - c)
                return r
            lib_mod.call = timed_call

        import cProfile
        cprof = cProfile.Profile() if os.environ.get("DOT_E2E_CPROFILE") == "1" else None

        def plan_next_timed():
            c = time.perf_counter()
            if cprof:
                cprof.enable()
            stager.plan_next()
            if cprof:
                cprof.disable()
            hp[5] += time.perf_counter() - c
            worst[5] = max(worst[5], time.perf_counter() - c)
        for k in range(steps):
            c0 = time.perf_counter()
            o_d, d_d, t_d, plan = stager.take_with_plan()
            c1 = time.perf_counter()
            if k + 1 < steps:
                stager.stage(*host[(k + 1) % len(host)])
            c2 = time.perf_counter()
            loss = train_step(tree, o_d, d_d, t_d, state, buf, sws, BG, EPS, grad_scale=gs,
                              exchange=ex, plan=plan,
                              after_backward=plan_next_timed if hostprof else stager.plan_next)
            c3 = time.perf_counter()
            stager.release()
            reader.push(loss)
            c4 = time.perf_counter()
            for j, dt in enumerate((c1 - c0, c2 - c1, c3 - c2, c4 - c3, c4 - c0)):
                hp[j] += dt
                worst[j] = max(worst[j], dt)
        reader.flush()
        if hostprof and steps > 5:
            print("e2e host ms/step: take %.3f stage %.3f train_step %.3f release+push(wait) %.3f total %.3f "
                  "(plan_next inside train_step %.3f)" % tuple(1e3 * x / steps for x in hp), file=sys.stderr)
            print("e2e host worst ms: take %.3f stage %.3f train_step %.3f release+push(wait) %.3f total %.3f "
                  "plan_next %.3f" % tuple(1e3 * x for x in worst), file=sys.stderr)
            print("e2e host worst ms per C-ABI call: " + ", ".join(
                f"{k} {1e3 * v:.3f}" for k, v in sorted(call_worst.items(), key=lambda x: -x[1])), file=sys.stderr)
            lib_mod.call = real_call
            if cprof:
                import pstats
                pstats.Stats(cprof, stream=sys.stderr).sort_stats("tottime").print_stats(12)
        return reader.values

    def timed(loop):
        loop(args.warmup)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        gc.collect()
        gc.disable()
        e0.record()
        loop(args.steps)
        e1.record()
        torch.cuda.synchronize()
        gc.enable()
        t = e0.elapsed_time(e1)
        if world > 1:
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    e2e_serial_ms = timed(serial_loop)
    trace_e2e = os.environ.get("DOT_TRACE_E2E")  # diagnostic (tools/step_gaps.py --e2e): never set for a bench line
    if trace_e2e:
        prof = torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA])
        prof.__enter__()
    e2e_ms = timed(staged_loop)
    if trace_e2e:
        prof.__exit__(None, None, None)
        prof.export_chrome_trace(trace_e2e)
    e2e_value = n_global * args.steps / (e2e_ms / 1e3)

    # the optimizer update alone on one batch's gradients (consume=False so
    # every repetition sees them): the reference's f64 state (the timed step
    # above) and the opt-in f32 state
    from paper_2307_15333_b200.optim import rmsprop_step
    from paper_2307_15333_b200.render import BackpropWorkspace, render_and_backprop
    rws = BackpropWorkspace.for_tree(tree)
    _, rg, _ = render_and_backprop(tree, origins, dirs, targets, BG, EPS, ray_index=perm[total_steps],
                                   grad_scale=gs, workspace=rws)
    rms = {}
    saved = (tree._sigma.clone(), tree._sh_store.clone())  # the timed updates move the payload
    for name, dt in (("f64_state_ms", torch.float64), ("f32_state_ms", torch.float32)):
        st = RmsPropState(tree, state_dtype=dt)
        for _ in range(3):
            rmsprop_step(tree, rg, st)
        torch.cuda.synchronize()
        r0, r1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        r0.record()
        for _ in range(10):
            rmsprop_step(tree, rg, st)
        r1.record()
        torch.cuda.synchronize()
        rms[name] = r0.elapsed_time(r1) / 10
    tree._sigma.copy_(saved[0])
    tree._sh_store.copy_(saved[1])
    del saved
    rms["touched_rows"] = int(rws.touched.sum())
    rms["note"] = ("rmsprop_step alone on one batch's gradients; f64 = the reference's state dtype (bit-exact, "
                   "the headline step), f32 = opt-in RmsPropState(state_dtype=torch.float32)")
    del rws, rg

    # signal-only forward (dot_signal_fwd) on a training batch: the
    # calibration-only pass, same rays, no gradients
    from paper_2307_15333_b200.render import signal_pass
    sig_out = torch.zeros(tree.capacity, dtype=torch.float64, device=dev)
    sidx = perm[total_steps + 1]
    sig_mode = os.environ.get("DOT_BENCH_SIGNAL_PLAN", "rank")  # rank (+ cost regroup) | keys

    def sig_call():
        # the batch's plan is part of the timed call: the ranked pool's order
        # regrouped by the cost column (lane efficiency), or the ray keys
        p = plan_batch(tree, origins, dirs, sidx, rank=prank, costs=pcosts) \
            if sig_mode == "rank" and prank is not None else None
        signal_pass(tree, origins, dirs, EPS, ray_index=sidx, signal=sig_out, plan=p)
    for _ in range(3):
        sig_call()
    torch.cuda.synchronize()
    s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(5):
        sig_call()
    s1.record()
    torch.cuda.synchronize()
    sig_ms = s0.elapsed_time(s1) / 5
    signal_fwd = {"rays_per_s": per_rank / (sig_ms / 1e3), "ms_per_batch": sig_ms, "rays": per_rank,
                  "api": "render.signal_pass (+ its batch plan: "
                         + ("plan_batch(rank=, costs=), key order regrouped by cost" if sig_mode == "rank"
                            and prank is not None else "ray keys + radix sort")
                         + ") -> dot_signal_fwd: sum Q per leaf, no gradients"}

    # render (configs[2]) and refine (configs[4]) side measurements
    side = wl.key == "c2"  # render/refine/CPU legs belong to the default (configs[1]) line
    render = None if (args.skip_render or not side) else bench_render(tree, dev, args, world)
    del origins, dirs, targets, perm
    torch.cuda.empty_cache()
    refine = None if (args.skip_refine or rank != 0 or not side) else bench_refine(dev, args)
    cpu = None
    refine_c2 = None
    if rank == 0 and not args.skip_cpu and side:
        cpu = cpu_baseline(tree, args)
        if not args.skip_refine:
            refine_c2 = refine_vs_cpu(tree, dev)

    if rank != 0:
        return None
    return {
        "metric": METRIC,
        "value": value,
        "unit": "rays/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": wl.scaling,
        "vs_baseline": None,
        "dtype": "mixed f64/f32",
        "dtype_detail": "f64 traversal, transmittance, colour accumulation, loss and per-leaf signal; "
                        "f32 SH dot products, sigmoid and leaf gradients (north star: fp32 tolerance "
                        "1e-4 abs / 1e-3 rel)",
        "data": "synthetic (seeded blob-field scene, random-init SH, targets from a perturbed copy)",
        "config": workload_config(wl, tree, world),
        "run": {
            "segments_per_ray": seg / per_rank, "composited_per_ray": comp / per_rank,
            "parallelism": f"rays sharded dp{world}, tree replicated",
            "exchange": args.exchange if world > 1 else "none",
            "batch_order": args.order,
            "plan": ("step k+1's plan (coherence order, cost regrouping in 128-ray windows, warp launch "
                     "order) queued behind step k's backward on a side stream, running beside its update: "
                     + ({"rank": "a counting sort of the batch's pool positions, the pool stored in 62-bit "
                                 "key order (render.pool_rank + PoolRank.permute, dot_plan_ranked)",
                         "rank-gather": "a counting sort over the resident pool's 62-bit key rank "
                                        "(render.pool_rank, dot_plan_ranked)",
                         "keys": "the resident pool's 31-bit ray keys (render.pool_keys) gathered and "
                                 "radix sorted"}[plan_kind])
                     + "; per-ray schedule costs (render.ray_costs; refreshed by every backward); the "
                       "rank / keys and costs computed once at setup; warps launched longest first by cost"),
        },
        # per step: the plan (rank: one cooperative plan_coop_kernel incl.
        # the warp order; keys: gather + radix sort histogram + exclusive sum
        # + 4 onesweep passes, then the cost order's warp cost + histogram +
        # scan + place), the backward and one rmsprop per all-reduce chunk (a
        # single update at N = 1)
        "gpu_launches": ((1 if plan_kind.startswith("rank") else 7 + 4) + 1
                         + (1 if world == 1 else len(chunk_bounds(tree.capacity, args.ar_chunks)))) * args.steps,
        "roofline": {
            "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "traffic_source": traffic_src,
            "l2_hit_pct": l2_hit,
            "kernel": "render_bwd_buffered_kernel<16, CoopSink> (K = 128 records)",
            "kernel_ms": kern_ms_avg, "alg_bytes_per_launch": alg_bytes, "peak_kind": peak_kind,
            "bytes_model": f"{RAY_BYTES} B/ray + {SEG_BYTES} B/composited segment",
            "atomics_per_launch": reds, "atomics_per_s": reds / (kern_ms_avg / 1e3),
        },
        "e2e": {"value": e2e_value, "unit": "rays/s", "h2d_bytes_per_step": per_rank * e2e_bytes_per_ray,
                "d2h_bytes_per_step": 8, "ms_per_step": e2e_ms / args.steps,
                "api": ("RayBatchStager (H2D of step k+1's rays, targets, costs"
                        + (" and dataset ids; its coherence order by the dataset's rank, dot_plan_ranked slot mode"
                           if e2e_ranked else "; its ray keys + radix sort")
                        + ", overlapping step k) + optim.train_step (render_and_backprop + rmsprop_step) + "
                          "LossReader (loss read one step late)"),
                "host_batches": E2E_BATCHES,
                "serial_ms_per_step": e2e_serial_ms / args.steps},
        "clocks": clk,
        "signal_fwd": signal_fwd,
        "rmsprop": rms,
        "render": render,
        "refine": refine,
        "refine_vs_cpu": refine_c2,
        "cpu_baseline": cpu,
        "setup_s": setup_s,
    }


def bench_render(tree, dev, args, world):
    import torch
    import torch.distributed as dist
    from paper_2307_15333_b200 import scenes
    from paper_2307_15333_b200.render import render_rays
    focal, poses = scenes.hemisphere_cameras(200, W, H, RADIUS, seed=4)
    n_views = max(4, min(2 * args.steps, 20))
    rank = dist.get_rank() if world > 1 else 0
    views = [view_rays_torch(focal, poses[(rank * n_views + i) % 200], dev) for i in range(n_views)]
    for i in range(min(3, n_views)):
        render_rays(tree, *views[i], BG, EPS)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for o, d in views:
        render_rays(tree, o, d, BG, EPS)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if world > 1:
        tt = torch.tensor([ms], device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
    rays_resident = W * H * n_views * world
    ms_resident = ms
    # configs[2]: all 200 views, sharded over the ranks, rays generated
    # in-kernel (8x4 warp tiles), one launch per rank (render_views); one
    # launch per view beside it
    from paper_2307_15333_b200.render import render_view, render_views
    from paper_2307_15333_b200.scene_io import Camera
    mine = [i for i in range(200) if i % world == rank]
    n_views = len(mine)
    cams = [Camera(W, H, focal, poses[i]) for i in mine]
    rays = W * H * 200

    def timed(fn, warm=3):
        for _ in range(warm):
            fn()
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        t = a.elapsed_time(b)
        if world > 1:
            tt = torch.tensor([t], device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            t = float(tt.item())
        return t

    ms_cam = timed(lambda: render_views(tree, cams, BG, EPS))
    ms_per_view_launch = timed(lambda: [render_view(tree, c, BG, EPS) for c in cams[:20]]) * n_views / min(20, n_views)
    # roofline of render_camera_kernel: per view 12 B/pixel rgb out (rays are
    # generated in-kernel: 0 B in) + per composited segment sigma 4 B + the
    # 192 B SH row when q > 0; counts from dot_ray_stats
    from paper_2307_15333_b200 import _lib
    stats = torch.zeros(3, dtype=torch.int64, device=dev)
    tv, _ = tree.tree_view()
    for o, d in views:
        _lib.call("dot_ray_stats", _lib.ctypes.byref(tv), _lib.ptr(o), _lib.ptr(d), o.shape[0], EPS,
                  _lib.ptr(stats), _lib.stream_ptr())
    seg, comp, qpos = [int(x) for x in stats.cpu()]
    n_res = len(views)  # per-ray segment counts sampled on the resident views
    alg_view = W * H * 12 + (comp * 4 + qpos * 12 * B_SH) / n_res
    hbm, peak_kind = peaks()
    achieved = alg_view / (ms_cam / n_views / 1e3) / 1e9
    prof = profile_entry("render_camera_kernel") or {}
    traffic, traffic_src, l2_hit = measured_traffic("render_camera_kernel")
    if traffic is not None:
        traffic /= 200.0  # the capture is the timed 200-view launch: DRAM bytes per view
    # HBM roofline of the kernel from its MEASURED DRAM bytes (ncu) over the
    # live per-view time; the algorithmic gather model is reported beside it
    # (coherent camera rays hit L1/L2, so it overstates DRAM traffic)
    dram_gbs = traffic / (ms_cam / n_views / 1e3) / 1e9 if traffic is not None else None
    return {"rays_per_s": rays / (ms_cam / 1e3), "fps_800x800": 200 / (ms_cam / 1e3),
            "roofline": {"bound": "hbm", "achieved": dram_gbs, "peak": hbm, "unit": "GB/s",
                         "frac": dram_gbs / hbm if dram_gbs is not None else None, "peak_kind": peak_kind,
                         "traffic": traffic, "traffic_source": traffic_src, "l2_hit_pct": l2_hit,
                         "achieved_note": "ncu DRAM bytes per view (200-view launch / 200) / live ms per view",
                         "kernel": "render_camera_kernel<16>",
                         "algorithmic": {"bytes_per_view": alg_view, "gbs": achieved, "frac_of_hbm": achieved / hbm,
                                         "model": "12 B/pixel + 4 B/composited segment + 192 B/segment with q>0"},
                         "composited_per_ray": comp / (W * H * n_res),
                         "segments_per_ray": seg / (W * H * n_res)},
            # the kernel is issue / latency bound, not HBM bound: its pipe
            # utilisations from the same ncu capture
            "l2_gather": {"gbs": (prof["l2_bytes_per_launch"] / 200.0) / (ms_cam / n_views / 1e3) / 1e9
                          if prof.get("l2_bytes_per_launch") else None,
                          "note": "ncu lts__t_bytes per view / live ms per view (L2 traffic the gathers "
                                  "generate; DRAM is the roofline above)"},
            "issue_roofline": {"bound": "issue", "issue_active_pct": prof.get("issue_active_pct"),
                               "fp64_pipe_pct": prof.get("fp64_pipe_pct"), "xu_pipe_pct": prof.get("xu_pipe_pct"),
                               "lsu_pipe_pct": prof.get("lsu_pipe_pct"),
                               "warps_active_pct": prof.get("warps_active_pct"), "source": traffic_src},
            "ms_per_view": ms_cam / n_views, "views": 200, "eps": EPS,
            "workload": "configs[2]: 800x800 random hemisphere views, render_views (in-kernel rays, "
                        "all views of a rank in one launch)",
            "one_launch_per_view": {"rays_per_s": rays / (ms_per_view_launch / 1e3),
                                    "ms_per_view": ms_per_view_launch / n_views},
            "rays_resident": {"rays_per_s": rays_resident / (ms_resident / 1e3),
                              "ms_per_view": ms_resident / n_res, "views": n_res * world,
                              "workload": "views through render_rays, f64 rays resident in HBM, "
                                          "one launch per view"}}


CONFIG5_SPLIT_THR = 750.0  # seed-5 field at depth 10: ~16M leaves (820 -> 11.2M, 600 -> 39M)


def config5_tree(dev):
    from paper_2307_15333_b200 import scenes
    field = scenes.BlobField.make(seed=5, n_blobs=64)
    tree = scenes.adaptive_tree(field, max_depth=10, basis_count=16, split_thr=CONFIG5_SPLIT_THR,
                                empty_thr=0.05, min_depth=4, sh_seed=50, device=dev)
    tree.max_depth = 11  # depth-10 leaves stay eligible for sampling
    return tree


def bench_refine(dev, args):
    import torch
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.octree import from_canonical_tensors
    from paper_2307_15333_b200.signals import SignalBuffer
    base = config5_tree(dev)
    topo = base.topology()
    node0, sig0, sh0 = topo.node, base._sigma, base._sh_store
    leaf = node0 < 0
    g = torch.Generator(device=dev)
    g.manual_seed(55)
    acc = torch.zeros(node0.shape[0], dtype=torch.float64, device=dev)
    acc[leaf] = torch.exp(-6.0 + 2.0 * torch.randn(int(leaf.sum()), generator=g, device=dev,
                                                  dtype=torch.float64))
    times, rep = [], None
    passes = 3
    ev_ms = None
    for k in range(passes + 2):
        tree = from_canonical_tensors(base.center, base.half_extent, 16, 11, node0.clone(),
                                      sig0.clone(), sh0.clone(), topo.level_offsets)
        buf = SignalBuffer(tree)
        buf.accumulator.copy_(acc)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        prof = k == passes and bool(os.environ.get("DOT_PROFILE_REFINE"))
        if prof:
            torch.cuda.profiler.start()
        # the drop-in default call: calibrate() with its (lazy) event report
        h0 = time.perf_counter()
        a.record()
        rep = calibrate(tree, buf, CalibrationConfig(tau=0.01, gamma=0.10))
        b.record()
        torch.cuda.synchronize()
        h1 = time.perf_counter()
        if prof:
            torch.cuda.profiler.stop()
        if 0 < k <= passes:
            times.append(a.elapsed_time(b))
            host_ms = (h1 - h0) * 1e3
        if k == passes + 1:  # materialising the reference-style event list, once
            e0 = time.perf_counter()
            n_events = len(rep.events)
            ev_ms = (time.perf_counter() - e0) * 1e3
        n_new = tree.topology().n_nodes
        del tree, buf
    ms = sum(times) / len(times)
    n_old = int(node0.shape[0])
    row = 4 + 4 * 48
    alg = (n_old * (4 + 8) + rep.merges_applied * 9 * row + rep.splits_applied * 9 * row
           + n_new * (4 + row + 9))
    hbm, peak_kind = peaks()
    pe = profile_entry("refine_pass")
    dram = float(pe["dram_bytes_per_launch"]) if pe else None
    achieved = dram / (ms / 1e3) / 1e9 if dram else None
    return {"ms_per_pass": ms, "leaves_before": rep.leaves_before, "leaves_after": rep.leaves_after,
            "merges": rep.merges_applied, "splits": rep.splits_applied, "nodes_before": n_old,
            "nodes_after": int(n_new), "alg_gbs": alg / (ms / 1e3) / 1e9,
            "call": "calibrate(tree, buffer, CalibrationConfig(tau=0.01, gamma=0.1)) -- the default "
                    "call, report.events lazy",
            "host_ms_per_call": host_ms,
            "events_materialise_ms": ev_ms, "events": n_events,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm if achieved else None, "peak_kind": peak_kind,
                         "traffic": dram, "traffic_source": pe["capture"] if pe else None,
                         "achieved_note": "ncu DRAM bytes of every launch of one pass / live ms per pass"},
            "workload": "configs[4]: depth-10 SH-3 tree, log-normal(-6,2) signals, tau 0.01, "
                        "gamma 0.1, prune+sample+canonical compaction"}


def cpu_baseline(tree, args, n_rays=1 << 20):
    """The C oracle port of the reference kernels on this host's cores, on a
    bounded sample of the same training workload (uniform random rays of the
    100-view pool, like the timed batches): all threads on 2^20 rays, and
    one thread on 2^16 rays."""
    from oracle import oracle as O
    from paper_2307_15333_b200 import scenes
    O.build()
    focal, poses = scenes.hemisphere_cameras(N_VIEWS, W, H, RADIUS, seed=3)
    rng = np.random.default_rng(9)
    o, d = pool_rays_np(focal, poses, W, H, rng.integers(0, N_VIEWS * W * H, n_rays))
    tg = rng.uniform(0.0, 1.0, o.shape)
    tree._host()  # pool arrays for the oracle (outside the timing)
    O.render_and_backprop(tree, o[:256], d[:256], tg[:256], BG, EPS)
    t = time.perf_counter()
    O.render_and_backprop(tree, o, d, tg, BG, EPS)
    dt = time.perf_counter() - t
    cores = O.num_threads()
    m = 1 << 16
    O.set_threads(1)
    t1 = time.perf_counter()
    O.render_and_backprop(tree, o[:m], d[:m], tg[:m], BG, EPS)
    dt1 = time.perf_counter() - t1
    O.set_threads(cores)
    # render (configs[2]'s op): render_rays = count + fill + composite on 2^18 rays of one view
    fo, fd = pool_rays_np(focal, poses, W, H, np.arange(1 << 18) + 3 * W * H)
    t = time.perf_counter()
    O.render_rays(tree, fo, fd, BG, EPS)
    dt_r = time.perf_counter() - t
    return {"value": o.shape[0] / dt, "unit": "rays/s", "cores": cores, "kind": "port",
            "sample": f"{o.shape[0]} uniform random rays of the 100-view pool, fwd+bwd through "
                      "oracle/dot_oracle.c (count+fill+grad+serial scatter, OpenMP)",
            "seconds": dt,
            "one_thread": {"value": m / dt1, "unit": "rays/s", "cores": 1,
                           "sample": f"{m} of the same rays, one OpenMP thread"},
            "render": {"value": (1 << 18) / dt_r, "unit": "rays/s", "cores": cores,
                       "sample": "262144 rays of one 800x800 training view, render_rays (count + fill + "
                                 "composite)"}}


def refine_vs_cpu(tree, dev):
    """One DOT refine pass on the configs[1] scene (2.6M leaves, log-normal(-6, 2)
    signals, tau 0.01, gamma 0.1): our calibrate() vs the reference's algorithm
    on the host (oracle.calibrate -- the faithful restatement, LIFO splits one
    by one like octree.split_leaf_many), same tree and signals."""
    import torch
    from oracle import oracle as O
    from paper_2307_15333_b200.calibrate import CalibrationConfig, calibrate
    from paper_2307_15333_b200.octree import from_canonical_tensors
    from paper_2307_15333_b200.signals import SignalBuffer
    topo = tree.topology()
    node = topo.node
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    acc = torch.zeros(node.shape[0], dtype=torch.float64, device=dev)
    leaf = node < 0
    acc[leaf] = torch.exp(-6.0 + 2.0 * torch.randn(int(leaf.sum()), generator=g, device=dev, dtype=torch.float64))
    times = []
    for k in range(4):
        t2 = from_canonical_tensors(tree.center, tree.half_extent, tree.basis_count, tree.max_depth, node.clone(),
                                    tree._sigma.clone(), tree._sh_store.clone(), topo.level_offsets)
        buf = SignalBuffer(t2)
        buf.accumulator.copy_(acc)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        rep = calibrate(t2, buf, CalibrationConfig(tau=0.01, gamma=0.10))
        b.record()
        torch.cuda.synchronize()
        if k:
            times.append(a.elapsed_time(b))
        del t2, buf
    pool = O.PoolTree.from_canonical_words(tree.center, tree.half_extent, tree.basis_count, tree.max_depth,
                                          node.cpu().numpy(), tree.sigma.cpu().numpy(), tree.sh.cpu().numpy())
    acc_h = acc.cpu().numpy()
    t = time.perf_counter()
    ref = O.calibrate(pool, acc_h, 0.01, 0.10)
    cpu_s = time.perf_counter() - t
    same = (ref.merges_applied, ref.splits_applied) == (rep.merges_applied, rep.splits_applied)
    ms = sum(times) / len(times)
    return {"ms_per_pass": ms, "leaves_before": rep.leaves_before, "merges": rep.merges_applied,
            "splits": rep.splits_applied, "same_counts_as_cpu": same,
            "cpu_baseline": {"ms_per_pass": cpu_s * 1e3, "kind": "port", "cores": 1,
                             "sample": "the same pass through oracle.calibrate (numpy + the reference's "
                                       "one-by-one LIFO split loop; single-threaded like the reference)"},
            "workload": "configs[1] scene (2.6M leaves), log-normal(-6,2) signals, tau 0.01, gamma 0.1"}


# ---------------------------------------------------------------------------
# reference arm

def pool_rays_np(focal, poses, W, H, flat):
    """Rays of pool entries ``flat`` (view-major, row-major pixels) of a
    pinhole camera rig -- the same pixel convention as scene_io.Camera.rays
    (scene_io.py:77-91), for a random subset of the pool."""
    view = flat // (W * H)
    pix = flat - view * (W * H)
    y = pix // W
    x = pix - y * W
    cam = np.stack([(x + 0.5 - 0.5 * W) / focal, -(y + 0.5 - 0.5 * H) / focal, -np.ones(flat.size)], axis=1)
    P = np.asarray(poses, dtype=np.float64)[view]
    world = np.einsum("nj,nij->ni", cam, P[:, :3, :3])
    world /= np.linalg.norm(world, axis=1, keepdims=True)
    return np.ascontiguousarray(P[:, :3, 3]), np.ascontiguousarray(world)


def run_reference(args):
    """The reference's algorithm on the host cores (the C oracle port of
    octrf's Numba kernels, OpenMP over rays -- the reference package is Python
    + Numba and does not travel to the GPU box): every step is the reference
    train_epoch loop body (optim.py:146-152) on a 2^20-ray batch drawn like
    our arm's -- uniform random rays of the 100-view pool --
    render_and_backprop (count + fill + grad + serial scatter) -> rmsprop_step
    over the touched leaves -> SignalBuffer.accumulate.  Rank 0 only."""
    from oracle import oracle as O
    O.build()
    wl = workloads()[args.workload]  # the same workload as our arm's line
    tree = wl.scene("cpu")
    tree._host()
    focal, poses = wl.cameras()
    n_pool = wl.views * wl.W * wl.H
    sample = args.ref_sample or wl.batch(1)
    rng = np.random.default_rng(11)

    def batch():
        flat = rng.integers(0, n_pool, sample)
        o, d = pool_rays_np(focal, poses, wl.W, wl.H, flat)
        return o, d, rng.uniform(0.0, 1.0, (sample, 3))

    sig = tree.sigma.numpy()
    sh = tree.sh.numpy()
    vs = np.zeros(tree.capacity)
    vh = np.zeros((tree.capacity, 3 * tree.basis_count))
    acc = np.zeros(tree.capacity)

    def step(b):
        o, d, tg = b
        loss, g, s = O.render_and_backprop(tree, o, d, tg, BG, EPS)
        O.rmsprop_step(sig, sh, vs, vh, g.dsigma, g.dsh, g.touched)
        acc[:] += s
        return loss

    batches = [batch() for _ in range(min(args.warmup + args.steps, 4))]  # drawn outside the timing
    for k in range(args.warmup):
        step(batches[k % len(batches)])
    t = time.perf_counter()
    for k in range(args.steps):
        step(batches[(args.warmup + k) % len(batches)])
    dt = time.perf_counter() - t
    value = sample * args.steps / dt
    cores = O.num_threads()
    # the scalar figure: one thread, a 2^16-ray slice
    o, d, tg = batches[0]
    m = 1 << 16
    O.set_threads(1)
    t1 = time.perf_counter()
    O.render_and_backprop(tree, o[:m], d[:m], tg[:m], BG, EPS)
    dt1 = time.perf_counter() - t1
    O.set_threads(cores)
    return {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "rays/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt / args.steps * 1e3,
        "higher_is_better": True, "scaling": wl.scaling, "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded blob-field scene, random-init SH, uniform random targets)",
        "config": workload_config(wl, tree, args.gpus),
        "cpu_baseline": {"value": value, "unit": "rays/s", "cores": cores, "kind": "port",
                         "sample": f"{sample} rays per step (uniform random rays of the {wl.views}-view pool; "
                                   f"{len(batches)} pre-drawn batches cycled), fwd+bwd (count + fill + grad + "
                                   "serial scatter) + RMSProp over the touched leaves + signal accumulate",
                         "one_thread": {"value": m / dt1, "unit": "rays/s", "cores": 1,
                                        "sample": f"{m} rays fwd+bwd, one OpenMP thread"}},
        "e2e": {"value": value, "unit": "rays/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "host": "CPU only (the reference path is CPU code); the line's GPUs are unused",
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--skip-render", action="store_true")
    ap.add_argument("--skip-refine", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--ref-sample", type=int, default=0,
                    help="rays per reference-arm step (default: our arm's per-GPU batch)")
    ap.add_argument("--workload", choices=["c2", "c4"], default="c2",
                    help="c2 = configs[1] (the headline line), c4 = configs[3] (8.5M leaves, 1080p)")
    ap.add_argument("--order", choices=["random", "raster", "morton"], default="random",
                    help="batch ray order handed to the kernel (same ray set)")
    ap.add_argument("--ar-chunks", type=int, default=4,
                    help="row chunks of the overlapped gradient all-reduce (N > 1)")
    ap.add_argument("--exchange", choices=["nccl", "peer"], default="nccl",
                    help="N > 1 gradient exchange: chunked NCCL all-reduce + RMSProp, or the fused "
                         "peer-memory update (dot_rmsprop_step_peers)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_ours(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
