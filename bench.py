#!/usr/bin/env python
"""LODGE per-frame render throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lodge|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one rank per GPU)

Workload (config 5 on config 3): a 4096-view camera sweep at
1920x1080 along a synthetic 20M-Gaussian, 5-LOD, 64-chunk corridor
(fixtures/scenes.py).  Views are block-cyclic over ranks, 16 consecutive
views per block; one step = one block per rank, every view rendered end to
end on the device (chunk selection, union + blend weights, projection, depth
sort, binning, tile sort, compositing, outputs resident in HBM).  Weak
scaling; the store is replicated on every GPU; NCCL gathers metrics only.

--impl reference times the reference algorithm on the host cores: the CPU
restatement in oracle/ (the reference is Python and cannot run on the GPU
box), rank 0 only.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "frames/sec at 1080p (1/2/4/8 B200, views sharded) vs CPU ref; % of HBM roofline"
UNIT = "frames/s"
SWEEP_VIEWS = 4096   # config 5: the sweep over config 3


def sweep_views(cfg_name):
    """Views of the timed path: the config-5 sweep (4096), or config 4's
    1024-view Lissajous path through the room."""
    return 1024 if cfg_name == "config4" else SWEEP_VIEWS
BLOCK = 16


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=24)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="lodge", choices=["lodge", "reference"])
    ap.add_argument("--config", default="config3")
    ap.add_argument("--precision", default="fast", choices=["fast", "exact"])
    ap.add_argument("--views-per-step", type=int, default=BLOCK)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--streams", type=int, default=8,
                    help="frames in flight per GPU (one liblodge context + stream each)")
    ap.add_argument("--cpu-views", type=int, default=1, help="views in the CPU baseline sample")
    ap.add_argument("--residency", default="full", choices=["full", "stream"],
                    help="full: the whole store resident; stream: chunk slabs loaded "
                         "asynchronously into --slots device slots (SURVEY.md 8f rank 4)")
    ap.add_argument("--slots", type=int, default=3)
    ap.add_argument("--store", default="flat", choices=["flat", "slab"],
                    help="full residency layout: flat level arrays, or chunk slabs (every "
                         "chunk's records contiguous in set order; paper_2505_23158_b200."
                         "device.SlabStore)")
    ap.add_argument("--phase-budget", type=int, default=1536,
                    help="FAST frames: first-phase pairs per tile of the two depth phases "
                         "(lodge_set_phase_budget); 0 = one pass over the full lists")
    ap.add_argument("--exact-steps", type=int, default=2,
                    help="steps of the secondary EXACT-precision (fp64 compositing) sample")
    ap.add_argument("--mode", default="blend", choices=["blend", "chunks", "lod", "full"],
                    help="render mode of the reference CLI (src/cli.py:219-243); the "
                         "metric is quoted on blend")
    return ap.parse_args()


def env_rank():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1)),
            int(os.environ.get("LOCAL_RANK", 0)))


def workload_name(cfg_name):
    return {"config3": "config5 sweep over config3: 4096 views, 1920x1080, 20M Gaussians, "
                       "5 LODs, 64 chunks, SH3, chunk opacity blending",
            "config2": "config2 scene (1M Gaussians, 3 LODs, 16 chunks, SH3) swept at 1920x1080",
            "config4": "config4 indoor room: 6M Gaussians, 4 LODs, 32 chunks on a 2-D Voronoi "
                       "tiling, SH3, 1024-view Lissajous path at 1920x1080 with chunk opacity "
                       "blending",
            "street1080": "46k-Gaussian street, 2 LODs, 4 chunks, SH1, 1920x1080"}[cfg_name]


def schedules(rank, world, steps, warmup, block, n_views=SWEEP_VIEWS):
    """Block-cyclic view assignment (paper_2505_23158_b200/shard.py): block b
    of `block` consecutive sweep views goes to rank b % world.  The timed
    steps take this rank's blocks spread evenly over the whole 4096-view
    sweep (step s -> block floor((s + 1/2) * n_mine / steps)); the warm-up
    steps take blocks in between."""
    from paper_2505_23158_b200.shard import spread_schedule
    return (spread_schedule(n_views, world, rank, steps, block, 0.5),
            spread_schedule(n_views, world, rank, warmup, block, 0.0))


def config_of(args, W=1920, H=1080):
    """The workload definition, identical in both arms (run statistics go
    under "run")."""
    return {"workload": workload_name(args.config), "mode": args.mode, "resolution": [W, H],
            "sweep_views": sweep_views(args.config), "views_per_block": BLOCK,
            "schedule": "block-cyclic over ranks, timed blocks spread over the sweep"}


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------
class Clocks:
    """nvidia-smi sampler (every 100 ms) started before the warm-up, so it is
    running when the timed region begins; stop() keeps the samples stamped
    inside [t0, t1] of the timed region, widened to the nearest sample on
    each side when the region is shorter than the sampling period."""
    Q = ("timestamp,index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None
        self.t0 = self.t1 = None

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except OSError:
            self.p = None

    def mark_start(self):
        self.t0 = time.time()

    def mark_end(self):
        self.t1 = time.time()
        time.sleep(0.25)  # let the sample after the region land

    @staticmethod
    def _stamp(s):
        import datetime
        try:
            return datetime.datetime.strptime(s, "%Y/%m/%d %H:%M:%S.%f").timestamp()
        except ValueError:
            return None

    def stop(self):
        if self.p is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.p.kill()
        self.f.flush()
        rows = []
        for line in open(self.f.name):
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 10:
                rows.append((self._stamp(parts[0]), parts[1:]))
        os.unlink(self.f.name)
        if self.t0 is not None and self.t1 is not None:
            inside = [r for ts, r in rows if ts is not None and self.t0 <= ts <= self.t1]
            before = [r for ts, r in rows if ts is not None and ts < self.t0][-1:]
            after = [r for ts, r in rows if ts is not None and ts > self.t1][:1]
            sel = inside if len(inside) >= 2 else before + inside + after
        else:
            sel = [r for _, r in rows]
        if not sel:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(r[1]) for r in sel if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in sel if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in sel for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(sel),
                "window": "inside the timed region" if len(sel) == len(
                    [1 for ts, _ in rows if ts is not None and self.t0 is not None
                     and self.t0 <= ts <= self.t1]) else "timed region plus one sample either side"}


# ---------------------------------------------------------------------------
# algorithmic bytes per stage
# ---------------------------------------------------------------------------
def stage_bytes(U, AB, M, P, W, H, sh_terms, geom_bytes=48, sh_elem=4, P1=None, P2=0.0,
                M1=None, M2=0.0, bl1=0.0, bl2=0.0, C=None):
    """Algorithmic bytes per frame of each stage.
    Two-phase frames (P1 = pairs of the first depth phase < P): the depth
    stage selects and sorts the C first-phase candidates,
    tile_setup is their counting pass, duplicate / tile_sort / composite the
    first phase, second_phase the owner filter over the survivors, the owner
    sort and the lists (sorted pairs or block lists) of the P2 pairs the
    unfinished tiles still need, composite_b their compositing.
    bl1 / bl2: the fraction of frames whose first / second phase kept block
    lists (stats.block_lists): no pairs emitted or sorted; the block-list
    pass reads each splat's rectangle and id (12 B) and writes at least one
    8 B entry per splat."""
    sh_b = 3 * sh_terms * sh_elem
    two = P1 is not None and (P1 < P or P2 > 0)
    P1 = P if P1 is None else P1
    M1 = M if (M1 is None or not two) else M1
    C = M if (C is None or not two) else C
    # a sort of n (32-bit key, index) pairs: histogram read, four passes
    # reading and writing key + index, the tie repair reading keys and
    # indices and writing indices
    sort = lambda n: n * 4.0 + 4 * n * 16.0 + n * 12.0  # noqa: E731
    count = C * (4.0 + 8.0 + 8.0 + 4.0)  # order + rect in, rect + offset out
    # k_payload: id, geometry and SH in, payload + fp64 record out, per
    # composited splat
    payload = 4.0 + 8.0 + geom_bytes + sh_b + 128.0
    blk = lambda m: m * (12.0 + 8.0)  # noqa: E731
    # candidate selection: the histogram reads key, index and rectangle of
    # every survivor, the compaction key and index and writes the candidates
    select = (M * 16.0 + M * 8.0 + C * 8.0) if two else 0.0
    return {
        "select": 0.0,
        "union": 4.0 * AB + 5.0 * U,
        # geometry only: union slot + record in; per survivor the full key and
        # rectangle by index and the compacted (32-bit key, index) out
        "project": U * (5.0 + geom_bytes) + M * 24.0,
        "depth_sort": select + sort(C),
        "tile_setup": (count if two else 0.0) + M1 * payload,
        "duplicate": (1.0 - bl1) * P1 * 8.0 if two else M * 12.0 + P * 8.0,
        # pass 1 reads u64 pairs, writes packed u32; pass 2 reads and writes u32
        "tile_sort": (1.0 - bl1) * (8.0 + 4.0 + 4.0 + 4.0) * P1 + bl1 * blk(M1),
        "composite": P1 * 4.0 + M1 * 64.0 + W * H * 16.0 + U * 4.0,
        # owner filter (key, index, rectangle per survivor; owners out), the
        # owner sort, the owners' counting pass and compositing records, the
        # emitted pairs (8 B) and their two tile passes (20 B) or block lists
        "second_phase": (M * 16.0 + M2 * 8.0 + sort(M2) + M2 * 24.0 + M2 * payload
                         + (1.0 - bl2) * P2 * (8.0 + 20.0) + bl2 * blk(M2)) if two else 0.0,
        "composite_b": (P2 * 4.0 + M2 * 64.0) if two else 0.0,
    }


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def load_traffic(kernel_stage):
    """dram bytes per launch from a committed ncu --set full summary, if any."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(kernel_stage)


# ---------------------------------------------------------------------------
# CPU reference (oracle restatement of the reference algorithm)
# ---------------------------------------------------------------------------
def lod_bounds_of(cfg):
    """select_active's bands for the fixture levels (src/lod.py:203)."""
    return [0.0] + [float(cfg.levels[l][2]) for l in range(1, cfg.L)] + [float("inf")]


def nearest_chunk(centers, position):
    """nearest_two_chunks' first id (src/blending.py:77-84): lexsort by (dist, id)."""
    d = np.linalg.norm(np.asarray(centers) - np.asarray(position), axis=1)
    return int(np.lexsort((np.arange(d.shape[0]), d))[0])


def cpu_render_view(cfg, cam, O, mode="blend"):
    """One view of the given mode on the host cores (oracle restatement):
    blend / chunks (src/blending.py:77-137), lod (src/lod.py:192-237), full
    (src/cli.py:221-226)."""
    oc = O.camera_from(cam)
    rc = O.cfg_struct(_raster_cfg())
    parts = []
    if mode in ("blend", "chunks"):
        f, o, tb, t = O.select(cfg.centers, cam.position)
        if mode == "chunks":
            o, t = None, 1.0
        for l in range(cfg.L):
            b = cfg.set(o, l).astype(np.int64) if o is not None else np.zeros(0, np.int64)
            idx, mod, _ = O.union(cfg.set(f, l).astype(np.int64), b, t)
            g, s, _ = cfg.levels[l]
            parts.append(O.project_f32(g, s, cfg.degree, idx, oc, rc, mod))
    else:
        bounds = lod_bounds_of(cfg)
        q = np.asarray(cam.position, float)
        for l in range(cfg.L):
            g, s, _ = cfg.levels[l]
            if mode == "full":
                idx = np.arange(g.shape[0]) if l == 0 else np.zeros(0, np.int64)
            else:
                dist = np.linalg.norm(g[:, 0:3].astype(np.float64) - q, axis=1)
                idx = np.flatnonzero((dist >= bounds[l]) & (dist < bounds[l + 1]))
            parts.append(O.project_f32(g, s, cfg.degree, idx.astype(np.int64), oc, rc, None))
    batch = O.concat(parts)
    w, h = cam.resolution
    return O.rasterize(batch, w, h, rc, lists=False), batch


def _raster_cfg():
    from paper_2505_23158_b200.types import RasterConfig
    return RasterConfig()


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def run_reference(args):
    rank, world, _ = env_rank()
    if rank != 0:
        return 0
    from fixtures import scenes
    from oracle import oracle as O
    O.lib()
    # all host cores, whatever OMP_NUM_THREADS the launcher exported
    O.set_threads(os.cpu_count() or 1)
    cfg = scenes.build(args.config, threads=os.cpu_count() or 1)
    nv = sweep_views(args.config)
    sweep = cfg.sweep(nv)
    timed, warm = schedules(0, 1, args.steps, args.warmup, BLOCK, nv)
    # one view per step: the first view of the block the GPU arm's rank 0
    # times at that step (the same spread over the sweep)
    for blk in warm:
        cpu_render_view(cfg, sweep[blk[0]], O, args.mode)
    times = []
    for blk in timed:
        t0 = time.perf_counter()
        cpu_render_view(cfg, sweep[blk[0]], O, args.mode)
        times.append(time.perf_counter() - t0)
    total = sum(times)
    fps = len(times) / total
    cores = O.num_threads()
    zs = [float(sweep[blk[0]].position[2]) for blk in timed]
    line = {"metric": METRIC, "value": fps, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * total / len(times),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": config_of(args),
            "cpu_baseline": {"value": fps, "unit": UNIT, "cores": cores, "kind": "port",
                             "sample": f"1 view per step ({len(times)} views, z {min(zs):.0f}.."
                                       f"{max(zs):.0f} of the sweep, the first view of each "
                                       f"block the GPU arm times), oracle/ C restatement with "
                                       f"OpenMP on {cores} threads, {cpu_model()}"},
            "e2e": {"value": fps, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------
FP32_LANES_PER_SM = 128   # FP32 FMA lanes per SM (sm_100)
MUFU_PER_SM = 16          # ex2 per SM per clock (sm_100; B200_PROFILING.md)
FLOPS_PER_PAIR = 20       # fp32 ops per (pixel, member) evaluation


def run_lodge(args):
    import torch
    import torch.distributed as dist

    from fixtures import scenes
    import paper_2505_23158_b200 as LG
    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200 import shard
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
    from paper_2505_23158_b200.renderer import STATS_BYTES

    rank, world, local = env_rank()
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", world))
    # LODGE_BENCH_PLUMBING=1: every rank on cuda:0 over gloo -- a check that
    # the torchrun path runs end to end on a one-GPU box (the ranks never
    # wait on each other's kernels); its numbers are not scaling numbers
    plumbing = os.environ.get("LODGE_BENCH_PLUMBING") == "1"
    if plumbing:
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if plumbing:
            dist.init_process_group("gloo")
        else:
            # NCCL's init log names every rank and its device (the driver's
            # rank check); the data path itself exchanges nothing
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
    barrier = dist.barrier if world > 1 else (lambda: None)
    t_setup = time.time()
    # the fixture is generated once per node (local rank 0, every host core)
    # and memory-mapped by the node's other ranks
    cfg = scenes.build_shared(args.config, local, local_world, barrier,
                              key=os.environ.get("MASTER_PORT", ""))
    store = None
    if args.residency == "stream":
        # residency-bounded store: chunk slabs streamed into args.slots slots
        if args.mode not in ("blend", "chunks"):
            raise SystemExit("--residency stream renders the chunk modes (blend, chunks)")
        from paper_2505_23158_b200.streaming import StreamingStore, host_pair
        store = StreamingStore([(g, s) for g, s, _ in cfg.levels], cfg.centers, cfg.offsets,
                               cfg.data, dev, n_slots=args.slots)
        levels = store.device_levels()
        plan = store.attach(DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L,
                                                   dev))
        store_gb = store.resident_bytes() / 1e9
    else:
        import warnings
        with warnings.catch_warnings():  # memory-mapped (read-only) fixture arrays
            warnings.simplefilter("ignore", UserWarning)
            levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev),
                                               torch.from_numpy(s).to(dev), cfg.degree)
                      for g, s, _ in cfg.levels]
        plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, np.asarray(cfg.data), cfg.L,
                                      dev)
        store_gb = sum(l.nbytes() for l in levels) / 1e9
        if args.store == "slab":
            from paper_2505_23158_b200.device import SlabStore
            slabs = SlabStore(levels, plan)
            plan = slabs.attach(plan)
            store_gb += slabs.nbytes() / 1e9
    r = LG.Renderer(levels, plan, device=dev, storage="fp32", precision=args.precision,
                    n_streams=args.streams, phase_budget=args.phase_budget)
    B = args.views_per_step
    nv = sweep_views(args.config)
    timed, warm = schedules(rank, world, args.steps, args.warmup, B, nv)
    sweep = cfg.sweep(nv)
    W, H = sweep[0].resolution
    flat = sorted({v for blk in timed + warm for v in blk})
    pos = {v: i for i, v in enumerate(flat)}
    cams = r.upload_cameras([sweep[v] for v in flat])
    frames = [r.alloc_frame(W, H) for _ in range(B)]
    n_timed = args.steps * B
    bounds = lod_bounds_of(cfg)
    near = {v: nearest_chunk(cfg.centers, sweep[v].position) for v in flat}
    pairs = ({v: host_pair(cfg.centers, sweep[v].position) for v in flat}
             if store is not None else None)

    def do_render(rr, cam_row, frame, slot, v, srgb8=None):
        """One frame of args.mode (the CLI's render modes, src/cli.py:219-243).
        srgb8: the 8-bit sRGB image written by the compositor itself (the
        float image is then not stored); else the float image."""
        kw = {} if srgb8 is None else {"srgb8_out": srgb8, "float_image": False}
        if store is not None:  # chunk pair decided on the host, slabs made resident
            f, o, t = pairs[v]
            if args.mode == "chunks":
                o, t = None, 1.0
            st = rr.stream_of(slot)
            store.require([f, o], st)
            rr.render(cam_row, frame, pair=(f, o), t=t, slot=slot, **kw)
            store.release([f, o], st)
        elif args.mode == "blend":
            rr.render(cam_row, frame, slot=slot, **kw)
        elif args.mode == "chunks":
            rr.render(cam_row, frame, pair=(near[v], None), slot=slot, **kw)
        else:
            if srgb8 is not None:  # render_lod has no 8-bit output: convert
                rr.render_lod(cam_row, frame, bounds, full=args.mode == "full", slot=slot)
                rr.to_srgb8(frame, srgb8, slot=slot)
            else:
                rr.render_lod(cam_row, frame, bounds, full=args.mode == "full", slot=slot)

    def read_stats(t):
        raw = t.cpu().numpy()
        return [N.FrameStats.from_buffer_copy(raw[i].tobytes()) for i in range(raw.shape[0])]

    # sizing: every scheduled view once, then reserve pairs for the largest
    sizing = torch.zeros((len(flat), STATS_BYTES), dtype=torch.uint8, device=dev)
    r.reserve(64 << 20)
    torch.cuda.synchronize()
    for i, v in enumerate(flat):
        do_render(r, cams[pos[v]], frames[0], 0, v)
        with torch.cuda.stream(r.stream_of(0)):
            sizing[i].copy_(frames[0].stats)
    torch.cuda.synchronize()
    P_max = max(s.P for s in read_stats(sizing))
    r.reserve(int(P_max * 1.05) + 4096)
    launches_per_frame = r.last_launch_count()
    clocks = Clocks(local)
    clocks.start()  # sampling before the timed region starts
    for blk in warm:
        for j, v in enumerate(blk):
            do_render(r, cams[pos[v]], frames[j], j % r.n_streams, v)
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    # ---- timed region ----------------------------------------------------
    # frame j of a step runs on slot j % n_streams (own context + stream); the
    # region is bracketed by events on the current stream that every slot
    # stream waits on / is waited for.
    S = r.n_streams
    stats_all = torch.zeros((n_timed, STATS_BYTES), dtype=torch.uint8, device=dev)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    clocks.mark_start()
    cur = torch.cuda.current_stream(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(cur)
    for q in range(S):
        r.stream_of(q).wait_event(e0)
    k = 0
    for blk in timed:
        for j, v in enumerate(blk):
            do_render(r, cams[pos[v]], frames[j], j % S, v)
            with torch.cuda.stream(r.stream_of(j % S)):
                stats_all[k].copy_(frames[j].stats, non_blocking=True)
            k += 1
    for q in range(S):
        cur.wait_stream(r.stream_of(q))
    e1.record(cur)
    torch.cuda.synchronize()
    clocks.mark_end()
    clk = clocks.stop()
    if world > 1:
        dist.barrier()
    ms = e0.elapsed_time(e1)
    ms_max = shard.max_over_ranks(ms, dev)
    total_frames = n_timed * world
    value = total_frames / (ms_max / 1000.0)
    stats = read_stats(stats_all)
    overflow = sum(1 for s in stats if s.overflow)
    faults = sum(1 for s in stats if s.fault)

    # ---- per-stage times: the timed views re-rendered serially on one
    # stream (with frames in flight a stage's events would also span the
    # other streams' kernels), with the single-frame persistent grids
    # (grid_share 0: a frame alone on the GPU)
    n_stage = min(n_timed, 64)
    share = r.grid_share
    r.grid_share = 0
    r.profile(True, n_stage)
    k = 0
    for blk in timed:
        for j, v in enumerate(blk):
            if k < n_stage:
                do_render(r, cams[pos[v]], frames[j], 0, v)
            k += 1
    torch.cuda.synchronize()
    stage_ms, nprof_frames = r.profile_read()
    r.profile(False)
    r.grid_share = share
    stage_timing = (f"events around each stage, {nprof_frames} of the timed views re-rendered "
                    "serially on one stream after the timed region, single-frame grids")

    # ---- per-stage roofline ----------------------------------------------
    mean = lambda f: float(np.mean([f(s) for s in stats]))  # noqa: E731
    U, M, P = mean(lambda s: s.U), mean(lambda s: s.M), mean(lambda s: s.P)

    def set_total(j):  # sum over levels of |set(j, l)|
        return int(cfg.offsets[(j + 1) * cfg.L] - cfg.offsets[j * cfg.L]) if j >= 0 else 0

    AB = mean(lambda s: set_total(s.f) + set_total(s.o))
    P1, P2 = mean(lambda s: s.P_first), mean(lambda s: s.P_second)
    M1, M2 = mean(lambda s: s.M_first), mean(lambda s: s.M_second)
    bl1 = mean(lambda s: s.block_lists & 1)
    bl2 = mean(lambda s: (s.block_lists >> 1) & 1)
    Cs = mean(lambda s: s.sorted_first)
    sb = stage_bytes(U, AB, M, P, W, H, (cfg.degree + 1) ** 2, P1=P1, P2=P2, M1=M1, M2=M2,
                     bl1=bl1, bl2=bl2, C=Cs)
    peak, peak_kind = load_peaks()
    stages = {}
    for i, name in enumerate(N.STAGES):
        per = stage_ms[i] / max(nprof_frames, 1)
        gbs = sb[name] / (per / 1000.0) / 1e9 if per > 0 else 0.0
        stages[name] = {"ms_per_frame": round(per, 5), "bytes_per_frame": round(sb[name]),
                        "GB_s": round(gbs, 1), "frac": round(gbs / peak, 4)}
    # compositing (K6) against the FP32 and MUFU pipes:
    # E = 256 * sum over tiles of m_t pixel-member evaluations per frame
    m_t = mean(lambda s: s.comp_members)
    E = 256.0 * m_t
    t_comp = (stages["composite"]["ms_per_frame"] + stages["composite_b"]["ms_per_frame"]) / 1e3
    props = torch.cuda.get_device_properties(dev)
    sm_hz = (clk.get("sm_mhz") or clk.get("sm_max_mhz") or 1965.0) * 1e6
    fp32_peak = props.multi_processor_count * FP32_LANES_PER_SM * 2 * sm_hz
    mufu_peak = props.multi_processor_count * MUFU_PER_SM * sm_hz
    compositor = {"members_iterated_per_frame": round(m_t), "E_per_frame": E,
                  "seconds_per_frame": round(t_comp, 7),
                  "fp32_frac": round(FLOPS_PER_PAIR * E / t_comp / fp32_peak, 4) if t_comp else None,
                  "mufu_frac": round(E / t_comp / mufu_peak, 4) if t_comp else None,
                  "fp32_peak_tflops": round(fp32_peak / 1e12, 1),
                  "mufu_peak_tex2": round(mufu_peak / 1e12, 2),
                  "clock_mhz": round(sm_hz / 1e6), "sms": props.multi_processor_count,
                  "note": "E = 256 x members a tile iterates before all its pixels have "
                          "T < t_min (stats.comp_members, both phases); 20 fp32 ops and one "
                          "ex2 per evaluation; time = composite + composite_b stages"}
    hbm_stages = ["union", "project", "depth_sort", "duplicate", "tile_sort"]
    dom = max(N.STAGES, key=lambda k: stages[k]["ms_per_frame"])
    rf_stage = max(hbm_stages, key=lambda k: stages[k]["ms_per_frame"])
    rs = stages[rf_stage]
    roofline = {"bound": "hbm", "kernel": rf_stage, "achieved": rs["GB_s"], "peak": peak,
                "unit": "GB/s", "frac": rs["frac"], "peak_kind": peak_kind,
                "traffic": load_traffic(rf_stage),
                "bytes_per_launch": rs["bytes_per_frame"], "ms_per_launch": rs["ms_per_frame"],
                "dominant_stage": dom,
                "note": ("the longest HBM-bound stage; composite is FP32/MUFU-bound, see "
                         "compositor" if dom.startswith("composite") else "")}

    # ---- EXACT precision (fp64 compositing) on a short sample --------------
    exact = None
    if args.precision == "fast" and args.exact_steps > 0 and args.mode == "blend" \
            and store is None:
        rx = LG.Renderer(levels, plan, device=dev, storage="fp32", precision="exact",
                         n_streams=S)
        rx.reserve(int(P_max * 1.05) + 4096)
        fx = [rx.alloc_frame(W, H) for _ in range(B)]
        sx = timed[:args.exact_steps]
        for j, v in enumerate(sx[0]):  # warm-up
            rx.render(cams[pos[v]], fx[j], slot=j % S)
        torch.cuda.synchronize()
        x0, x1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        x0.record(cur)
        for q in range(S):
            rx.stream_of(q).wait_event(x0)
        for blk in sx:
            for j, v in enumerate(blk):
                rx.render(cams[pos[v]], fx[j], slot=j % S)
        for q in range(S):
            cur.wait_stream(rx.stream_of(q))
        x1.record(cur)
        torch.cuda.synchronize()
        xms = shard.max_over_ranks(x0.elapsed_time(x1), dev)
        nx = sum(len(b) for b in sx)
        exact = {"value": nx * world / (xms / 1000.0), "unit": UNIT, "frames": nx * world,
                 "note": "fp64 compositing reproducing the reference's blocked transmittance "
                         "(image <= 1e-12 of the oracle), same views, frames in flight"}
        del rx, fx
        torch.cuda.empty_cache()

    # ---- end to end through the public API --------------------------------
    e2e = None
    if not args.no_e2e:
        # double-buffered pinned camera upload (the host refills a buffer only
        # after its previous copy completed), renders on the slot streams;
        # each frame's 8-bit image is written by the compositor straight into
        # pinned host memory (zero-copy: 16-byte row segments over PCIe as the
        # tiles finish -- a separate copy-engine read-back of a device image
        # cost ~7%) and its stats are read back by a D2H copy
        cam_host = [torch.empty((B, cams.shape[1]), dtype=torch.uint8).pin_memory()
                    for _ in range(2)]
        cam_dev = [torch.empty((B, cams.shape[1]), dtype=torch.uint8, device=dev)
                   for _ in range(2)]
        copied = [torch.cuda.Event(), torch.cuda.Event()]
        # per parity and slot: the renders that read cam_dev[parity] are done
        # (the upload two steps later must not overwrite a camera in use)
        used = [[torch.cuda.Event() for _ in range(S)] for _ in range(2)]
        # frame and 8-bit image buffers double-buffered by step parity, so a
        # buffer's read-back has a whole step to finish before it is reused
        frames2 = [frames, [r.alloc_frame(W, H) for _ in range(B)]]
        # LOD / full modes convert with a separate full-grid kernel
        # (render_lod has no 8-bit output): writing over PCIe from it would
        # hold every SM for the transfer, so those modes convert into HBM
        # and read back with the copy engine
        direct = args.mode in ("blend", "chunks")
        img8 = None if direct else torch.empty((2, B, H, W, 3), dtype=torch.uint8, device=dev)
        img8_host = torch.empty((2, B, H, W, 3), dtype=torch.uint8).pin_memory()
        st_host = torch.empty((2, B, STATS_BYTES), dtype=torch.uint8).pin_memory()
        cams_host = cams.cpu()
        # read-backs on one copy stream per slot: a frame's D2H copy overlaps
        # the next frames of its slot; a frame buffer is re-rendered only
        # after its previous copy completed
        copy_s = [torch.cuda.Stream(device=dev) for _ in range(S)]
        ready = [[torch.cuda.Event() for _ in range(B)] for _ in range(2)]
        drained = [[torch.cuda.Event() for _ in range(B)] for _ in range(2)]
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(cur)
        for si, blk in enumerate(timed):
            par = si & 1
            if si >= 2:
                copied[par].synchronize()
            for j, v in enumerate(blk):
                cam_host[par][j].copy_(cams_host[pos[v]])
            if si >= 2:
                for q in range(S):
                    cur.wait_event(used[par][q])
            cam_dev[par].copy_(cam_host[par], non_blocking=True)
            copied[par].record(cur)
            for q in range(S):
                r.stream_of(q).wait_stream(cur)
            for j, v in enumerate(blk):
                q = j % S
                fr = frames2[par][j]
                if si >= 2:  # this buffer's read-back two steps ago is done
                    r.stream_of(q).wait_event(drained[par][j])
                do_render(r, cam_dev[par][j], fr, q, v,
                          srgb8=img8_host[par, j] if direct else img8[par, j])
                ready[par][j].record(r.stream_of(q))
                with torch.cuda.stream(copy_s[q]):
                    copy_s[q].wait_event(ready[par][j])
                    if not direct:
                        img8_host[par, j].copy_(img8[par, j], non_blocking=True)
                    st_host[par, j].copy_(fr.stats, non_blocking=True)
                    drained[par][j].record(copy_s[q])
            for q in range(S):
                used[par][q].record(r.stream_of(q))
        for q in range(S):
            cur.wait_stream(r.stream_of(q))
            cur.wait_stream(copy_s[q])
        f1.record(cur)
        torch.cuda.synchronize()
        ems = shard.max_over_ranks(f0.elapsed_time(f1), dev)
        # after the timed region: the last step's first host image equals the
        # same view rendered again into a device buffer
        lp, lv = (len(timed) - 1) & 1, timed[-1][0]
        chk = torch.empty((H, W, 3), dtype=torch.uint8, device=dev)
        do_render(r, cams[pos[lv]], frames2[lp][0], 0, lv, srgb8=chk)
        torch.cuda.synchronize()
        host_ok = bool(torch.equal(chk.cpu(), img8_host[lp, 0]))
        e2e = {"value": total_frames / (ems / 1000.0), "unit": UNIT,
               "host_image_check": host_ok,
               "h2d_bytes_per_step": int(B * cams.shape[1]),
               "d2h_bytes_per_step": int(B * (H * W * 3 + STATS_BYTES)),
               "path": ("Renderer.render(srgb8_out=<pinned host tensor>): the compositor writes "
                        "the 8-bit sRGB image (byte for byte to_srgb8, like splatlod render's "
                        "to_uint8) straight into pinned host memory (zero-copy D2H over PCIe)"
                        if direct else
                        "Renderer.render_lod + to_srgb8 into HBM (byte for byte like splatlod "
                        "render's to_uint8), D2H copy of the 8-bit image")
                       + "; pinned host camera upload (H2D copy) and stats read-back (D2H copy) "
                         "every step"}
        if not host_ok:
            e2e["invalid"] = "the host image differs from a device re-render of the same view"
            print("[bench] e2e host image check FAILED", file=sys.stderr)

    # ---- gather per-rank metrics and the timed view ids over NCCL ----------
    per_rank = torch.tensor([ms, float(n_timed), P, float(overflow), float(faults)],
                            dtype=torch.float64, device=dev)
    gathered = shard.gather_rows(per_rank)
    overflow_all = int(gathered[:, 3].sum().item())
    faults_all = int(gathered[:, 4].sum().item())
    my_ids = torch.tensor([v for blk in timed for v in blk], dtype=torch.int64, device=dev)
    last = timed[-1]
    sums = torch.stack([frames[j].image.double().sum() for j in range(len(last))]).reshape(-1, 1)
    g_ids, _ = shard.gather_views(my_ids, torch.zeros((my_ids.numel(), 1), device=dev),
                                  max_per_rank=n_timed)
    _, g_sums = shard.gather_views(torch.tensor(last, dtype=torch.int64, device=dev), sums,
                                   max_per_rank=B)
    ids = g_ids.cpu().numpy()
    coverage = {"views": int(ids.size), "distinct": int(np.unique(ids).size),
                "expected": total_frames, "first": int(ids.min()), "last": int(ids.max()),
                "z_range": [round(float(sweep[int(ids.min())].position[2]), 1),
                            round(float(sweep[int(ids.max())].position[2]), 1)],
                "image_checksum_last_step": float(g_sums.sum().item()),
                "how": "all_gather over " + ("NCCL" if world > 1 and not plumbing else
                                            "gloo" if world > 1 else "(single rank)")}
    coverage["all_distinct"] = coverage["distinct"] == coverage["views"] == total_frames

    # ---- CPU baseline and parity sample (rank 0, after the timed region) ---
    cpu = None
    parity = None
    if rank == 0 and not args.no_cpu_baseline:
        from oracle import oracle as O
        O.lib()
        O.set_threads(os.cpu_count() or 1)
        v = timed[0][0]
        cam = sweep[v]
        t0 = time.perf_counter()
        for _ in range(args.cpu_views):
            ref, batch = cpu_render_view(cfg, cam, O, args.mode)
        dt = (time.perf_counter() - t0) / args.cpu_views
        cpu = {"value": 1.0 / dt, "unit": UNIT, "cores": O.num_threads(), "kind": "port",
               "sample": f"{args.cpu_views} view(s) of the same sweep (z={cam.position[2]:.2f}), "
                         f"oracle/ C restatement, OpenMP {O.num_threads()} threads, "
                         f"{cpu_model()}, {dt:.1f} s/view"}
        fr = frames[0]
        do_render(r, cams[pos[v]], fr, 0, v)
        torch.cuda.synchronize()
        st = fr.read_stats()
        img = fr.image.double().cpu().numpy()
        err = float(np.abs(img - ref["image"]).max())
        mse = float(np.mean((img - ref["image"]) ** 2))
        parity = {"view": int(v), "tile_count_exact": bool(np.array_equal(
            fr.tile_count.cpu().numpy(), ref["per_tile_count"])), "P": int(st.P),
            "P_oracle": int(ref["P"]), "M": int(st.M), "M_oracle": int(len(batch["src"])),
            "image_max_abs": err, "psnr_db": (math.inf if mse == 0 else -10 * math.log10(mse)),
            "lists": "bit-exact per-tile lists at this scale: tests/test_gpu_bench_parity.py"}

    sticky = r.fault_flags()  # every frame of the run, timed or not
    invalid = []
    if overflow_all:
        invalid.append(f"{overflow_all} timed frame(s) overflowed their pair buffers")
    if faults_all or sticky:
        invalid.append(f"device bounds checks fired ({faults_all} timed frame(s), "
                       f"flags {sticky:#x})")
    if invalid:
        print("[bench] INVALID: " + "; ".join(invalid), file=sys.stderr)
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64 projection / f32 compositing (fp64 guard band)", "data": "synthetic",
            "config": config_of(args, W, H),
            "run": {"precision": args.precision,
                    "phase_budget": args.phase_budget if args.precision == "fast" else 0,
                    "frames_in_flight_per_gpu": S, "views_per_step_per_gpu": B,
                    "frames_timed": total_frames,
                    "store": (f"fp32 records, replicated ({args.store} layout)" if store is None else
                              f"fp32 chunk slabs, {args.slots} resident slots, "
                              f"{store.loads} loads ({store.bytes_loaded / 1e9:.1f} GB)"),
                    "store_gb": round(store_gb, 2),
                    "l2": "inputs larger than L2: per-frame working set "
                          f"~{(sb['project'] + sb['tile_sort'] + sb['composite']) / 1e9:.2f} GB"
                          f" and a {store_gb:.1f} GB store >> 126 MB L2; no explicit flush",
                    "mean_U": round(U), "mean_M": round(M), "mean_P": round(P),
                    "mean_P_phase": [round(P1), round(P2)],
                    "mean_M_composited": [round(M1), round(M2)],
                    "block_list_frames": [round(bl1, 3), round(bl2, 3)],
                    "mean_sorted": [round(Cs), round(M2)],
                    "levels": cfg.n_gaussians(), "chunks": cfg.K,
                    "pairs_per_s": P * value, "gaussians_per_s": U * value,
                    "overflow_frames": overflow_all, "fault_frames": faults_all,
                    "fault_flags": int(sticky), "setup_s": round(setup_s, 1)},
            "e2e": e2e, "gpu_launches": int(launches_per_frame * total_frames),
            "roofline": roofline, "compositor": compositor, "stages": stages,
            "stage_timing": stage_timing, "exact": exact,
            "cpu_baseline": cpu, "clocks": clk,
            "parity_sample": parity, "gathered": coverage,
        }
        if invalid:
            line["invalid"] = "; ".join(invalid)
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 1 if invalid else 0


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_lodge(args)


if __name__ == "__main__":
    sys.exit(main())
