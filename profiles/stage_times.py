"""Per-stage device times of serial frames (CUDA events on the context
stream, lodge_profile): a quick A/B harness for kernel variants
(LODGE_LIB=<variant> picks a diagnostic build).

    python profiles/stage_times.py [--config config3] [--frames 64]
"""

from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--frames", type=int, default=64)
    ap.add_argument("--store", default="flat", choices=["flat", "slab"])
    ap.add_argument("--phase-budget", type=int, default=1536)
    a = ap.parse_args()
    import torch

    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan, SlabStore
    from fixtures import scenes
    import bench

    dev = torch.device("cuda", 0)
    cfg = scenes.build(a.config)
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    if a.store == "slab":
        plan = SlabStore(levels, plan).attach(plan)
    r = L.Renderer(levels, plan, device=dev, storage="fp32", precision="fast",
                   phase_budget=a.phase_budget)
    nv = bench.sweep_views(a.config)
    sweep = cfg.sweep(nv)
    timed, _ = bench.schedules(0, 1, a.frames, 0, 16, nv)
    views = [blk[0] for blk in timed]
    cams = r.upload_cameras([sweep[v] for v in views])
    fr = r.alloc_frame(*sweep[0].resolution)
    r.reserve(200 << 20)
    for i in range(min(4, len(views))):
        r.render(cams[i], fr)
    torch.cuda.synchronize()
    r.profile(True, len(views))
    for i in range(len(views)):
        r.render(cams[i], fr)
    torch.cuda.synchronize()
    ms, n = r.profile_read()
    st = fr.read_stats()
    import ctypes as C
    cnt = (C.c_uint64 * 8)()
    N.check(N.lib().lodge_debug_counters(r.ctx.ptr, cnt), "counters")
    out = {"lib": os.environ.get("LODGE_LIB", "") or "liblodge", "config": a.config,
           "frames": n, "store": a.store, "phase_budget": a.phase_budget,
           "counters_last_frame": list(cnt), "comp_members": int(st.comp_members),
           "stage_ms": {k: round(float(v) / max(n, 1), 5) for k, v in zip(N.STAGES, ms)},
           "frame_ms": round(float(sum(ms)) / max(n, 1), 4), "last_fault": int(st.fault)}
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
