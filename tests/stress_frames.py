"""Frames-in-flight stress of the fused frame path (a diagnostic runner; the
pytest wrapper is tests/test_gpu_stress.py).

    LODGE_LIB=verify python -m tests.stress_frames --config config3 \\
        --streams 4 --frames 432 --reps 3

Renders `frames` views spread over the whole config-5 sweep, frame j on slot
j % streams (one liblodge context + CUDA stream each, as bench.py does), and
reads every frame's stats; every frame's outputs (image, per_pixel_visible,
per_tile_count, max weights) are checksummed and compared with the same
view rendered serially on one stream (frames are bitwise deterministic).  With a LODGE_VERIFY library (LODGE_LIB=verify)
the device checks the depth order after the sort (FAULT_DEPTH) and every
per-tile list after each tile sort (FAULT_LISTORD); the bounds checks of
every build report the rest.  Prints one JSON line: frames rendered, frames
with each fault bit, overflowed attempts, and the sticky per-context flags.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

FAULT_BITS = {1: "owners", 2: "compact", 4: "scatter", 8: "list", 16: "tile", 32: "payload",
              64: "depth_order", 128: "member", 256: "src", 512: "list_order"}


def run(config="config3", streams=4, frames=432, reps=1, phase_budget=1536, views=4096,
        seed_views=0, cfg=None):
    import numpy as np
    import torch

    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
    from paper_2505_23158_b200.renderer import STATS_BYTES
    from fixtures import scenes

    dev = torch.device("cuda", 0)
    t0 = time.time()
    if cfg is None:
        cfg = scenes.build(config)
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    r = L.Renderer(levels, plan, device=dev, storage="fp32", precision="fast",
                   n_streams=streams, phase_budget=phase_budget)
    sweep = cfg.sweep(views)
    rng = np.random.default_rng(seed_views)
    order = rng.permutation(len(sweep))[:frames] if frames < len(sweep) else \
        np.arange(frames) % len(sweep)
    cams = r.upload_cameras([sweep[int(v)] for v in order])
    W, H = sweep[0].resolution
    B = 16
    outs = [r.alloc_frame(W, H) for _ in range(B)]
    # sizing pass (one stream), then pair buffers for the largest view
    st_all = torch.zeros((len(order), STATS_BYTES), dtype=torch.uint8, device=dev)
    r.reserve(64 << 20)
    for i in range(len(order)):
        r.render(cams[i], outs[0], slot=0)
        with torch.cuda.stream(r.stream_of(0)):
            st_all[i].copy_(outs[0].stats)
    torch.cuda.synchronize()
    raw = st_all.cpu().numpy()
    P_max = max(N.FrameStats.from_buffer_copy(raw[i].tobytes()).P for i in range(len(order)))
    r.reserve(int(P_max * 1.05) + 4096)

    def checksum(fr, row):
        # image, per_pixel_visible, per_tile_count and max weights as integer
        # sums of their bit patterns: any silent corruption changes one
        row[0] = fr.image.view(torch.int32).to(torch.int64).sum()
        row[1] = fr.visible.to(torch.int64).sum()
        row[2] = fr.tile_count.to(torch.int64).sum()
        row[3] = fr.maxw.view(torch.int32).to(torch.int64).sum()

    # reference outputs: every view once more, serially on one stream
    ref = torch.zeros((len(order), 4), dtype=torch.int64, device=dev)
    for i in range(len(order)):
        r.render(cams[i], outs[0], slot=0)
        with torch.cuda.stream(r.stream_of(0)):
            checksum(outs[0], ref[i])
    torch.cuda.synchronize()
    sums = torch.zeros_like(ref)
    setup_s = time.time() - t0
    counts = {name: 0 for name in FAULT_BITS.values()}
    n = overflow = mismatch = 0
    t1 = time.time()
    for _ in range(reps):
        for i in range(len(order)):
            j = i % B
            slot = j % streams
            r.render(cams[i], outs[j], slot=slot)
            with torch.cuda.stream(r.stream_of(slot)):
                st_all[i].copy_(outs[j].stats, non_blocking=True)
                checksum(outs[j], sums[i])
        torch.cuda.synchronize()
        mismatch += int((sums != ref).any(dim=1).sum().item())
        raw = st_all.cpu().numpy()
        for i in range(len(order)):
            st = N.FrameStats.from_buffer_copy(raw[i].tobytes())
            n += 1
            overflow += int(st.overflow != 0)
            for bit, name in FAULT_BITS.items():
                if st.fault & bit:
                    counts[name] += 1
    run_s = time.time() - t1
    sticky = r.fault_flags()
    return {"lib": os.environ.get("LODGE_LIB", "") or "liblodge", "config": config,
            "streams": streams, "frames": n, "overflow": overflow,
            "output_mismatch": mismatch,
            "fault_frames": {k: v for k, v in counts.items() if v},
            "sticky": int(sticky), "setup_s": round(setup_s, 1), "run_s": round(run_s, 2)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--frames", type=int, default=432)
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--phase-budget", type=int, default=1536)
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    res = run(a.config, a.streams, a.frames, a.reps, a.phase_budget, seed_views=a.seed)
    print(json.dumps(res), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
