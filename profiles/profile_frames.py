"""Short, serial frame loop for ncu (profiles/*): builds a bench config,
renders `warm` frames, then `frames` frames of the bench's timed views on
one stream, and prints the kernels per frame.  Under

    ncu --profile-from-start off --metrics gpu__time_duration.sum \\
        --clock-control none --csv --log-file ... python profiles/profile_frames.py

it gives the per-launch device times of whole frames (cold-cache and
serialised: shares, not absolutes); with --set full and -k it gives the
per-kernel counters (DRAM bytes, pipes, stalls) the bench's roofline cites.
"""

from __future__ import annotations

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="config3")
    ap.add_argument("--warm", type=int, default=3)
    ap.add_argument("--frames", type=int, default=2)
    ap.add_argument("--view", type=int, default=-1, help="one sweep view (default: bench views)")
    a = ap.parse_args()
    import torch

    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
    from fixtures import scenes
    import bench

    dev = torch.device("cuda", 0)
    cfg = scenes.build(a.config)
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    r = L.Renderer(levels, plan, device=dev, storage="fp32", precision="fast")
    nv = bench.sweep_views(a.config)
    sweep = cfg.sweep(nv)
    timed, _ = bench.schedules(0, 1, max(a.frames, 1), 0, 16, nv)
    views = [a.view] * a.frames if a.view >= 0 else [blk[0] for blk in timed][:a.frames]
    cams = r.upload_cameras([sweep[v] for v in views])
    fr = r.alloc_frame(*sweep[0].resolution)
    r.reserve(200 << 20)
    for _ in range(a.warm):
        r.render(cams[0], fr)
    torch.cuda.synchronize()
    launches = r.last_launch_count()
    print(f"[profile_frames] config={a.config} views={views} kernels/frame={launches}",
          flush=True)
    torch.cuda.profiler.start()  # ncu --profile-from-start off: only these frames
    for i in range(a.frames):
        r.render(cams[i], fr)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    st = fr.read_stats()
    print(f"[profile_frames] last frame U={st.U} M={st.M} P={st.P} P1={st.P_first} "
          f"P2={st.P_second} fault={st.fault}", flush=True)
    assert st.fault == 0 and st.overflow == 0


if __name__ == "__main__":
    main()
