"""Where the end-to-end frame rate goes (bench.py's e2e loop, config 3,
four frames in flight): the device loop alone, + 8-bit sRGB conversion,
+ the image/stats read-back, + the per-step pinned camera upload.

    python profiles/e2e_breakdown.py [--steps 24]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=24)
    a = ap.parse_args()
    import torch
    import paper_2505_23158_b200 as L
    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
    from fixtures import scenes
    import bench
    dev = torch.device("cuda", 0)
    cfg = scenes.build("config3")
    levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev),
                                       cfg.degree) for g, s, _ in cfg.levels]
    plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
    S, B = 4, 16
    r = L.Renderer(levels, plan, device=dev, storage="fp32", precision="fast", n_streams=S)
    nv = bench.sweep_views("config3")
    sweep = cfg.sweep(nv)
    timed, _ = bench.schedules(0, 1, a.steps, 0, B, nv)
    flat = sorted({v for blk in timed for v in blk})
    pos = {v: i for i, v in enumerate(flat)}
    cams = r.upload_cameras([sweep[v] for v in flat])
    W, H = sweep[0].resolution
    frames = [r.alloc_frame(W, H) for _ in range(B)]
    r.reserve(200 << 20)
    img8 = torch.empty((B, H, W, 3), dtype=torch.uint8, device=dev)
    img8_host = torch.empty((B, H, W, 3), dtype=torch.uint8).pin_memory()
    st_host = torch.empty((B, frames[0].stats.numel()), dtype=torch.uint8).pin_memory()
    cur = torch.cuda.current_stream(dev)

    def run(srgb, readback, upload):
        cam_host = [torch.empty((B, cams.shape[1]), dtype=torch.uint8).pin_memory()
                    for _ in range(2)]
        cam_dev = [torch.empty((B, cams.shape[1]), dtype=torch.uint8, device=dev)
                   for _ in range(2)]
        cams_host = cams.cpu()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(cur)
        t0 = time.perf_counter()
        for si, blk in enumerate(timed):
            par = si & 1
            if upload:
                for j, v in enumerate(blk):
                    cam_host[par][j].copy_(cams_host[pos[v]])
                cam_dev[par].copy_(cam_host[par], non_blocking=True)
            for q in range(S):
                r.stream_of(q).wait_stream(cur)
            for j, v in enumerate(blk):
                cam = cam_dev[par][j] if upload else cams[pos[v]]
                r.render(cam, frames[j], slot=j % S)
                if srgb:
                    r.to_srgb8(frames[j], img8[j], slot=j % S)
                if readback:
                    with torch.cuda.stream(r.stream_of(j % S)):
                        img8_host[j].copy_(img8[j], non_blocking=True)
                        st_host[j].copy_(frames[j].stats, non_blocking=True)
        for q in range(S):
            cur.wait_stream(r.stream_of(q))
        e1.record(cur)
        t1 = time.perf_counter()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        n = len(timed) * B
        return {"fps": round(n / (ms / 1e3), 1), "host_ms_per_frame": round((t1 - t0) * 1e3 / n, 4)}

    run(False, False, False)  # warm-up
    out = {"device": run(False, False, False), "+srgb": run(True, False, False),
           "+readback": run(True, True, False), "+upload": run(True, True, True),
           "device_again": run(False, False, False)}
    print(json.dumps(out))


if __name__ == "__main__":
    main()
