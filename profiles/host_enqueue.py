import time, sys, os, json
sys.path.insert(0, '/root/repo')
import torch
import paper_2505_23158_b200 as L
from paper_2505_23158_b200.device import DeviceLevel, DevicePlan
from fixtures import scenes
import bench
dev = torch.device("cuda", 0)
cfg = scenes.build("config3")
levels = [DeviceLevel.from_tensors(torch.from_numpy(g).to(dev), torch.from_numpy(s).to(dev), cfg.degree) for g, s, _ in cfg.levels]
plan = DevicePlan.from_arrays(cfg.centers, cfg.offsets, cfg.data, cfg.L, dev)
r = L.Renderer(levels, plan, device=dev, storage="fp32", precision="fast", n_streams=4)
sweep = cfg.sweep(4096)
views = list(range(0, 4096, 16))[:64]
cams = r.upload_cameras([sweep[v] for v in views])
frames = [r.alloc_frame(*sweep[0].resolution) for _ in range(16)]
r.reserve(200 << 20)
for i in range(16):
    r.render(cams[i], frames[i], slot=i % 4)
torch.cuda.synchronize()
out = {}
for n in (4, 8, 16):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for i in range(n):
        r.render(cams[i], frames[i], slot=i % 4)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out[n] = {"host_ms_per_frame": (t1 - t0) * 1e3 / n, "total_ms_per_frame": (t2 - t0) * 1e3 / n}
# srgb + copy cost on host
img8 = torch.empty((16, 1080, 1920, 3), dtype=torch.uint8, device=dev)
torch.cuda.synchronize()
t0 = time.perf_counter()
for i in range(16):
    r.render(cams[i], frames[i], slot=i % 4)
    r.to_srgb8(frames[i], img8[i], slot=i % 4)
t1 = time.perf_counter()
torch.cuda.synchronize()
out["render+srgb"] = (t1 - t0) * 1e3 / 16
print(json.dumps(out))
