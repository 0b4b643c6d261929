import os, sys
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
r = L.Renderer(levels, plan, device=dev, storage="fp32", precision="fast")
sweep = cfg.sweep(4096)
cams = r.upload_cameras([sweep[1000]])
fr = r.alloc_frame(*sweep[0].resolution)
r.reserve(400 << 20)
bounds = None
for _ in range(3):
    r.render_lod(cams[0], fr, bounds, full=True)
torch.cuda.synchronize()
torch.cuda.profiler.start()
r.render_lod(cams[0], fr, bounds, full=True)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
st = fr.read_stats(); print("U", st.U, "M", st.M, "P", st.P, "fault", st.fault)
