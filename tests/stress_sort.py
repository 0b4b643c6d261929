"""Depth-sort stress (diagnostic runner): the frame depth sort alone
(lodge_debug_depth_sort) on several contexts and streams at once, each
result checked against torch's stable sort of the same keys
(np.lexsort((index, depth)) for depth keys: sort by key, ties by index).

    python -m tests.stress_sort --streams 4 --n 1600000 --rounds 200 [--noise]

Keys look like a frame's: positive fp64 depths as bit patterns, a fraction
culled (~0, dropped), many exact ties.  --noise adds a stream of unrelated
kernels (matmuls) competing for the SMs.  Prints one JSON line.
"""

from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def make_keys(n, gen, device, culled=0.2):
    import torch
    z = 0.05 + torch.rand(n, generator=gen, device=device, dtype=torch.float64) * 500.0
    # exact ties: a slice of the depths snapped to a coarse grid
    snap = torch.rand(n, generator=gen, device=device) < 0.1
    z = torch.where(snap, torch.round(z * 4) / 4 + 0.05, z)
    k = z.view(torch.int64)
    cull = torch.rand(n, generator=gen, device=device) < culled
    return torch.where(cull, torch.full_like(k, -1), k)


def classify(got, ref, keys, rnd, slot):
    """What a wrong sort looks like: size, permutation or not, key order,
    and where the differing positions lie (5120-element partitions)."""
    import torch
    d = {"round": rnd, "slot": slot, "m": int(got.numel()), "m_ref": int(ref.numel())}
    if got.numel() != ref.numel():
        return d
    diff = torch.nonzero(got != ref).squeeze(1)
    d["n_diff"] = int(diff.numel())
    d["first"] = int(diff[0]) if diff.numel() else -1
    d["last"] = int(diff[-1]) if diff.numel() else -1
    d["parts"] = sorted({int(x) // 5120 for x in diff[:4096].tolist()})[:16]
    d["perm"] = bool(torch.equal(torch.sort(got).values, torch.sort(ref).values))
    valid = (got >= 0) & (got < keys.numel())
    d["in_range"] = bool(valid.all())
    if d["in_range"]:
        kg = keys[got]
        d["key_sorted"] = bool((kg[1:] >= kg[:-1]).all())
        d["keys_equal_ref"] = bool(torch.equal(kg, keys[ref]))
    return d


def run(streams=4, n=1_600_000, rounds=100, noise=False, seed=0):
    import torch

    from paper_2505_23158_b200 import _native as N
    from paper_2505_23158_b200.device import Context

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    ctxs = [Context(dev) for _ in range(streams)]
    sts = [torch.cuda.Stream(dev) for _ in range(streams)]
    lib = N.lib()
    bufs = []
    for _ in range(streams):
        bufs.append({"keys": torch.empty(n, dtype=torch.int64, device=dev),
                     "ko": torch.empty(n, dtype=torch.int64, device=dev),
                     "vo": torch.empty(n, dtype=torch.int32, device=dev),
                     "m": torch.zeros(2, dtype=torch.int32, device=dev)})
    nz = None
    if noise:
        ns = torch.cuda.Stream(dev)
        a = torch.randn(4096, 4096, device=dev, dtype=torch.bfloat16)
    bad = 0
    frames = 0
    details = []
    faults = {}
    t0 = time.time()
    for r in range(rounds):
        for q in range(streams):
            bufs[q]["keys"].copy_(make_keys(n, gen, dev))
        torch.cuda.synchronize()
        if noise:
            with torch.cuda.stream(ns):
                for _ in range(24):
                    a = (a @ a).clamp_(-1, 1)
        for q in range(streams):
            b = bufs[q]
            with torch.cuda.stream(sts[q]):
                p = ctxs[q].bind("fast")
                N.check(lib.lodge_debug_depth_sort(p, C.c_void_p(b["keys"].data_ptr()), n,
                                                   C.c_void_p(b["ko"].data_ptr()),
                                                   C.c_void_p(b["vo"].data_ptr()),
                                                   C.c_void_p(b["m"].data_ptr())),
                        "lodge_debug_depth_sort")
        torch.cuda.synchronize()
        for q in range(streams):
            b = bufs[q]
            keys = b["keys"]
            keep = keys != -1
            idx = torch.nonzero(keep).squeeze(1)
            kk = keys[idx]
            # unsigned order of the bit patterns = order of the positive depths
            _, order = torch.sort(kk, stable=True)
            ref = idx[order].to(torch.int32)
            m, fault = (int(x) for x in b["m"].cpu().tolist())
            frames += 1
            if fault:
                faults[fault] = faults.get(fault, 0) + 1
            if m != ref.numel() or not torch.equal(b["vo"][:m], ref):
                bad += 1
                if len(details) < 8:
                    det = classify(b["vo"][:m].long(), ref.long(), keys, r, q)
                    details.append(det)
    return {"streams": streams, "n": n, "sorts": frames, "bad": bad, "noise": noise,
            "details": details, "fault_bits": {hex(k): v for k, v in faults.items()},
            "lib": os.environ.get("LODGE_LIB", "") or "liblodge", "s": round(time.time() - t0, 1)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--streams", type=int, default=4)
    ap.add_argument("--n", type=int, default=1_600_000)
    ap.add_argument("--rounds", type=int, default=100)
    ap.add_argument("--noise", action="store_true")
    ap.add_argument("--seed", type=int, default=0)
    a = ap.parse_args()
    print(json.dumps(run(a.streams, a.n, a.rounds, a.noise, a.seed)), flush=True)
    return 0


if __name__ == "__main__":
    sys.exit(main())
