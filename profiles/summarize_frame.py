"""Map one frame's `ncu --set full` launches (profiles/profile_frames.py
--frames 1, every kernel captured) to bench.py's stages and write
profiles/traffic.json (DRAM read+write bytes per stage per frame -- the
`roofline.traffic` the bench line cites) plus a per-kernel table.

    python profiles/summarize_frame.py gpurun_out/p3_full.ncu-rep \\
        --traffic profiles/traffic.json --table profiles/r02_ncu_frame.md

Stages follow the frame's launch order (csrc/lodge_api.cu render_tail): the
first pair of k_onesweep tile passes belongs to the first depth phase
("tile_sort"), the second pair to the second phase ("second_phase").
"""

from __future__ import annotations

import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from summarize_ncu import launches  # noqa: E402

STAGE_OF = [
    ("k_begin_frame", "select"), ("k_select_frame", "select"),
    ("k_sel_hist", "depth_sort"), ("k_sel_scan", "depth_sort"), ("k_sel_compact", "depth_sort"),
    ("k_owner_filter", "second_phase"),
    ("k_union_check", "union"), ("k_union_split", "union"), ("k_union_merge", "union"),
    ("k_union_sizes", "union"),
    ("k_project_frame", "project"),
    ("k_dup_count<0>", "tile_setup"), ("k_payload", "tile_setup"), ("k_tile_setup", "tile_setup"),
    ("k_dup_emit", "duplicate"),
    ("k_block_lists<1>", "tile_sort"),
    ("k_block_lists<2>", "second_phase"),
    ("k_composite<0, 3, 1>", "composite"),
    ("k_setup_b", "second_phase"), ("k_dup_count<1>", "second_phase"),
    ("k_emit_b", "second_phase"),
    ("k_composite<0, 3, 2>", "composite_b"),
]


SORT_KERNELS = ("k_depth_hist", "k_depth_scan", "k_depth_pass", "k_depth_ties")


def stage_of(name, state):
    # two-phase frames sort twice: the first-phase candidates (depth_sort)
    # and, after k_owner_filter, the second-phase owners (second_phase)
    if any(k in name for k in SORT_KERNELS):
        return "second_phase" if state.get("owners") else "depth_sort"
    if "k_owner_filter" in name:
        state["owners"] = True
    if "k_onesweep" in name:
        state["tile_passes"] += 1
        return "tile_sort" if state["tile_passes"] <= 2 else "second_phase"
    if "k_payload" in name:
        state["payloads"] += 1
        return "tile_setup" if state["payloads"] == 1 else "second_phase"
    for key, st in STAGE_OF:
        if key in name:
            return st
    return "other"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("--traffic")
    ap.add_argument("--table")
    a = ap.parse_args()
    ls = launches(a.rep)
    state = {"tile_passes": 0, "payloads": 0, "owners": False}
    per = {}
    rows = []
    for l in ls:
        st = stage_of(l["kernel"], state)
        t = float(l["gpu__time_duration.sum"].split()[0].replace(",", ""))
        unit = l["gpu__time_duration.sum"].split()[1] if " " in l["gpu__time_duration.sum"] else "us"
        us = t / 1000.0 if unit in ("ns", "nsecond") else (t * 1000.0 if unit in ("ms", "msecond") else t)
        d = per.setdefault(st, {"dram_bytes": 0.0, "us": 0.0, "kernels": []})
        d["dram_bytes"] += l["dram_bytes"]
        d["us"] += us
        d["kernels"].append(l["kernel"].replace("void ", ""))
        rows.append((st, l["kernel"].replace("void ", ""), us, l["dram_bytes"],
                     l.get("sm__warps_active.avg.pct_of_peak_sustained_active", ""),
                     l.get("smsp__issue_active.avg.pct_of_peak_sustained_active", ""),
                     l["stalls"]))
    src = (f"ncu --set full --clock-control none, config 3, one frame of the bench's timed "
           f"views ({os.path.basename(a.rep)}, profiles/profile_frames.py --frames 1)")
    if a.traffic:
        out = {st: {"dram_bytes_per_launch": round(d["dram_bytes"]),
                    "kernel": " + ".join(d["kernels"]), "ncu_us": round(d["us"], 1),
                    "source": src} for st, d in per.items()}
        json.dump(out, open(a.traffic, "w"), indent=1)
    if a.table:
        lines = [f"# One config-3 frame under ncu --set full ({os.path.basename(a.rep)})", "",
                 "Cold-cache, serialised replays: compare shares, not absolutes, with the "
                 "bench's stage events.", "",
                 "| stage | kernel | us | DRAM MB | warps active | issue active | top stalls |",
                 "|---|---|---|---|---|---|---|"]
        for st, k, us, b, wa, ia, stl in rows:
            top = ", ".join(f"{n} {v}%" for n, v in list(stl.items())[:3])
            lines.append(f"| {st} | `{k[:60]}` | {us:.1f} | {b / 1e6:.1f} | {wa.split()[0][:5]} | "
                         f"{ia.split()[0][:5]} | {top} |")
        lines += ["", "| stage | ncu us | DRAM MB |", "|---|---|---|"]
        for st, d in per.items():
            lines.append(f"| {st} | {d['us']:.1f} | {d['dram_bytes'] / 1e6:.1f} |")
        open(a.table, "w").write("\n".join(lines) + "\n")
    print(json.dumps({st: (round(d["us"], 1), round(d["dram_bytes"] / 1e6, 1))
                      for st, d in per.items()}))


if __name__ == "__main__":
    main()
