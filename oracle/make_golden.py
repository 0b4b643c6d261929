"""Generate golden vectors by running the REFERENCE in place (this container only).

    PYTHONDONTWRITEBYTECODE=1 python oracle/make_golden.py

Imports `splatlod` from /root/reference/pkg/src (read-only) and writes
tests/golden/*.npz.  The per-tile member lists are internal to
`splatlod.raster.rasterize` (src/raster.py:421-438); they are captured by
wrapping `splatlod.raster._composite_tile`, which rasterize looks up in its
module globals for every tile (src/raster.py:430).

Files:
  cases.npz    small projection/raster cases mirroring tests/test_raster.py
               (random_scene, face_on_camera, SH degrees 0..3, culling, empty,
               modulation, alpha_min=0, dilation 0, odd resolutions).
  config1.npz  BASELINE config 1 (SURVEY.md 8d recipe): deep_street 10k,
               2 LOD levels, 4 chunks, 8 views at 128x128, stateless blend.
  importance / asset / thresholds / modes / street .npz: see each make_*.

    python oracle/make_golden.py street      # regenerate one file
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")
sys.path.insert(0, REF)

import splatlod.raster as R  # noqa: E402
from splatlod.blending import blend_factor, compose_active, nearest_two_chunks  # noqa: E402
from splatlod.chunks import (ChunkBuildConfig, build_chunk_active_sets, chunk_radii,  # noqa: E402
                             kmeans_positions, visibility_filter_chunk)
from splatlod.lod import (LodBuildConfig, build_levels, mean_focal,  # noqa: E402
                          project_selection)
from splatlod.scene import Camera, ChunkPlan, LodLevel, Scene  # noqa: E402
from splatlod.synthetic import deep_street, face_on_camera, random_scene  # noqa: E402
from splatlod.thresholds import default_grid, greedy_search  # noqa: E402

_captured = []
_orig_composite = R._composite_tile


def _capture(tile_x, tile_y, members, *args, **kw):
    _captured.append((tile_x, tile_y, np.array(members)))
    return _orig_composite(tile_x, tile_y, members, *args, **kw)


R._composite_tile = _capture


def rasterize_with_lists(batch, cam, cfg, need_image=True, record_max_weight=True):
    """Run the reference rasterize and return its output plus its per-tile
    lists as (tile_offsets (T+1), tile_src (P)) in tile-major order."""
    _captured.clear()
    out = R.rasterize(batch, cam, cfg, need_image=need_image, record_max_weight=record_max_weight)
    w, h = cam.resolution
    tx, ty = -(-w // 16), -(-h // 16)
    T = tx * ty
    lists = [np.zeros(0, np.int64)] * T
    if len(batch):
        order = np.lexsort((batch.source_index, batch.depth))
        src_sorted = batch.source_index[order]
        for (x, y, members) in _captured:
            lists[y * tx + x] = src_sorted[members]
    offs = np.zeros(T + 1, np.int64)
    offs[1:] = np.cumsum([len(l) for l in lists])
    tile_src = np.concatenate(lists) if offs[-1] else np.zeros(0, np.int64)
    return out, offs, tile_src


def cam_arrays(cam: Camera, prefix: str, d: dict):
    d[prefix + "R"] = cam.rotation_matrix
    d[prefix + "pos"] = cam.position
    d[prefix + "focal"] = cam.focal
    d[prefix + "pp"] = cam.principal_point
    d[prefix + "res"] = np.array(cam.resolution, np.int64)
    d[prefix + "near"] = np.array(cam.near_plane)
    d[prefix + "quat"] = cam.orientation


def scene_arrays(scene: Scene, prefix: str, d: dict):
    d[prefix + "means"] = scene.means
    d[prefix + "scales"] = scene.scales
    d[prefix + "rotations"] = scene.rotations
    d[prefix + "opacities"] = scene.opacities
    d[prefix + "sh"] = scene.sh_coeffs
    d[prefix + "fv"] = scene.filter_variance
    d[prefix + "deg"] = np.array(scene.sh_degree)


def batch_arrays(b, prefix, d):
    d[prefix + "n_inputs"] = np.array(b.n_inputs)
    d[prefix + "src"] = b.source_index
    d[prefix + "mean2d"] = b.mean2d
    d[prefix + "cov2d"] = b.cov2d
    d[prefix + "conic"] = b.conic
    d[prefix + "extent"] = b.extent
    d[prefix + "depth"] = b.depth
    d[prefix + "opacity"] = b.opacity_eff
    d[prefix + "color"] = b.color


def out_arrays(out, offs, tile_src, prefix, d):
    if out.image is not None:
        d[prefix + "image"] = out.image
    d[prefix + "tile_count"] = out.per_tile_count
    d[prefix + "visible"] = out.per_pixel_visible
    if out.per_gaussian_max_weight is not None:
        d[prefix + "maxw"] = out.per_gaussian_max_weight
    d[prefix + "tile_offsets"] = offs
    d[prefix + "tile_src"] = tile_src


def cfg_arrays(cfg, prefix, d):
    d[prefix + "cfg"] = np.array([cfg.alpha_clamp, cfg.alpha_min, cfg.t_min, cfg.dilation2d])


def make_cases():
    d = {}
    cases = []
    face = face_on_camera()
    # (name, scene, camera, cfg, indices, modulation)
    for seed in range(3):
        cases.append((f"rand{seed}_amin0", random_scene(seed, 300), face,
                      R.RasterConfig(alpha_min=0.0), None, None))
    cases.append(("rand21_default", random_scene(21, 400), face, R.RasterConfig(), None, None))
    cases.append(("rand6_behind", random_scene(6, 200, box_min=(-3, -3, -6), box_max=(3, 3, 12)),
                  face, R.RasterConfig(), None, None))
    cases.append(("rand5_nodil", random_scene(5, 400), face, R.RasterConfig(dilation2d=0.0),
                  None, None))
    for deg in (0, 2, 3):
        cases.append((f"sh{deg}", random_scene(30 + deg, 350, sh_degree=deg), face,
                      R.RasterConfig(), None, None))
    sc = random_scene(40, 900, box_min=(-3, -3, -2), box_max=(3, 3, 12))
    rng = np.random.default_rng(3)
    idx = np.sort(rng.choice(900, 500, replace=False))
    cases.append(("subset_mod", sc, face, R.RasterConfig(), idx, rng.uniform(0, 1, 500)))
    cases.append(("empty", Scene.empty(1), face, R.RasterConfig(), None, None))
    far = random_scene(41, 50, box_min=(100, 100, 2), box_max=(120, 120, 12))
    cases.append(("all_culled", far, face, R.RasterConfig(), None, None))
    odd = Camera((0.0, 0.0, 0.0), (1.0, 0.0, 0.0, 0.0), (60.0, 55.0), (50.0, 35.0), (100, 70),
                 near_plane=0.05)
    cases.append(("odd_res", random_scene(42, 700), odd, R.RasterConfig(), None, None))
    yaw = Camera((0.3, -0.2, -1.0), (0.9659258262890683, 0.0, 0.25881904510252074, 0.0),
                 (48.0, 48.0), (40.0, 32.0), (80, 64), near_plane=0.05)
    cases.append(("yawed", random_scene(43, 800, box_min=(-6, -3, -2), box_max=(6, 3, 12)), yaw,
                  R.RasterConfig(), None, None))
    big = random_scene(44, 60, box_min=(-1, -1, 3), box_max=(1, 1, 4))
    big = Scene(big.means, big.scales * 4.0, big.rotations, big.opacities, big.sh_coeffs,
                np.full(60, 0.05), 1)
    cases.append(("huge_filtered", big, face, R.RasterConfig(), None, None))
    names = []
    for (name, scene, cam, cfg, idx, mod) in cases:
        p = name + "/"
        names.append(name)
        scene_arrays(scene, p, d)
        cam_arrays(cam, p, d)
        cfg_arrays(cfg, p, d)
        if idx is not None:
            d[p + "idx"] = np.asarray(idx, np.int64)
        if mod is not None:
            d[p + "mod"] = np.asarray(mod, np.float64)
        b = R.project_scene(scene, cam, cfg, indices=idx, modulation=mod)
        batch_arrays(b, p + "b_", d)
        out, offs, tsrc = rasterize_with_lists(b, cam, cfg)
        out_arrays(out, offs, tsrc, p + "o_", d)
    d["names"] = np.array(names)
    return d


def make_config1():
    t0 = time.time()
    scene, cams = deep_street(seed=7, n_fine=4380, n_views=8, resolution=(128, 128),
                              focal=104.0, length=200.0)
    assert len(scene) == 10000, len(scene)
    cfg = LodBuildConfig(importance_views=tuple(cams), reference_focal=mean_focal(cams))
    base = LodLevel.base(scene)
    grid = list(default_grid(base, cams, 12))
    accepted, _ = greedy_search(base, cams, cfg, grid, max_levels=1)
    levels, _ = build_levels(scene, accepted, cfg)
    positions = np.stack([c.position for c in cams])
    centers, assign = kmeans_positions(positions, 4, seed=0)
    radii = chunk_radii(centers, positions)
    plan = build_chunk_active_sets(levels, centers, radii, assign)
    ccfg = ChunkBuildConfig(d1=accepted[0], kmeans_seed=0, perturb_count=4, perturb_seed=0,
                            vis_threshold=cfg.gamma)
    filtered = []
    for j in range(plan.n_chunks):
        cams_j = [cams[i] for i in np.flatnonzero(assign == j)]
        filtered.append(visibility_filter_chunk(plan, j, levels, cams_j, ccfg, cfg.raster))
    plan = ChunkPlan(centers, radii, tuple(filtered), assign)
    print("config1 build", round(time.time() - t0, 1), "s; d1", accepted,
          "levels", [len(l) for l in levels],
          "sets", [[len(s) for s in ch] for ch in plan.active_sets])
    d = {"thresholds": np.array(accepted, np.float64)}
    for l, lv in enumerate(levels):
        scene_arrays(lv.scene, f"L{l}/", d)
        d[f"L{l}/depth_threshold"] = np.array(lv.depth_threshold)
    d["n_levels"] = np.array(len(levels))
    d["centers"] = plan.centers
    d["radii"] = plan.radii
    for j in range(plan.n_chunks):
        for l in range(plan.n_levels):
            d[f"set/{j}/{l}"] = plan.active_sets[j][l]
    rc = R.RasterConfig()
    cfg_arrays(rc, "", d)
    for v, cam in enumerate(cams):
        p = f"v{v}/"
        cam_arrays(cam, p, d)
        f, o = nearest_two_chunks(plan, cam.position)
        t_bar, t = blend_factor(cam.position, plan.centers[f], plan.centers[o])
        d[p + "pair"] = np.array([f, o])
        d[p + "t"] = np.array([t_bar, t])
        sel = compose_active(plan, levels, f, o, t)
        for l in range(len(levels)):
            d[p + f"sel{l}"] = sel.sets[l]
            d[p + f"mod{l}"] = sel.modulations[l]
        batch = project_selection(levels, sel.sets, cam, rc, modulations=sel.modulations)
        batch_arrays(batch, p + "b_", d)
        out, offs, tsrc = rasterize_with_lists(batch, cam, rc)
        out_arrays(out, offs, tsrc, p + "o_", d)
    return d


def _config1_objects():
    """Reference objects rebuilt from the committed config1.npz."""
    d = np.load(os.path.join(OUT, "config1.npz"))
    levels = []
    for l in range(int(d["n_levels"])):
        p = f"L{l}/"
        sc = Scene(d[p + "means"], d[p + "scales"], d[p + "rotations"], d[p + "opacities"],
                   d[p + "sh"], d[p + "fv"], int(d[p + "deg"]))
        levels.append(LodLevel(l, float(d[p + "depth_threshold"]), sc,
                               np.arange(len(sc), dtype=np.int64)))
    cams = []
    for v in range(8):
        p = f"v{v}/"
        cams.append(Camera(d[p + "pos"], d[p + "quat"], d[p + "focal"], d[p + "pp"],
                           tuple(int(x) for x in d[p + "res"]), float(d[p + "near"]), f"v{v}"))
    K, L = d["centers"].shape[0], int(d["n_levels"])
    sets = tuple(tuple(d[f"set/{j}/{l}"] for l in range(L)) for j in range(K))
    plan = ChunkPlan(d["centers"], d["radii"], sets, np.zeros(0, np.int64))
    return d, levels, cams, plan


def make_importance():
    """Importance scoring on the config-1 data:
    a  compute_importance(level 0, views 0-3, PerturbSpec(2, 5))
    b  score_active_selection(both levels, chunk 2's sets, views 4-5, PerturbSpec(1, 9))
    c  visibility_filter_chunk(chunk 0, views 0-1, perturb_count 2, seed 3)"""
    from splatlod.lod import PerturbSpec, compute_importance, score_active_selection
    d, levels, cams, plan = _config1_objects()
    rc = R.RasterConfig()
    out = {}
    t0 = time.time()
    cfg = LodBuildConfig()
    imp = compute_importance(levels[0], cams[0:4], cfg, PerturbSpec(2, 5))
    out["a/scores"] = imp.scores
    out["a/gamma"] = np.array(imp.threshold_base)
    sc = score_active_selection(levels, plan.active_sets[2], cams[4:6], rc, PerturbSpec(1, 9))
    for l, s in enumerate(sc):
        out[f"b/scores{l}"] = s
    ccfg = ChunkBuildConfig(d1=float(d["thresholds"][0]), perturb_count=2, perturb_seed=3,
                            vis_threshold=cfg.gamma)
    kept = visibility_filter_chunk(plan, 0, levels, cams[0:2], ccfg, rc)
    for l, s in enumerate(kept):
        out[f"c/kept{l}"] = np.asarray(s, np.int64)
    out["c/vis_threshold"] = np.array(ccfg.vis_threshold)
    print("importance", round(time.time() - t0, 1), "s; a", int((imp.scores > 0).sum()),
          "b", [int((s > 0).sum()) for s in sc], "c", [len(s) for s in kept])
    return out


ASSET_CORRUPTIONS = [
    # (name, kind, args) applied by tests/asset_util.py corrupt(); the
    # reference's read_asset message for each is recorded below
    ("nan_mean", "f32", ("L0", 5, 0, "nan")),
    ("neg_scale", "f32", ("L0", 7, 4, -0.5)),
    ("opacity_gt1", "f32", ("L1", 3, 10, 1.5)),
    ("neg_fv", "f32", ("L1", 0, 11, -1.0)),
    ("bad_rot", "f32", ("L0", 11, 6, 3.0)),
    ("nan_sh", "f32", ("L1", 9, 13, "inf")),
    ("unsorted_set", "u32swap", (1, 0, 2)),
    ("set_oob", "u32set", (2, 1, -1, 4076)),
    ("bad_version", "manifest", ("format_version", 2)),
    ("bad_degree", "manifest", ("sh_degree", 5)),
    ("count_mismatch", "level_field", (1, "gaussian_count", 4075)),
    ("prov_mismatch", "level_field", (0, "provenance_length", 4)),
    ("range_overflow", "level_field", (1, "length", 10 ** 9)),
    ("set_count", "set_field", (3, 1, "count", 1)),
    ("missing_sets", "drop_set", (2,)),
    ("bad_magic", "container_magic", ()),
    ("bad_container_version", "container_version", (9,)),
    ("short_container", "container_truncate", (10,)),
    ("bad_json", "manifest_bytes", (b"{not json",)),
]


def make_asset():
    """config-1 levels + plan written by the reference's write_asset
    (directory and container), read_asset's error message for each entry of
    ASSET_CORRUPTIONS, and two views rendered from the reference's
    read_asset result (the asset stores fp32 and normalises rotations)."""
    import json
    import shutil
    import splatlod.assets as A
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))
    import asset_util as AU
    d, levels, cams, plan = _config1_objects()
    plan = ChunkPlan(plan.centers, plan.radii, plan.active_sets,
                     np.array([0, 0, 1, 1, 2, 2, 3, 3], np.int64))
    adir = os.path.join(OUT, "asset_c1")
    shutil.rmtree(adir, ignore_errors=True)
    A.write_asset(adir, levels, plan, sh_degree=int(levels[0].scene.sh_degree),
                  reference_focal=104.0, filter_scale=1.0, gamma=LodBuildConfig().gamma,
                  seeds={"golden": 7}, config_hash="golden")
    msgs = {}
    tmp = os.path.join("/tmp", "lodge_asset_corrupt")
    for name, kind, args in ASSET_CORRUPTIONS:
        shutil.rmtree(tmp, ignore_errors=True)
        path = AU.corrupt(adir, tmp, kind, args)
        try:
            A.read_asset(path)
            msgs[name] = ""
        except A.AssetError as e:
            msgs[name] = str(e).replace(str(path), "<path>")
    out = {"messages": np.array(json.dumps(msgs))}
    asset = A.read_asset(adir)
    rc = R.RasterConfig()
    for v in (1, 6):
        cam = cams[v]
        p = f"v{v}/"
        f, o = nearest_two_chunks(asset.plan, cam.position)
        t_bar, t = blend_factor(cam.position, asset.plan.centers[f], asset.plan.centers[o])
        out[p + "pair"] = np.array([f, o])
        out[p + "t"] = np.array([t_bar, t])
        sel = compose_active(asset.plan, asset.levels, f, o, t)
        batch = project_selection(asset.levels, sel.sets, cam, rc, modulations=sel.modulations)
        res = R.rasterize(batch, cam, rc)
        out[p + "image"] = res.image
        out[p + "tile_count"] = res.per_tile_count
        out[p + "visible"] = res.per_pixel_visible
        out[p + "maxw"] = res.per_gaussian_max_weight
        out[p + "src"] = batch.source_index
        out[p + "depth"] = batch.depth
    for l, lv in enumerate(asset.levels):
        out[f"L{l}/rotations"] = lv.scene.rotations
        out[f"L{l}/provenance"] = lv.provenance
    print("asset", {k: v[:40] for k, v in msgs.items()})
    return out


def make_thresholds():
    """Threshold-search cost tables on config-1 data:
    the reference ThresholdSearcher over views 0-3 with the config-1 build
    config; _table for the base level and for provisional levels at d1 and
    2.5 d1 (built by the reference, stored so the tests need no LOD build),
    and evaluate() of [d1] and [d1, 2.5 d1]."""
    from splatlod.thresholds import ThresholdSearcher
    d, levels, cams, plan = _config1_objects()
    base = LodLevel.base(levels[0].scene)
    cfg = LodBuildConfig(importance_views=tuple(cams), reference_focal=mean_focal(cams))
    views = cams[0:4]
    s = ThresholdSearcher(base, views, cfg)
    d1 = float(d["thresholds"][0])
    depths = [0.0, d1, 2.5 * d1]
    out = {"depths": np.array(depths)}
    t0 = time.time()
    for k, dep in enumerate(depths):
        lv = s.provisional_level(dep)
        if k:
            scene_arrays(lv.scene, f"P{k}/", out)
            out[f"P{k}/provenance"] = lv.provenance
        for vi in range(len(views)):
            dist, prefix = s._table(dep, vi)
            out[f"T{k}/{vi}/dist"] = dist
            out[f"T{k}/{vi}/prefix"] = prefix
    for name, ths in (("e1", [d1]), ("e2", [d1, 2.5 * d1])):
        ev = s.evaluate(ths)
        out[name + "/thresholds"] = np.array(ev.thresholds)
        out[name + "/mean"] = np.array(ev.mean_gaussians_per_tile)
        out[name + "/per_view"] = np.array(ev.per_view_cost)
        out[name + "/build"] = np.array(ev.build_cost_proxy)
    print("thresholds", round(time.time() - t0, 1), "s; levels",
          [len(s.provisional_level(x)) for x in depths],
          "mean cost", float(out["e1/mean"]), float(out["e2/mean"]))
    return out


def make_modes():
    """LOD-mode and full-mode frames on config-1 data:
    render_lod (src/lod.py:230-237) for views 1 and 5, with and without depth
    offsets, and the CLI's full mode (src/cli.py:221-226 + :236-243)."""
    from splatlod.lod import render_lod, select_active
    d, levels, cams, plan = _config1_objects()
    rc = R.RasterConfig()
    out = {}
    t0 = time.time()
    for v in (1, 5):
        cam = cams[v]
        for tag, offs in (("lod", None), ("lodoff", [0.0, 1.5])):
            res = render_lod(levels, cam, rc, depth_offsets=offs)
            p = f"v{v}/{tag}/"
            out[p + "image"] = res.image
            out[p + "tile_count"] = res.per_tile_count
            out[p + "visible"] = res.per_pixel_visible
            out[p + "maxw"] = res.per_gaussian_max_weight
            for l, s in enumerate(select_active(levels, cam.position, offs)):
                out[p + f"set{l}"] = s
        sets = [np.arange(len(levels[0]), dtype=np.int64)]
        sets += [np.zeros(0, dtype=np.int64) for _ in levels[1:]]
        mods = [np.ones(len(s)) for s in sets]
        batch = project_selection(levels, sets, cam, rc, modulations=mods)
        res = R.rasterize(batch, cam, rc)
        p = f"v{v}/full/"
        out[p + "image"] = res.image
        out[p + "tile_count"] = res.per_tile_count
        out[p + "visible"] = res.per_pixel_visible
        out[p + "maxw"] = res.per_gaussian_max_weight
    print("modes", round(time.time() - t0, 1), "s")
    return out


def make_street():
    """Residency streaming and blend renders (src/blending.py:140-203) on the
    reference's own street_runtime fixture (tests/test_blending.py:21-33):
    deep_street(6, 1500 fine, 8 views, 80x64, f 70, length 70), one built
    level at 9.0 (single round), three chunk centres on the corridor axis.
    Records the stream_step walk z = 8..44 (400 steps, every state and
    event), a teleport, and render_blend_state frames at six walk positions,
    plus the swap-instant and t = 1 renders of TestSwapConsistency."""
    from splatlod.blending import render_blend_state, render_selection, stream_step
    t0 = time.time()
    scene, cams = deep_street(seed=6, n_fine=1500, n_views=8, resolution=(80, 64),
                              focal=70.0, length=70.0)
    cfg = LodBuildConfig(importance_views=tuple(cams), reference_focal=70.0)
    levels, _ = build_levels(scene, [9.0], cfg, single_round=True)
    positions = np.stack([c.position for c in cams])
    centers = np.array([[0.0, 0.5, 12.0], [0.0, 0.5, 28.0], [0.0, 0.5, 44.0]])
    radii = chunk_radii(centers, positions)
    plan = build_chunk_active_sets(levels, centers, radii)
    d = {"n_levels": np.array(len(levels)), "centers": plan.centers, "radii": plan.radii}
    for l, lv in enumerate(levels):
        scene_arrays(lv.scene, f"L{l}/", d)
        d[f"L{l}/depth_threshold"] = np.array(lv.depth_threshold)
    for j in range(plan.n_chunks):
        for l in range(plan.n_levels):
            d[f"set/{j}/{l}"] = plan.active_sets[j][l]
    for v, cam in enumerate(cams):
        cam_arrays(cam, f"v{v}/", d)
    rc = R.RasterConfig()
    kinds = {"load": 0, "unload": 1, "swap_primary": 2}

    def walk(tag, zs, render_at=()):
        state, ev, st = None, [], []
        for i, z in enumerate(zs):
            pos = np.array([0.0, 0.5, z])
            state, events = stream_step(state, plan, pos)
            ev += [(i, kinds[e.kind], e.chunk_id) + tuple(e.camera_position) for e in events]
            lc = state.loaded_chunks + (-1,) * (2 - len(state.loaded_chunks))
            st.append(lc + (state.primary_id, state.t_bar, state.t))
            if i in render_at:
                cam = cams[0]
                view = Camera(pos, cam.orientation, cam.focal, cam.principal_point,
                              cam.resolution, cam.near_plane)
                out = render_blend_state(state, plan, levels, view, rc)
                p = f"{tag}/r{i}/"
                d[p + "image"] = out.image
                d[p + "tile_count"] = out.per_tile_count
                d[p + "visible"] = out.per_pixel_visible
                d[p + "maxw"] = out.per_gaussian_max_weight
        d[tag + "/zs"] = np.asarray(zs, np.float64)
        d[tag + "/events"] = np.array(ev, np.float64).reshape(-1, 6)
        d[tag + "/states"] = np.array(st, np.float64)

    walk("walk", np.linspace(8.0, 44.0, 400), render_at=(0, 90, 170, 200, 260, 399))
    walk("teleport", np.array([10.0, 60.0]))
    # swap instant (tests/test_blending.py:201-215) and t = 1 (:108-115)
    cam = cams[0]
    swap_pos = plan.centers[1]
    view = Camera(swap_pos, cam.orientation, cam.focal, cam.principal_point, cam.resolution,
                  cam.near_plane)
    for tag, o in (("swap_old", 0), ("swap_new", 2)):
        t = blend_factor(swap_pos, plan.centers[1], plan.centers[o])[1]
        d[tag + "/t"] = np.array(t)
        d[tag + "/image"] = render_selection(levels, compose_active(plan, levels, 1, o, t),
                                             view, rc).image
    d["t_one/image"] = render_selection(levels, compose_active(plan, levels, 0, 1, 1.0),
                                        cams[2], rc).image
    print("street", round(time.time() - t0, 1), "s; levels", [len(l) for l in levels],
          "sets", [[len(s) for s in ch] for ch in plan.active_sets],
          "events", d["walk/events"].shape[0])
    return d


REPORT_EDGES = {"default": [0, 1, 2, 4, 8, 16, 32, 64, 128, 256], "coarse": [1, 3, 5],
                "fractional": [2.5, 7.5, 100.0], "wide": [-5.0, 0.0, 1e6],
                "fine": list(range(0, 64, 3))}


def make_report():
    """The reference bench's per-frame report fields (src/cli.py:283-320) on
    the config-1 frames the reference rendered (config1.npz o_* outputs):
    visibility_histogram for several edge sets (src/raster.py:464-479),
    mean_per_tile and visible_gaussians, plus the edge-validation messages."""
    from types import SimpleNamespace
    c1 = np.load(os.path.join(OUT, "config1.npz"))
    d = {}
    for v in range(8):
        p = f"v{v}/"
        out = SimpleNamespace(per_pixel_visible=c1[p + "o_visible"])
        for name, edges in REPORT_EDGES.items():
            d[p + "hist/" + name] = R.visibility_histogram(out, np.asarray(edges))
        d[p + "mean_per_tile"] = np.float64(c1[p + "o_tile_count"].mean())
        d[p + "visible_gaussians"] = np.int64(np.count_nonzero(c1[p + "o_maxw"]))
    for name, edges in REPORT_EDGES.items():
        d["edges/" + name] = np.asarray(edges, np.float64)
    msgs = []
    for bad in ([1.0], [3.0, 2.0], [0.0, 1.0, 1.0]):
        try:
            R.visibility_histogram(SimpleNamespace(per_pixel_visible=np.zeros(4, np.int64)),
                                   np.asarray(bad))
            msgs.append("")
        except ValueError as e:
            msgs.append(str(e))
    d["bad_edges_messages"] = np.asarray(msgs)
    return d


GENERATORS = {"cases": make_cases, "config1": make_config1, "importance": make_importance,
              "asset": make_asset, "thresholds": make_thresholds, "modes": make_modes,
              "street": make_street, "report": make_report}


def main(names=None):
    """Regenerate the named golden files (default: all); config1 must exist
    (or be generated first) for the generators that reuse its objects."""
    os.makedirs(OUT, exist_ok=True)
    for name in names or list(GENERATORS):
        t0 = time.time()
        np.savez_compressed(os.path.join(OUT, name + ".npz"), **GENERATORS[name]())
        print(name, round(time.time() - t0, 1), "s")
    for f in sorted(os.listdir(OUT)):
        print(f, os.path.getsize(os.path.join(OUT, f)) // 1024, "KiB")


if __name__ == "__main__":
    main(sys.argv[1:])
