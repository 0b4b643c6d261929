"""B200-native LODGE (arXiv 2505.23158) per-frame renderer.

Drop-in for the reference `splatlod` render / chunk-selection API
(reference src/__init__.py:3-21): the same names and signatures, computed by
hand-written sm_100a kernels in liblodge.so (C ABI: include/lodge.h).
There is no CPU fallback; importing works without a GPU, calling does not.
"""

from .types import (ActiveSelection, BlendState, Camera, ChunkPlan, Gaussian, LodLevel,
                    RasterConfig, Scene, Splat2D, Splat2DBatch, StreamEvent, TileRenderOutput,
                    quat_to_matrix)
from .raster import (project_gaussian, project_scene, rasterize, render_scene,
                     tile_cover_counts, visibility_histogram)
from .lod import (build_chunk_active_sets, lod_bounds, project_selection, render_full,
                  render_lod, select_active)
from .blending import (blend_factor, compose_active, nearest_two_chunks, render_blend_state,
                       render_selection, stream_step)
from .renderer import Frame, Renderer
from .device import default_precision, set_default_precision
from .types import ImportanceScores, PerturbSpec
from .importance import (compute_importance, random_rotations, score_active_selection,
                         visibility_filter_chunk)
from .asset import AssetError, DeviceAsset, load_asset
from .thresholds import CostEvaluation, ThresholdSearcher, cover_table, evaluate_cost
from .streaming import StreamingStore, host_pair

__version__ = "0.1.0"

__all__ = [
    "ActiveSelection", "BlendState", "Camera", "ChunkPlan", "Gaussian", "LodLevel",
    "RasterConfig", "Scene", "Splat2D", "Splat2DBatch", "StreamEvent", "TileRenderOutput",
    "quat_to_matrix", "project_gaussian", "project_scene", "rasterize", "render_scene",
    "tile_cover_counts", "visibility_histogram", "project_selection", "blend_factor",
    "compose_active", "nearest_two_chunks", "render_blend_state", "render_selection",
    "stream_step", "Frame", "Renderer", "default_precision", "set_default_precision",
    "ImportanceScores", "PerturbSpec", "compute_importance", "random_rotations",
    "score_active_selection", "visibility_filter_chunk", "AssetError", "DeviceAsset",
    "load_asset", "CostEvaluation", "ThresholdSearcher", "cover_table", "evaluate_cost",
    "lod_bounds", "render_full", "render_lod", "select_active", "build_chunk_active_sets",
    "StreamingStore", "host_pair",
]
