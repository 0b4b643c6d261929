"""Loaders for the committed golden vectors (tests/golden/, made by
oracle/make_golden.py from the reference itself)."""

import os
from types import SimpleNamespace

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def scene(d, p):
    return SimpleNamespace(means=d[p + "means"], scales=d[p + "scales"],
                           rotations=d[p + "rotations"], opacities=d[p + "opacities"],
                           sh_coeffs=d[p + "sh"], filter_variance=d[p + "fv"],
                           sh_degree=int(d[p + "deg"]))


def camera(d, p):
    return SimpleNamespace(rotation_matrix=d[p + "R"], position=d[p + "pos"],
                           focal=d[p + "focal"], principal_point=d[p + "pp"],
                           resolution=tuple(int(v) for v in d[p + "res"]),
                           near_plane=float(d[p + "near"]), orientation=d[p + "quat"])


def cfg(d, p):
    a = d[p + "cfg"]
    return SimpleNamespace(alpha_clamp=float(a[0]), alpha_min=float(a[1]), t_min=float(a[2]),
                           dilation2d=float(a[3]), threads=1)


def batch(d, p):
    return {"src": d[p + "src"], "mean2d": d[p + "mean2d"], "cov2d": d[p + "cov2d"],
            "conic": d[p + "conic"], "extent": d[p + "extent"], "depth": d[p + "depth"],
            "opacity": d[p + "opacity"], "color": d[p + "color"],
            "n_inputs": int(d[p + "n_inputs"])}


def config1_levels(d):
    return [scene(d, f"L{l}/") for l in range(int(d["n_levels"]))]


def config1_sets(d):
    K = d["centers"].shape[0]
    L = int(d["n_levels"])
    return [[d[f"set/{j}/{l}"] for l in range(L)] for j in range(K)]
