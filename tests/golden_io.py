"""Loader for tests/golden/*.npz fixtures (made by tests/golden/make_golden.py
from the reference itself)."""
import glob
import json
import os

import numpy as np

from paper_1611_03631_b200._capi import VxgTsdfConfig

GOLDEN_DIR = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def fixtures():
    return sorted(glob.glob(os.path.join(GOLDEN_DIR, "*.npz")))


def load(path):
    z = np.load(path)
    meta = json.loads(bytes(z["meta"]).decode())
    frames = []
    for i in range(meta["frames"]):
        rgb = z[f"rgb{i}"] if f"rgb{i}" in z.files else None
        frames.append((z[f"xyz{i}"], rgb, z[f"pose{i}"]))
    c = meta["config"]
    cfg = VxgTsdfConfig(c["truncation"], c["dropoff_epsilon"], c["max_weight"], c["weight_mode"], c["merge_mode"],
                        c["min_ray_length"], c["max_ray_length"])
    return meta, cfg, frames, bytes(z["vxblx"])


def tsdf_config_from(meta):
    from paper_1611_03631_b200 import MergeMode, TsdfConfig, WeightMode
    c = meta["config"]
    return TsdfConfig(truncation=c["truncation"], dropoff_epsilon=c["dropoff_epsilon"], max_weight=c["max_weight"],
                      weight_mode=WeightMode(c["weight_mode"]), merge_mode=MergeMode(c["merge_mode"]),
                      min_ray_length=c["min_ray_length"], max_ray_length=c["max_ray_length"])
