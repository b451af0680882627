"""Shared helpers for GPU-vs-oracle parity (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle_bindings import OracleLayer, parse_vxblx


def diff_report(gpu_bytes: bytes, ora_bytes: bytes) -> str:
    """Human-readable summary of how two VXBLX streams differ."""
    if gpu_bytes == ora_bytes:
        return "identical"
    try:
        _, _, gi, gv = parse_vxblx(gpu_bytes)
        _, _, oi, ov = parse_vxblx(ora_bytes)
    except Exception as e:  # pragma: no cover
        return f"unparseable: {e}"
    msg = [f"blocks gpu={len(gi)} oracle={len(oi)}"]
    gs = {tuple(x) for x in gi.tolist()}
    os_ = {tuple(x) for x in oi.tolist()}
    if gs != os_:
        msg.append(f"block sets differ: only gpu={len(gs - os_)} only oracle={len(os_ - gs)}")
        return "; ".join(msg)
    d = gv["distance"] != ov["distance"]
    w = gv["weight"] != ov["weight"]
    c = (gv["r"] != ov["r"]) | (gv["g"] != ov["g"]) | (gv["b"] != ov["b"])
    msg.append(f"voxels differing: distance={int(d.sum())} weight={int(w.sum())} color={int(c.sum())}")
    if d.any():
        rel = np.abs(gv["distance"][d] - ov["distance"][d]) / np.maximum(np.abs(ov["distance"][d]), 1e-30)
        msg.append(f"max rel distance diff={float(rel.max()):.3g}")
    return "; ".join(msg)


def run_pair(layer, integrator, cfg, voxel_size, vps, frames, batch=False):
    """Integrates frames [(xyz, rgb, pose)] on the GPU (per frame or as one batch)
    and on the oracle; returns (gpu_stats, oracle_stats, gpu_bytes, oracle_bytes)."""
    from paper_1611_03631_b200 import Scan
    ora = OracleLayer(cfg, voxel_size, vps)
    o_stats = [ora.integrate(x, c, p) for (x, c, p) in frames]
    scans = [Scan(x, c, p) for (x, c, p) in frames]
    if batch:
        g = integrator.integrate_batch(scans)
        g_stats = [tuple(int(v) for v in row) for row in g]
    else:
        g_stats = []
        for s in scans:
            u = integrator.integrate(s)
            g_stats.append((u, integrator.raycasts_last_scan(), integrator.skipped_points_last_scan()))
    return g_stats, o_stats, layer.save_bytes(), ora.save_bytes()
