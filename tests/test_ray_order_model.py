"""CPU: the merged-mode ray-order model used by the GPU
against std::unordered_map itself.

integrate_grouped (tsdf_integrator.cpp:199-223) casts one ray per bucket in
IndexMap iteration order. The GPU reproduces that order without a hash map:
per rehash epoch, sort keys by (first occupation of their bucket desc,
insertion position desc). This test restates that model in Python (the same
rule as k_order_fo/k_order_keys and order_rehash_frame) and checks it against
the oracle's real libstdc++ container, with and without rehashes.
"""
import ctypes

import numpy as np
import pytest

from oracle_bindings import oracle_lib
from paper_1611_03631_b200 import TsdfConfig


def teschner(x, y, z):
    h = ((x * 73856093) ^ (y * 19349669) ^ (z * 83492791)) & 0xFFFFFFFF
    h = h - (1 << 32) if h >= (1 << 31) else h  # int wrap, then sign-extend to size_t
    return h & 0xFFFFFFFFFFFFFFFF


def schedule(n_points, max_keys):
    out = (ctypes.c_uint64 * 128)()
    k = oracle_lib().vxo_bucket_schedule(n_points, max_keys, out, 64)
    return [(int(out[2 * i]), int(out[2 * i + 1])) for i in range(k)]


def model_order(keys, n_points):
    """keys: distinct terminal keys in first-appearance order."""
    K = len(keys)
    h = [teschner(*k) for k in keys]
    sch = schedule(n_points, K)
    order = []
    for e, (t_lo, bc) in enumerate(sch):
        t_hi = sch[e + 1][0] if e + 1 < len(sch) else float("inf")
        if t_lo >= K and e > 0:
            break
        prev = {r: i for i, r in enumerate(order)}
        members = [r for r in range(K) if r < t_hi]
        pos = {r: (prev[r] if r < t_lo else r) for r in members}
        fo = {}
        for r in members:
            b = h[r] % bc
            fo[b] = min(fo.get(b, float("inf")), pos[r])
        members.sort(key=lambda r: (-fo[h[r] % bc], -pos[r]))
        order = members
    return [keys[r] for r in order]


def unordered_map_order(g, v):
    """Terminal keys in IndexMap iteration order, from the oracle (std::unordered_map)."""
    pts = ((g.astype(np.float32) + np.float32(0.5)) * np.float32(v)).astype(np.float32)
    cfg = TsdfConfig(max_ray_length=1e6, min_ray_length=0.0).to_c()
    pose = np.array([1, 0, 0, 0, 0, 1, 0, 0, 0, 0, 1, 0], np.float32)
    keys = np.zeros((len(g), 3), np.int32)
    k = oracle_lib().vxo_grouped_ray_order(ctypes.byref(cfg), v, pts.ctypes.data_as(ctypes.c_void_p), len(pts),
                                           pose.ctypes.data_as(ctypes.POINTER(ctypes.c_float)),
                                           keys.ctypes.data_as(ctypes.c_void_p), len(g))
    return [tuple(int(x) for x in r) for r in keys[:k]]


def first_appearance(g):
    seen, out = set(), []
    for r in map(tuple, g.tolist()):
        if r not in seen:
            seen.add(r)
            out.append(r)
    return out


def test_initial_bucket_counts_match_survey():
    # SURVEY.md Appendix B table (probed from libstdc++ 13).
    assert schedule(307200, 1)[0][1] == 78779
    assert schedule(360960, 1)[0][1] == 92203
    assert schedule(135552, 1)[0][1] == 35933
    assert schedule(4194304, 1)[0][1] == 1056323
    s = schedule(307200, 307200)
    assert [bc for _, bc in s[:3]] == [78779, 159871, 324503]
    assert s[1][0] == 78779  # rehash fires when size == bucket count


@pytest.mark.parametrize("seed,n,span,repeat", [(1, 50, 3, 4), (2, 400, 40, 1), (3, 2000, 200, 1),
                                                (4, 3000, 6, 3), (5, 1, 1, 1), (6, 9000, 100, 1)])
def test_model_matches_unordered_map(seed, n, span, repeat):
    rng = np.random.default_rng(seed)
    g = rng.integers(-span, span + 1, (n, 3)).astype(np.int32)
    g = np.repeat(g, repeat, axis=0)
    rng.shuffle(g)
    v = 0.1
    truth = unordered_map_order(g, v)
    assert model_order(first_appearance(g), len(g)) == truth


def test_rehash_epochs_are_exercised():
    rng = np.random.default_rng(11)
    g = rng.integers(-500, 500, (2500, 3)).astype(np.int32)  # ~all distinct: K >> reserve(n/4+1)
    sch = schedule(len(g), len(g))
    assert len([e for e in sch if e[0] < len(g)]) >= 3
    assert model_order(first_appearance(g), len(g)) == unordered_map_order(g, 0.1)
