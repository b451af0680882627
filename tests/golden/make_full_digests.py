#!/usr/bin/env python3
"""Digests of FULL-SIZE reference layers that are too large to commit as bytes
(tests/golden/full_digests.json), made by the REFERENCE ITSELF (oracle/_ref,
the unmodified /root/reference sources) and cross-checked against the oracle
restatement. Run in the build container:
    python tests/golden/make_full_digests.py
Each case stores the sha256 of the generated inputs (so generator drift is
caught), the reference's per-frame integrate() counters, the block count and
the sha256 of the reference's VXBLX bytes. tests/test_gpu_parity.py replays the
inputs on the B200 and must reproduce the digest.
"""
import hashlib
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

from oracle_bindings import OracleLayer, RefLayer, ref_available  # noqa: E402
from paper_1611_03631_b200 import workload as W  # noqa: E402

# (name, config id, first frame, frame count): two full 2048x2048 cfg4 frames, the
# 100-frame cfg1 batch bench.py times, and 40-frame prefixes of cfg2 and cfg3
CASES = [("cfg4_full_f1_f2", 4, 1, 2), ("cfg1_bench_x100", 1, 0, 100), ("cfg2_x40", 2, 0, 40), ("cfg3_x40", 3, 0, 40)]


def input_digest(frames) -> str:
    h = hashlib.sha256()
    for x, c, p in frames:
        h.update(np.ascontiguousarray(x).tobytes())
        if c is not None:
            h.update(np.ascontiguousarray(c).tobytes())
        h.update(np.ascontiguousarray(p).tobytes())
    return h.hexdigest()


def main():
    assert ref_available(), "oracle/_ref not built"
    path = os.path.join(HERE, "full_digests.json")
    out = json.load(open(path)) if os.path.exists(path) and "--all" not in sys.argv else {}
    for name, cfg_id, start, count in CASES:
        if name in out:  # kept (cfg4 alone is minutes of reference time); --all regenerates everything
            continue
        wc = W.CONFIGS[cfg_id]
        cfg = W.tsdf_config(wc)
        frames = W.frames(cfg_id, count=count, start=start)
        t = time.time()
        ref = RefLayer(cfg, wc.voxel_size, wc.vps)
        stats = [list(ref.integrate(*f)) for f in frames]
        ref_bytes = ref.save_bytes()
        t_ref = time.time() - t
        ora = OracleLayer(cfg, wc.voxel_size, wc.vps)
        o_stats = [list(ora.integrate(*f)) for f in frames]
        assert o_stats == stats and ora.save_bytes() == ref_bytes, "oracle restatement differs from _ref"
        out[name] = {"config": cfg_id, "start": start, "count": count, "input_sha256": input_digest(frames),
                     "stats": stats, "blocks": ref.block_count(), "vxblx_bytes": len(ref_bytes),
                     "vxblx_sha256": hashlib.sha256(ref_bytes).hexdigest(), "ref_seconds": round(t_ref, 1)}
        print(name, out[name], flush=True)
    json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
