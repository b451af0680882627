"""Pipeline shapes that only large inputs reach, forced on small ones through
the library's environment knobs (read once per process, so each case runs in
its own subprocess) and compared bit-exactly with the oracle:

* chunked batches: records produced, sorted and folded in chunks of
  consecutive rays with two buffer sets (cfg4-size frames exceed 2^29
  records per batch) — VXG_CHUNK_RECORDS;
* host inputs split into sub-batches whose H2D copies overlap the previous
  sub-batch's compute — VXG_H2D_PARTS;
* the synchronous fold (every call joins its fold) — VXG_SYNC_FOLD.
"""
import os
import subprocess
import sys
import tempfile

import numpy as np
import pytest

from paper_1611_03631_b200 import workload as W
from oracle_bindings import OracleLayer
from parity_helpers import diff_report

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

_CHILD = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1611_03631_b200 import TsdfIntegrator, TsdfLayer
from paper_1611_03631_b200 import workload as W
wc = W.CONFIGS[{cfg}]
cfg = W.tsdf_config(wc)
layer = TsdfLayer(wc.voxel_size, wc.vps)
integ = TsdfIntegrator(cfg, layer)
stats = []
for b in range({batches}):
    fr = W.frames({cfg}, count={count}, scale={scale}, start=b * {count})
    xyz, rgb, off, poses = W.pack(fr)
    if {host}:
        import torch
        hx = torch.from_numpy(xyz).pin_memory()
        hc = torch.from_numpy(rgb).pin_memory() if rgb is not None else None
        st = integ.integrate_packed(hx.data_ptr(), hc.data_ptr() if hc is not None else None, off, poses, False)
    else:
        import torch
        dx = torch.from_numpy(xyz).cuda()
        dc = torch.from_numpy(rgb).cuda() if rgb is not None else None
        st = integ.integrate_packed(dx.data_ptr(), dc.data_ptr() if dc is not None else None, off, poses, True)
    stats += [tuple(int(v) for v in row) for row in st]
open({out!r}, "wb").write(layer.save_bytes())
np.save({out!r} + ".stats.npy", np.array(stats, dtype=np.uint64))
"""


def _run(env_extra, cfg=1, batches=2, count=3, scale=0.5, host=False):
    with tempfile.TemporaryDirectory() as td:
        out = os.path.join(td, "layer.vxblx")
        code = _CHILD.format(root=ROOT, cfg=cfg, batches=batches, count=count, scale=scale, host=host, out=out)
        env = dict(os.environ)
        env.update(env_extra)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        data = open(out, "rb").read()
        stats = [tuple(int(v) for v in row) for row in np.load(out + ".stats.npy")]
    wc = W.CONFIGS[cfg]
    ora = OracleLayer(W.tsdf_config(wc), wc.voxel_size, wc.vps)
    o_stats = []
    for b in range(batches):
        for (x, c, p) in W.frames(cfg, count=count, scale=scale, start=b * count):
            o_stats.append(ora.integrate(x, c, p))
    assert stats == o_stats
    ob = ora.save_bytes()
    assert data == ob, diff_report(data, ob)


@pytest.mark.parametrize("chunk", [150_000, 1_000_000])
def test_chunked_batches(gpu, chunk):
    """Several record chunks per batch (and a fold per chunk that outlives the
    next chunk's emit and sort), over two consecutive batches."""
    _run({"VXG_CHUNK_RECORDS": str(chunk)})


def test_chunked_cfg3_lidar(gpu):
    _run({"VXG_CHUNK_RECORDS": "200000"}, cfg=3, batches=1, count=2, scale=0.5)


@pytest.mark.parametrize("parts", [2, 3])
def test_host_input_subbatches(gpu, parts):
    """Pinned host input split into sub-batches (the H2D copy of part k+1
    overlaps part k); with chunking inside the parts as well."""
    _run({"VXG_H2D_PARTS": str(parts), "VXG_CHUNK_RECORDS": "400000"}, host=True)


def test_synchronous_fold(gpu):
    _run({"VXG_SYNC_FOLD": "1"})


@pytest.mark.parametrize("prod", [1, 2])
def test_long_run_layouts(gpu, prod):
    """Both long-run layouts of the fold on the same batches: producer/consumer
    pairs (full batches) and two-producer teams (small folds), which the host
    otherwise picks by the fold's record count (VXG_FOLD_PROD forces one); the
    fixed long-run threshold (full-batch behaviour) on small batches as well."""
    _run({"VXG_FOLD_PROD": str(prod)})
    _run({"VXG_FOLD_PROD": str(prod), "VXG_FIXED_LONG_RUN": "1"}, batches=1, count=4)
