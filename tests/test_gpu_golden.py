"""GPU vs the committed golden fixtures (generated from the reference itself by
tests/golden/make_golden.py): counters and VXBLX bytes must match exactly,
per-scan and batched."""
import os

import pytest

from golden_io import fixtures, load, tsdf_config_from
from paper_1611_03631_b200 import Scan, TsdfIntegrator, TsdfLayer
from parity_helpers import diff_report

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("batch", [False, True])
@pytest.mark.parametrize("path", fixtures(), ids=lambda p: os.path.basename(p)[:-4])
def test_gpu_matches_golden(gpu, path, batch):
    meta, _, frames, expected = load(path)
    layer = TsdfLayer(meta["voxel_size"], meta["vps"])
    integ = TsdfIntegrator(tsdf_config_from(meta), layer)
    scans = [Scan(x, c, p) for (x, c, p) in frames]
    if batch:
        stats = [[int(v) for v in row] for row in integ.integrate_batch(scans)]
    else:
        stats = []
        for s in scans:
            u = integ.integrate(s)
            stats.append([u, integ.raycasts_last_scan(), integ.skipped_points_last_scan()])
    assert stats == [list(s) for s in meta["stats"]]
    got = layer.save_bytes()
    assert got == expected, diff_report(got, expected)
