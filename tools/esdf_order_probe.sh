#!/bin/bash
# Builds and runs tools/esdf_order_probe.cpp (needs /root/reference; CPU only).
set -e
R=/root/reference/proj
H=$(cd "$(dirname "$0")/.." && pwd)
OUT=${TMPDIR:-/tmp}/esdf_probe
mkdir -p $OUT
g++ -std=c++20 -O2 -ffp-contract=off -I$H/oracle/eigen_shim -I$R/include -o $OUT/probe \
  $H/tools/esdf_order_probe.cpp $R/src/esdf_integrator.cpp $R/src/serialization.cpp
python - "$OUT" <<'PY'
import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_1611_03631_b200 import workload as W
from oracle_bindings import OracleLayer
out = sys.argv[1]
for c, nf in ((1, 10), (2, 5), (3, 3)):
    wc = W.CONFIGS[c]; o = OracleLayer(W.tsdf_config(wc), wc.voxel_size, wc.vps)
    for f in range(nf):
        o.integrate(*W.frame(c, f * (10 if c == 1 else 1)))
    open(f'{out}/cfg{c}.vxblx', 'wb').write(o.save_bytes())
    print(f'cfg{c} {W.CONFIGS[c].truncation}', file=open(f'{out}/cfg{c}.trunc', 'w'))
PY
for c in 1 2 3; do echo "cfg$c:"; $OUT/probe $OUT/cfg$c.vxblx $(cut -d' ' -f2 $OUT/cfg$c.trunc); done
