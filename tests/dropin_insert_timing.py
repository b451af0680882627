"""Per-scan insert time of a caller of the reference's C++ API (cli.cpp:168-186),
once with the reference's own integrator on one host core and once with the
B200 drop-in (vxf::TsdfIntegrator over libvxg.so, updated blocks written back
into the caller's host TsdfLayer). Both binaries are built by oracle/Makefile
from oracle/bench_insert.cpp (oracle/_ref travels to the GPU box).
Test infrastructure: run(cfg, frames) is called by tests/test_gpu_dropin.py;
as a script: python tests/dropin_insert_timing.py <cfg> <frames> [out.json]"""
import json, os, struct, subprocess, sys, tempfile
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
from paper_1611_03631_b200 import workload as W


def run(cfg: int, n: int) -> dict:
    wc = W.CONFIGS[cfg]
    fr = W.frames(cfg, count=n)
    with tempfile.NamedTemporaryFile(suffix='.scans', delete=False) as f:
        f.write(struct.pack('<I', len(fr)))
        for x, c, p in fr:
            x = np.ascontiguousarray(x, dtype=np.float32)
            c = np.ascontiguousarray(c, dtype=np.uint8) if c is not None else np.zeros((len(x), 3), np.uint8)
            f.write(struct.pack('<I', len(x)))
            f.write(np.ascontiguousarray(p, dtype=np.float32).tobytes())
            f.write(x.tobytes()); f.write(c.tobytes())
        path = f.name
    args = [path, repr(wc.voxel_size), repr(wc.truncation), repr(wc.dropoff_epsilon), repr(wc.max_ray), str(wc.merge_mode),
            str(wc.weight_mode), repr(wc.min_ray), repr(wc.max_weight)]
    out = {'workload': wc.name, 'scans': len(fr)}
    for name in ('vxg', 'ref'):
        exe = os.path.join(ROOT, 'oracle', '_ref', f'bench_insert_{name}')
        cmd = (['taskset', '-c', '0'] if name == 'ref' else []) + [exe] + args
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=1200)
        assert r.returncode == 0, r.stderr[-2000:]
        out[name] = json.loads(r.stdout.strip().splitlines()[-1])
    os.unlink(path)
    assert out['vxg']['updates'] == out['ref']['updates'] and out['vxg']['blocks'] == out['ref']['blocks']
    out['speedup_median'] = out['ref']['median_ms'] / out['vxg']['median_ms']
    return out


if __name__ == "__main__":
    out = run(int(sys.argv[1]), int(sys.argv[2]))
    line = json.dumps(out)
    print(line)
    if len(sys.argv) > 3:
        open(sys.argv[3], 'w').write(line + '\n')
