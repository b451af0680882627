"""Prints the bench lines of tools/ab_env.sh (ms/step, e2e, stage times)."""
import glob, json, os
for f in sorted(glob.glob('gpurun_out/ab/run_*.json')):
    env = open(f[:-5] + '.env').read().strip() or '(defaults)'
    try:
        d = json.load(open(f))
    except Exception:
        print(env, 'FAILED:', open(f[:-5] + '.err').read()[-300:]); continue
    st = ' '.join(f'{k}={v:.3f}' for k, v in d['stages_ms_per_step'].items() if k not in ('h2d', 'd2h'))
    print(f"{env:40s} {d['ms_per_step']:.3f} ms  e2e {d['e2e']['ms_per_step']:.3f}  {st}")
