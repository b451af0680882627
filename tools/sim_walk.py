"""Dev probe (CPU, numpy fp32): how a free-space voxel's distance moves under
the exact update arithmetic when every record pulls it towards +truncation
(update_tsdf_voxel, tsdf_integrator.cpp:51-67, weight saturated at max_weight).
Prints the fraction of identity steps and the fraction of 32-record chunks whose
walk stays inside a window of +-k ulp around the chunk's start value — the case
for the speculative walk of the long-run fold."""
import numpy as np
f = np.float32
rng = np.random.default_rng(1)


def run(wlo, whi, n=64000, Wmax=f(10000), delta=f(0.1)):
    D = delta
    offs = []
    ws = np.exp(rng.uniform(np.log(wlo), np.log(whi), n)).astype(np.float32)
    u = np.spacing(delta)
    ident = 0
    for w in ws:
        T = f(Wmax + w)
        wc = f(w * delta)
        a = f(f(Wmax * D) + wc)
        q = f(a / T)
        ident += q == D
        D = q
        offs.append(int(round((D - delta) / u)))
    offs = np.array(offs).reshape(-1, 32)
    start = np.concatenate([[0], offs[:-1, -1]])
    rel = offs - start[:, None]
    out = {k: float(((rel.min(1) >= -k) & (rel.max(1) <= k)).mean()) for k in (3, 7)}
    return ident / n, out, (int(offs.min()), int(offs.max()))


for lo, hi in [(0.05, 1), (1, 10), (10, 100), (30, 300)]:
    print(f"w in [{lo}, {hi}]: identity steps, chunks inside +-3 / +-7 ulp, range in ulp:", run(lo, hi))
