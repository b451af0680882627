"""Dev probe: run-length distribution of a VXG_DUMP_RECORDS dump."""
import sys
import numpy as np
f = open(sys.argv[1], "rb")
T, kbits = np.frombuffer(f.read(16), np.uint64)
keys = np.frombuffer(f.read(int(T) * 4), np.uint32)
keys = keys[keys != 0xFFFFFFFF]
cnt = np.bincount(keys)
cnt = cnt[cnt > 0]
tot = cnt.sum()
print("records", tot, "runs", len(cnt), "max", cnt.max())
for th in [32, 128, 512, 1024, 2048, 4096, 8192, 16384, 32768]:
    m = cnt >= th
    print(f">= {th:6d}: runs {m.sum():7d}  records {cnt[m].sum() / tot:.3f}")
