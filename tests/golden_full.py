"""Input digest shared by tests/golden/make_full_digests.py and the GPU test."""
import hashlib

import numpy as np


def input_digest(frames) -> str:
    h = hashlib.sha256()
    for x, c, p in frames:
        h.update(np.ascontiguousarray(x).tobytes())
        if c is not None:
            h.update(np.ascontiguousarray(c).tobytes())
        h.update(np.ascontiguousarray(p).tobytes())
    return h.hexdigest()
