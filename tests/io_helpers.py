"""Seeded PLY / TUM files for the scan I/O parity tests."""
import numpy as np

TYPES = {"float": "<f4", "float32": "<f4", "double": "<f8", "float64": "<f8", "uchar": "u1", "uint8": "u1",
         "char": "i1", "int8": "i1", "short": "<i2", "int16": "<i2", "ushort": "<u2", "uint16": "<u2",
         "int": "<i4", "int32": "<i4", "uint": "<u4", "uint32": "<u4", "int64": "<i8", "uint64": "<u8"}


def write_ply(path, props, n, seed, binary=True, crlf=False, extra_elements=False, comments=True):
    """props: list of (type, name). Values: x,y,z in [-50, 50] (rounded to the type), colours 0..255,
    other props random. Returns the structured array written."""
    rng = np.random.default_rng(seed)
    dt = np.dtype([(name, TYPES[t]) for t, name in props])
    a = np.zeros(n, dt)
    for t, name in props:
        if name in ("x", "y", "z"):
            v = rng.uniform(-50, 50, n)
        elif name in ("red", "green", "blue"):
            v = rng.integers(0, 256, n)
        else:
            v = rng.uniform(-100, 100, n)
        if np.dtype(TYPES[t]).kind in "iu":
            info = np.iinfo(TYPES[t])
            v = np.clip(np.round(v), info.min, info.max)
        a[name] = v
    nl = "\r\n" if crlf else "\n"
    hdr = ["ply", f"format {'binary_little_endian' if binary else 'ascii'} 1.0"]
    if comments:
        hdr += ["comment seeded by tests/io_helpers.py", "obj_info synthetic"]
    hdr.append(f"element vertex {n}")
    hdr += [f"property {t} {name}" for t, name in props]
    if extra_elements:
        hdr += ["element face 0", "property list uchar int vertex_indices"]
    hdr.append("end_header")
    with open(path, "wb") as f:
        f.write((nl.join(hdr) + nl).encode())
        if binary:
            f.write(a.tobytes())
        else:
            for row in a:
                f.write((" ".join(repr(float(x)) if np.dtype(TYPES[t]).kind == "f" else str(int(x))
                                  for (t, _), x in zip(props, row)) + nl).encode())
    return a


def write_tum(path, n, seed, comments=True, crlf=False):
    rng = np.random.default_rng(seed)
    q = rng.normal(size=(n, 4))
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    t = rng.uniform(-5, 5, (n, 3))
    ts = 1.3e9 + np.cumsum(rng.uniform(0.01, 0.1, n))
    nl = "\r\n" if crlf else "\n"
    with open(path, "w", newline="") as f:
        if comments:
            f.write("# timestamp tx ty tz qx qy qz qw" + nl + nl)
        for i in range(n):
            f.write(f"{ts[i]:.6f} {t[i,0]:.6f} {t[i,1]:.6f} {t[i,2]:.6f} "
                    f"{q[i,0]:.7f} {q[i,1]:.7f} {q[i,2]:.7f} {q[i,3]:.7f}" + nl)
            if comments and i % 7 == 3:
                f.write("   # interleaved comment" + nl)
