"""Reader for the MTFA archives written by oracle/mtfa.hpp.

TEST INFRASTRUCTURE ONLY (oracle/): used to turn reference dumps into the
committed golden fixtures under tests/golden/.
"""
import struct

import numpy as np

_DT = {0: np.float32, 1: np.float64, 2: np.int32, 3: np.int64, 4: np.uint8}


def read(path):
    out = {}
    with open(path, "rb") as f:
        if f.read(6) != b"MTFA1\n":
            raise ValueError(f"{path}: not an MTFA archive")
        while True:
            head = f.read(4)
            if not head:
                break
            (n,) = struct.unpack("<I", head)
            name = f.read(n).decode()
            code, nd = struct.unpack("<BI", f.read(5))
            dims = struct.unpack(f"<{nd}q", f.read(8 * nd))
            dt = np.dtype(_DT[code])
            cnt = int(np.prod(dims)) if nd else 1
            arr = np.frombuffer(f.read(cnt * dt.itemsize), dtype=dt).reshape(dims)
            out[name] = arr.copy()
    return out
