"""DNT1 ingest throughput (developer tool): write a file with the given dims,
then time dmtk_gpu_tensor_load (file -> pinned staging -> HBM).

python tools/perf_ingest.py [--dims 500,500,500] [--path /tmp/t.dnt]
"""
import argparse
import json
import os
import struct
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1708_08976_b200 as dg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dims", default="500,500,500")
    ap.add_argument("--path", default="/tmp/dmtk_ingest.dnt")
    a = ap.parse_args()
    dims = tuple(int(v) for v in a.dims.split(","))
    n = int(np.prod(dims))
    with open(a.path, "wb") as f:
        f.write(b"DNT1" + struct.pack("<II", 1, len(dims)) + b"".join(struct.pack("<Q", d) for d in dims))
        chunk = 1 << 24
        rng = np.random.default_rng(1)
        for s in range(0, n, chunk):
            f.write(rng.random(min(chunk, n - s)).astype("<f8").tobytes())
    dg.DenseTensor.load(a.path).release()  # warm (page cache, context)
    t0 = time.perf_counter()
    t = dg.DenseTensor.load(a.path)
    dt = time.perf_counter() - t0
    t.release()
    os.unlink(a.path)
    print(json.dumps({"dims": dims, "GB": round(8 * n / 1e9, 3), "s": round(dt, 3),
                      "GBs": round(8 * n / dt / 1e9, 2), "note": "file in the page cache (second load)"}))


if __name__ == "__main__":
    main()
