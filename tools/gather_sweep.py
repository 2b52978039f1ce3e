"""Random-access gather roofline sweep on the local GPU (measurement tool; prints one JSON per point)."""
import json
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3692_b200 as sa  # noqa: E402

for nbytes in (16 << 30,):
    for acc in (4, 8, 16, 32):
        for mult in (1, 2, 4, 8):
            r = sa.random_gather(0, buffer_bytes=nbytes, access_bytes=acc, n_threads=148 * 2048 * mult, loads=64)
            r.update(buffer=nbytes, threads=148 * 2048 * mult)
            print(json.dumps(r), flush=True)
r = sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=32, n_threads=148 * 2048 * 2, loads=64, dependent=True)
r.update(dependent=True)
print(json.dumps(r))
r = sa.random_gather(0, buffer_bytes=64 << 20, access_bytes=32, n_threads=148 * 2048 * 4, loads=64)
r.update(buffer=64 << 20, note="L2-resident")
print(json.dumps(r))
