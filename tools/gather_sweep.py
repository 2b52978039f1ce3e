"""Random-access gather roofline sweep on the local GPU (measurement tool; prints one JSON per point).

Footprint sweep at 32-B accesses: separates the DRAM random-sector rate from address-translation
(TLB reach) effects; access-size sweep at 16 GiB; dependent-chain latency."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1303_3692_b200 as sa  # noqa: E402

T = 148 * 2048 * 4
for nbytes in (64 << 20, 256 << 20, 1 << 30, 4 << 30, 16 << 30, 64 << 30):
    r = sa.random_gather(0, buffer_bytes=nbytes, access_bytes=32, n_threads=T, loads=64)
    r.update(buffer=nbytes, threads=T, sweep="footprint")
    print(json.dumps(r), flush=True)
for acc in (4, 8, 16, 32):
    r = sa.random_gather(0, buffer_bytes=16 << 30, access_bytes=acc, n_threads=T, loads=64)
    r.update(buffer=16 << 30, threads=T, sweep="access_bytes")
    print(json.dumps(r), flush=True)
for nbytes in (256 << 20, 16 << 30):
    r = sa.random_gather(0, buffer_bytes=nbytes, access_bytes=32, n_threads=148 * 2048, loads=64, dependent=True)
    r.update(buffer=nbytes, dependent=True, sweep="latency")
    r["ns_per_dependent_load"] = r["ms"] * 1e6 / 64
    print(json.dumps(r), flush=True)
