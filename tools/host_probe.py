"""Host-side cost of one decode step, per C-ABI entry point (run on the GPU box).

  python tools/host_probe.py
"""
import collections
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_11470_b200 as sf  # noqa: E402
from paper_2602_11470_b200 import _native  # noqa: E402

be = sf.Backend(bench.SLOTS, 7, alpha=2, seed=1)
layer = bench.LlamaLayer(be, sf, log=lambda *a: None)
for _ in range(3):
    layer.step()
be.synchronize()
lib = _native.lib()
tot, cnt = collections.Counter(), collections.Counter()
for name in list(_native.SIGNATURES):
    f = getattr(lib, name)

    def wrap(*a, _f=f, _n=name):
        t = time.perf_counter()
        r = _f(*a)
        tot[_n] += time.perf_counter() - t
        cnt[_n] += 1
        return r
    setattr(lib, name, wrap)
steps = 3
t0 = time.perf_counter()
for _ in range(steps):
    layer.step()
t1 = time.perf_counter()
be.synchronize()
t2 = time.perf_counter()
print(f"host issue {1e3 * (t1 - t0) / steps:.2f} ms/step, drain {1e3 * (t2 - t1):.2f} ms, "
      f"C-ABI total {1e3 * sum(tot.values()) / steps:.2f} ms/step")
for n, v in tot.most_common(25):
    print(f"  {n:28s} {1e3 * v / steps:8.2f} ms/step  {cnt[n] // steps:6d} calls/step  {1e6 * v / cnt[n]:8.1f} us/call")

if os.environ.get("SF_HOST_PROF"):
    import ctypes
    lib.sf_host_profile(None, 0, 1)
    th = 0.0
    for _ in range(steps):
        be.synchronize()  # empty launch queue: host time below is not queue back-pressure
        t = time.perf_counter()
        layer.step()
        th += time.perf_counter() - t
    be.synchronize()
    print(f"host issue from an idle queue: {1e3 * th / steps:.2f} ms/step")
    buf = ctypes.create_string_buffer(1 << 16)
    lib.sf_host_profile(buf, 1 << 16, 1)
    rows = [l.split() for l in buf.value.decode().splitlines()]
    rows.sort(key=lambda r: -float(r[1]))
    print("host scopes (inclusive):")
    for name, us, n in rows[:40]:
        print(f"  {name:28s} {float(us) / 1e3 / steps:8.2f} ms/step  {int(n) // steps:6d} calls/step")
