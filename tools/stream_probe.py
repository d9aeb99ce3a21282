"""Host/device cost of the T-token decode stream (bench.token_stream), per token
and per host scope (run on the GPU box):

  SF_HOST_PROF=1 python tools/stream_probe.py [T]
"""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
import paper_2602_11470_b200 as sf  # noqa: E402
from paper_2602_11470_b200 import _native  # noqa: E402

T = int(sys.argv[1]) if len(sys.argv) > 1 else 16
be = sf.Backend(bench.SLOTS, 7, alpha=2, seed=1)
layer = bench.LlamaLayer(be, sf, log=lambda *a: None)
for _ in range(3):
    layer.step()
be.synchronize()
lib = _native.lib()
buf = ctypes.create_string_buffer(1 << 16)
if os.environ.get("SF_HOST_PROF"):
    lib.sf_host_profile(buf, len(buf), 1)
t0 = time.perf_counter()
print("---- stream", file=sys.stderr, flush=True)
r = bench.token_stream(be, sf, layer, T)
print(f"stream: {r}")
if os.environ.get("SF_STREAM_TWICE"):  # first-use effects: a second pass from the same cache
    r2 = bench.token_stream(be, sf, layer, T)
    print(f"second pass: {r2['token_ms']}")
print(f"wall {1e3 * (time.perf_counter() - t0) / T:.1f} ms/token")
if os.environ.get("SF_HOST_PROF"):
    lib.sf_host_profile(buf, len(buf), 1)
    rows = [ln.split() for ln in buf.value.decode().splitlines()]
    rows.sort(key=lambda x: -float(x[1]))
    print("host scopes (inclusive), per token:")
    for name, us, n in rows[:40]:
        print(f"  {name:28s} {float(us) / 1e3 / T:8.2f} ms  {int(n) / T:8.1f} calls")
