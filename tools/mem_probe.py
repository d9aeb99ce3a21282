"""Device memory after the bench layer's warm-up steps (run on the GPU box):
   python tools/mem_probe.py"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import bench  # noqa: E402
import paper_2602_11470_b200 as sf  # noqa: E402


def mem(tag):
    free, tot = torch.cuda.mem_get_info()
    g, p = be.mem_stats()
    print(f"{tag:28s} used {(tot - free) / 2**30:7.2f} GiB of {tot / 2**30:.1f}; pool {p / 2**30:.2f} GiB graph {g / 2**30:.2f}",
          flush=True)


be = sf.Backend(bench.SLOTS, 7, alpha=2, seed=1)
mem("context")
layer = bench.LlamaLayer(be, sf, log=lambda *a: None)
mem("layer (plans, cache)")
for i in range(3):
    t0 = time.perf_counter()
    layer.step()
    be.synchronize()
    mem(f"step {i} ({(time.perf_counter() - t0) * 1e3:.0f} ms)")
for rep in range(2):
    t0 = time.perf_counter()
    for i in range(5):  # queued, as bench.py's eager loop
        outs = layer.step()
    t1 = time.perf_counter()
    be.synchronize()
    print(f"5 queued steps: host {(t1 - t0) * 1e3 / 5:.1f} ms/step, total {(time.perf_counter() - t0) * 1e3 / 5:.1f}")
    mem("after queued")
    for i in range(3):
        be.synchronize()
        t0 = time.perf_counter()
        outs = layer.step()
        t1 = time.perf_counter()
        be.synchronize()
        print(f"idle-queue step host {(t1 - t0) * 1e3:.1f} ms total {(time.perf_counter() - t0) * 1e3:.1f} ms")
    mem("after idle")
