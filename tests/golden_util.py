"""Loading and replaying the reference-pinned golden cases (tests/golden/*.json.gz).

Each case was produced by the reference itself (oracle/ref_golden.cpp linked
against /root/reference/proj/src compiled by oracle/ref.mk). The replay
helpers run the same case through any slotforge-shaped backend (numpy slot sim,
CKKS CPU oracle, or the GPU product) using the oracle protocol restatements,
so one function serves every parity level.
"""
from __future__ import annotations

import functools
import gzip
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))


@functools.lru_cache(maxsize=None)
def load(which: str = "small"):
    with gzip.open(os.path.join(HERE, "golden", f"ref_{which}.json.gz"), "rt") as f:
        return json.load(f)


def cases(which: str, kind: str):
    return [c for c in load(which)["cases"] if c["kind"] == kind]


def layout_from(j):
    from oracle.layout import Layout
    if j is None:
        return None
    return Layout(j["kind"], j["d"], j["t"], j["offset"], j["heads"], j["deferred_mask"])


def counts_dict(c):
    return {k: getattr(c, k) for k in ("rotations", "hoisted_rotations", "ct_pt_mults",
                                       "ct_ct_mults", "additions", "bootstraps")}
