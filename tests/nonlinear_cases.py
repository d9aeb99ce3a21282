"""TEST INFRASTRUCTURE: replays the reference's nonlinear golden cases
(tests/golden/ref_nonlinear.json.gz, oracle/ref_golden.cpp `nonlinear` set) on
any backend through paper_2602_11470_b200.nonlinear."""
import gzip
import json
import os

import numpy as np

from paper_2602_11470_b200 import nonlinear as NL

GOLD = os.path.join(os.path.dirname(__file__), "golden", "ref_nonlinear.json.gz")


def cases():
    with gzip.open(GOLD, "rt") as f:
        return json.load(f)["cases"]


def run_case(c, be, make_layout, seed_base=100):
    """Encrypt the case inputs on `be`, run the op, return (outputs, levels)."""
    ly = None
    if c["layout"]:
        j = c["layout"]
        ly = make_layout(j["d"], c["N"], j["offset"], j["heads"], j["deferred_mask"])
    xs = [be.encrypt(np.array(s), c["L"], ly, seed=seed_base + i) for i, s in enumerate(c["inputs"])]
    spec = NL.ApproxSpec.from_json(c["spec"]) if "spec" in c else None
    e = c["extra"]
    op = c["op"]
    if op == "eval_cheb":
        outs = [NL.eval_cheb(be, xs[0], e["lo"], e["hi"], e["coeffs"])]
    elif op == "eval_cheb_masked":
        outs = [NL.eval_cheb(be, xs[0], e["lo"], e["hi"], e["coeffs"], np.array(e["mask"]))]
    elif op in ("inverse", "rsqrt"):
        outs = [NL.goldschmidt(be, xs[0], op, spec)]
    elif op == "exp":
        outs = [NL.approx_exp(be, xs[0], spec)]
    elif op == "softmax":
        outs = NL.approx_softmax(be, xs, e["n_prime"], e["heads"], spec)
    elif op == "norm":
        outs = [NL.approx_norm(be, xs[0], np.array(e["gamma"]), np.array(e["beta"]), e["eps"], spec)]
    elif op == "silu":
        outs = [NL.approx_silu(be, xs[0], spec)]
    else:
        raise ValueError(op)
    return outs
