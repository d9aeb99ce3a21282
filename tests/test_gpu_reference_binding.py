"""The reference's OWN hot-path code on the GPU through the reference-side
binding (VERDICT r1 "Next" #2).

oracle/_ref/ref_on_b200 is built by oracle/ref.mk from the unmodified reference
sources (/root/reference/proj/src/{engine,layouts,vmm,kv_attention}.cpp) plus
integration/b200_backend.cpp -- a `slotforge::Backend` whose virtual operators
call include/sf_b200.h -- and runs vmm_interleaved (vmm.cpp:179-236) and a
decode loop (Q/K/V projections, rope_apply, make_v_pieces, v_append, k_append,
qk_dot, exact softmax, softmax_times_v; kv_attention.cpp:111-241) on three
backends: the reference SimBackend, B200Backend and the CPU CKKS twin behind
the same interface (oracle/twin_backend.hpp). For every case:
  * decrypt(B200) matches SimBackend on ALL N slots (deferred garbage included)
    within the CKKS tolerance;
  * B200 ciphertext words == twin words (op-by-op, bit-exact);
  * levels and layouts == SimBackend's;
  * the inherited ledger (B200Backend::ledger(), what the reference's callers
    read), the library's own sf_ledger_totals and the twin's == SimBackend's.
"""
import json
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "ref_on_b200")

# CKKS precision bars (max |decrypt - SimBackend| relative to the largest slot):
# rings 2^12 carry ~2^-30 noise per op; ring 2^16 one hybrid key switch ~2^-18
TOL = {"vmm_small": 1e-6, "vmm_bsgs_deferred": 1e-6, "decode_small": 1e-5, "vmm_ring16": 1e-4,
       "decode_ring16": 1e-4}


def _run(*cases):
    assert os.path.exists(EXE), "build oracle/_ref/ref_on_b200 first (make -f oracle/ref.mk)"
    out = subprocess.run([EXE, *cases], capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout + out.stderr
    return [json.loads(line) for line in out.stdout.splitlines() if line.startswith("{")]


@pytest.mark.parametrize("case", ["vmm_small", "vmm_bsgs_deferred", "decode_small", "vmm_ring16",
                                  "decode_ring16"])
def test_reference_protocols_on_b200_backend(case):
    (r,) = _run(case)
    assert r["case"] == case
    assert r["words_equal"], r          # B200 == CPU twin, word for word
    assert r["words_compared"] > 0
    assert r["levels_equal"] and r["layouts_equal"], r
    assert r["ledger_equal"] and r["lib_ledger_equal"] and r["twin_ledger_equal"], r
    assert r["max_err"] <= TOL[case] * max(1.0, r["max_abs_ref"]), r


def test_reference_error_contract_through_binding():
    (r,) = _run("errors")
    assert r["ok"] and r["raised"] == r["expected"] > 0, r
