"""The reference's OWN test suite, compiled unmodified from /root/reference
(oracle/ref.mk, over the small Eigen / doctest / json shims in oracle/shim):
every test binary must pass. This pins the shims -- and hence every golden
vector and report the reference-built tools emit (tests/golden/*) -- to the
reference's own expectations. Skipped where the reference build is absent
(the GPU box ships the prebuilt binaries)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SUITES = ["test_engine", "test_layouts", "test_vmm", "test_kv", "test_harness", "test_nonlinear", "test_placement"]


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes(suite):
    exe = os.path.join(ROOT, "oracle", "_ref", suite)
    if not os.path.exists(exe):
        pytest.skip("reference not built here (make -f oracle/ref.mk)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    last = (r.stdout.strip().splitlines() or [""])[-1]
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "failed: 0 | assertions:" in last and last.rstrip().endswith("failed: 0"), last
