#!/usr/bin/env bash
# Regenerates the reference-pinned golden vectors from the reference itself:
# oracle/ref.mk compiles /root/reference/proj/src (unmodified) + oracle/ref_golden.cpp
# into oracle/_ref/ref_golden, whose JSON output is committed here (gzip).
set -euo pipefail
cd "$(dirname "$0")/../.."
make -s -f oracle/ref.mk oracle/_ref/ref_golden
./oracle/_ref/ref_golden small  | gzip -9n > tests/golden/ref_small.json.gz
./oracle/_ref/ref_golden medium | gzip -9n > tests/golden/ref_medium.json.gz
./oracle/_ref/ref_golden harness | gzip -9n > tests/golden/ref_harness.json.gz
./oracle/_ref/ref_golden nonlinear | gzip -9n > tests/golden/ref_nonlinear.json.gz
ls -la tests/golden/
