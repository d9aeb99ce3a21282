#!/usr/bin/env bash
# Quick GPU check: selected GPU tests + a short bench (no CPU baselines, no emulation).
#   gpurun -- bash tools/quick.sh TAG "pytest -k expr"
TAG=${1:-q}
K=${2:-"benchconfig or parity"}
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q -k "$K" > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-emulate --no-sweep --no-extras > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("$OUT/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "eager", d.get("eager_ms_per_step"))
print({k: round(v["ms_per_step"], 3) for k, v in d["kernel_families"].items()})
print(d["phase_ms"])
print("parity", d.get("parity"))
PY
