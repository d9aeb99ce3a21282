#!/usr/bin/env bash
# GPU check after a change: all GPU tests (durations), smoke, default bench line.
#   gpurun -- bash tools/s2.sh TAG
TAG=${1:-s}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x --durations=10 > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py ${BENCH_ARGS:-} > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
python - <<PY
import json
d = json.loads(open("$OUT/bench.json").read().strip().splitlines()[-1])
print("value", d["value"], "e2e", d["e2e"]["value"], "stream", (d.get("e2e_stream") or {}).get("value"))
print({k: round(v["ms_per_step"], 3) for k, v in d["kernel_families"].items()})
print(d["phase_ms"])
print("parity", d.get("parity"))
PY
