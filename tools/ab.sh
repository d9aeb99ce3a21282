#!/usr/bin/env bash
# GPU parity tests + A/B bench of environment toggles:  bash tools/ab.sh TAG "ENV1=.. ENV2=.." ["ENVx=.."]
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
i=0
for envs in "$@"; do
  i=$((i+1))
  env $envs timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_$i.json 2> $OUT/bench_$i.err
  echo "[$envs] rc=$?"; python -c "
import json,sys; d=json.load(open('$OUT/bench_$i.json')); print(d['value'], d['e2e'], d['phase_ms'], d['gpu_launches'], {k:round(v['ms_per_step'],2) for k,v in d['kernel_families'].items()})"
done
