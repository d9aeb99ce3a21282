#!/usr/bin/env bash
# One gpurun call: GPU parity tests, smoke, bench line, ncu launch list of one
# decode step, and ncu --set full captures of the top kernels.
#   gpurun --timeout 3000 -- bash tools/gpu_round.sh [tag] [what]
set -u
TAG=${1:-r1}
WHAT=${2:-all}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $OUT/gpu.txt 2>&1
if [[ $WHAT == all || $WHAT == *tests* ]]; then
  timeout 1200 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
  tail -3 $OUT/pytest_gpu.log
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
  tail -2 $OUT/smoke.log
fi
if [[ $WHAT == all || $WHAT == *bench* ]]; then
  timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
  cat $OUT/bench.json
fi
if [[ $WHAT == all || $WHAT == *ncu* ]]; then
  timeout 900 ncu --nvtx --nvtx-include "sf_step/" --metrics gpu__time_duration.sum --clock-control none \
      --csv --log-file $OUT/launches.csv python bench.py --nvtx-step --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
  echo "launch list rc=$?"
  for K in ${NCU_KERNELS:-fused_col_kernel ks_sum_kernel ks_row_kernel ntt_row_epi vmm_mac_kernel}; do
    timeout 900 ncu --nvtx --nvtx-include "sf_step/" --set full --clock-control none --import-source on \
        -k regex:$K -c 2 -o $OUT/full_$K python bench.py --nvtx-step --warmup 3 --no-cpu-baseline > $OUT/ncu_$K.log 2>&1
    echo "ncu $K rc=$?"
  done
fi
