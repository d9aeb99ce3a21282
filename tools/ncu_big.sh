#!/usr/bin/env bash
# ncu --set full captures of chosen launches (kernel regex + launch-skip within the NVTX step)
#   gpurun -- bash tools/ncu_big.sh TAG "regex:skip regex:skip ..."
TAG=$1; shift
OUT=gpurun_out/$TAG; mkdir -p $OUT
for spec in $1; do
  K=${spec%%:*}; S=${spec##*:}
  timeout 900 ncu --nvtx --nvtx-include "sf_step/" --set full --clock-control none --import-source on \
      -k regex:$K -s $S -c 1 -o $OUT/big_${K}_$S python bench.py --nvtx-step --warmup 3 --no-cpu-baseline > $OUT/ncu_${K}_$S.log 2>&1
  echo "ncu $K $S rc=$?"
done
