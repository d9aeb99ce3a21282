#!/usr/bin/env bash
# launch list of one decode step + ncu --set full of the largest launch of the top kernels,
# summarised ON THE BOX (the .ncu-rep files are too large to bring back: only the
# markdown summary, the launch list and raw-metric / instruction-mix CSVs return)
#   gpurun -- bash tools/gpu_profile.sh TAG [K]
TAG=$1; K=${2:-5}
OUT=gpurun_out/$TAG; mkdir -p $OUT
timeout 900 ncu --nvtx --nvtx-include "sf_step/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    --csv --log-file $OUT/launches.csv python bench.py --nvtx-step --warmup 3 --no-cpu-baseline > $OUT/ncu_launch.log 2>&1
echo "launch list rc=$?"
SPECS=$(python tools/pick_launches.py $OUT/launches.csv $K); echo "picked: $SPECS"
bash tools/ncu_big.sh $TAG "$SPECS"
python tools/traffic.py $OUT/launches.csv > $OUT/traffic.json
REPS=$(ls $OUT/*.ncu-rep | paste -sd, -)
python tools/ncu_summary.py --rep "$REPS" --launches $OUT/launches.csv > $OUT/summary.md
for r in $OUT/*.ncu-rep; do
  b=${r%.ncu-rep}
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv --print-details all > $b.details.csv 2>/dev/null
  ncu -i $r --page source --csv --print-source sass > $b.sass.csv 2>/dev/null; gzip -f $b.sass.csv
  rm -f $r
done
du -sh $OUT
