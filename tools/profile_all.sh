#!/bin/bash
# Launch lists (per-kernel device time) for every workload + a full ncu capture
# of the dominant kernel of C2; run under gpurun from the repo root.
set -u
mkdir -p gpurun_out
for w in 2 1 3 4 5; do
  python tools/prof_c2.py $w 1 > gpurun_out/plain_c$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_c$w.csv python tools/prof_c2.py $w 1 > gpurun_out/ncu_c$w.log 2>&1
  echo "c$w rc=$?"
done
