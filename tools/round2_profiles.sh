#!/bin/bash
# Round-2 evidence on one GPU (run under gpurun from the repo root): launch
# lists (per-kernel device time and DRAM bytes) of every config and full ncu
# captures of the passes changed this round.  Every ncu command runs only
# after the same program exited 0 without ncu.
set -u
mkdir -p gpurun_out
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for w in 1 2 3 4 5; do
  python tools/prof_c2.py $w 1 > gpurun_out/plain_c$w.log 2>&1 && \
  timeout 900 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_launches_c$w.csv \
      python tools/prof_c2.py $w 1 > gpurun_out/ncu_c$w.log 2>&1
  echo "launches c$w rc=$?"
  python tools/summarize_launches.py gpurun_out/r02_launches_c$w.csv > gpurun_out/r02_launches_c$w.txt 2>&1
done
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"fft_tma" -c 4 \
    -o gpurun_out/r02_full_c4 python tools/prof_c2.py 4 1 > gpurun_out/ncu_full_c4.log 2>&1
echo "full c4 rc=$?"
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"fft_tma|wlr_kernel" -c 10 \
    -o gpurun_out/r02_full_c5 python tools/prof_c2.py 5 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "full c5 rc=$?"
for w in 4 5; do python tools/ncu_summary.py gpurun_out/r02_full_c$w.ncu-rep > gpurun_out/r02_full_c${w}_summary.txt 2>&1; done
rm -f gpurun_out/r02_full_c*.ncu-rep
ls gpurun_out
