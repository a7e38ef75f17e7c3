#!/bin/bash
# Full ncu capture of one forward + backward of C5's passes, summarised on the
# box: per-launch summary and the top stall lines of each launch (the report
# itself stays on the box).
set -u
mkdir -p gpurun_out
python tools/prof_c2.py 5 1 > gpurun_out/plain_c5.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"fft_tma|wlr_kernel" -c 10 \
    -o /tmp/full_c5 python tools/prof_c2.py 5 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "full c5 rc=$?"
python tools/ncu_summary.py /tmp/full_c5.ncu-rep > gpurun_out/full_c5_summary.txt 2>&1
: > gpurun_out/full_c5_hotspots.txt
for i in 0 1 2 3 4 5 6 7 8 9; do python tools/ncu_hotspots.py /tmp/full_c5.ncu-rep $i 22 >> gpurun_out/full_c5_hotspots.txt 2>&1; done
ls -la gpurun_out/
