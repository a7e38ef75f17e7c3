#!/bin/bash
# Full ncu capture (source-level) of one forward + backward of C5's passes.
set -u
mkdir -p gpurun_out
python tools/prof_c2.py 5 1 > gpurun_out/plain_c5.log 2>&1 || { echo "plain failed"; exit 1; }
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"fft_tma|wlr_kernel" -c 10 \
    -o gpurun_out/full_c5 python tools/prof_c2.py 5 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "full c5 rc=$?"
python tools/ncu_summary.py gpurun_out/full_c5.ncu-rep > gpurun_out/full_c5_summary.txt 2>&1
ls -la gpurun_out/
