#!/bin/bash
# Round evidence on one GPU (run under gpurun from the repo root):
#   smoke(), the default bench line (C2 with e2e + cpu_baseline), the reference
#   arm, one bench line per workload, ncu launch lists (per-kernel device time
#   and DRAM bytes) for every workload, and a full ncu capture of the C2 passes.
# Every ncu command runs only after the same program exited 0 without ncu.
set -u
mkdir -p gpurun_out
# (ncu reports stay in /tmp: gpurun copies back at most 64 MiB of gpurun_out/)
rm -f /tmp/full_c2.ncu-rep /tmp/full_c3.ncu-rep /tmp/full_c4.ncu-rep /tmp/full_c5.ncu-rep
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1
echo "smoke rc=$?"
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1
echo "pytest gpu rc=$?"
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
echo "bench default rc=$?"
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
echo "bench reference rc=$?"
for w in c1 c2 c3 c4 c5; do
  python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_$w.json 2> gpurun_out/bench_$w.err
  echo "bench $w rc=$?"
done
python bench.py --workload cg --steps 60 --warmup 4 > gpurun_out/bench_cg.json 2> gpurun_out/bench_cg.err
echo "bench cg rc=$?"
python tools/prof_cg.py 4 > gpurun_out/plain_cg.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_cg.csv python tools/prof_cg.py 4 > gpurun_out/ncu_cg.log 2>&1
echo "launches cg rc=$?"
python bench.py --workload ista --steps 50 --warmup 3 > gpurun_out/bench_ista.json 2> gpurun_out/bench_ista.err
echo "bench ista rc=$?"
python tools/prof_ista.py 2 > gpurun_out/plain_ista.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_ista.csv python tools/prof_ista.py 2 > gpurun_out/ncu_ista.log 2>&1
echo "launches ista rc=$?"
for w in 2 1 3 4 5; do
  python tools/prof_c2.py $w 1 > gpurun_out/plain_c$w.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
      --log-file gpurun_out/launches_c$w.csv python tools/prof_c2.py $w 1 > gpurun_out/ncu_c$w.log 2>&1
  echo "launches c$w rc=$?"
done
python tools/prof_c2.py 2 1 > /dev/null 2>&1 && \
  ncu --set full --import-source on --clock-control none -k regex:fft_tma_kernel -c 3 \
      -o /tmp/full_c2 python tools/prof_c2.py 2 1 > gpurun_out/ncu_full_c2.log 2>&1
echo "full c2 rc=$?"
python tools/prof_c2.py 5 1 > /dev/null 2>&1 && \
  timeout 1200 ncu --set full --import-source on --clock-control none -k regex:"fft_tma|wht_tile|lr_" -c 9 \
      -o /tmp/full_c5 python tools/prof_c2.py 5 1 > gpurun_out/ncu_full_c5.log 2>&1
echo "full c5 rc=$?"
for w in 3 4; do
  python tools/prof_c2.py $w 1 > /dev/null 2>&1 && \
    ncu --set full --import-source on --clock-control none -k regex:"fft_tma|fft_tile|wht_tile" -c 8 \
        -o /tmp/full_c$w python tools/prof_c2.py $w 1 > gpurun_out/ncu_full_c$w.log 2>&1
  echo "full c$w rc=$?"
  python tools/ncu_summary.py /tmp/full_c$w.ncu-rep > gpurun_out/full_c${w}_summary.txt 2>&1
done
python tools/ncu_summary.py /tmp/full_c2.ncu-rep > gpurun_out/full_c2_summary.txt 2>&1
python tools/ncu_summary.py /tmp/full_c5.ncu-rep > gpurun_out/full_c5_summary.txt 2>&1
