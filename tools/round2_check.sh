#!/bin/bash
# GPU check of the round-2 build: GPU tests, smoke(), the default bench line
# (C5 with parity gate, e2e, cpu_baseline, per_config), the reference arm, and
# the C5 launch list (ncu, cold-cache serialised per-launch times).
set -u
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest gpu rc=$? $(tail -1 gpurun_out/r02_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/r02_smoke.log)"
timeout 900 python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
echo "bench default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
echo "bench reference rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches_c5.csv python bench.py --steps 2 --warmup 1 --no-e2e \
  --no-cpu-baseline --no-per-config > gpurun_out/r02_ncu_c5.log 2>&1
echo "ncu c5 rc=$?"
nproc
