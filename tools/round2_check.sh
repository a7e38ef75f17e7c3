#!/bin/bash
# GPU check of the round-2 build: GPU tests, smoke(), the default bench line
# (C5 with parity gate, e2e, cpu_baseline, per_config) and the reference arm.
set -u
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x > gpurun_out/r02_pytest_gpu.log 2>&1
echo "pytest gpu rc=$? $(tail -1 gpurun_out/r02_pytest_gpu.log)"
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1
echo "smoke rc=$? $(tail -1 gpurun_out/r02_smoke.log)"
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err
echo "bench default rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
echo "bench reference rc=$?"
nproc
