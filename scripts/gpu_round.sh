#!/bin/bash
# One GPU call: build, gpu tests, bench lines (C2 default, C4, reference arm), launch list of the C2 step.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
nvidia-smi > gpurun_out/nvsmi.txt 2>&1; nproc > gpurun_out/host.txt; lscpu | head -20 >> gpurun_out/host.txt
timeout 1500 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS:-} > gpurun_out/gputests.log 2>&1; echo "gputests exit $?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench C2 exit $?"; cat gpurun_out/bench_C2.json
timeout 600 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 exit $?"; cat gpurun_out/bench_C4.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"; cat gpurun_out/bench_ref.json
