#!/bin/bash
# Quick GPU check: build, the step/pipeline parity tests, C2 + C4 bench lines, launch lists of one step.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || { echo BUILD FAILED; tail -30 gpurun_out/build.log; exit 1; }
timeout 1500 python -m pytest -m gpu -x -q ${TESTS:-tests/test_gpu_steps.py tests/test_gpu_pipeline.py} > gpurun_out/gputests.log 2>&1; T=$?; echo "gputests exit $T"; tail -15 gpurun_out/gputests.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench C2 exit $?"; cat gpurun_out/bench_C2.json; tail -3 gpurun_out/bench_C2.err
timeout 300 python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 exit $?"; cat gpurun_out/bench_C4.json; tail -3 gpurun_out/bench_C4.err
if [ -n "${LAUNCHES:-}" ] && [ $T -eq 0 ]; then
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_C2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_C4.csv python bench.py --config C4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
  echo "ncu done"
fi
