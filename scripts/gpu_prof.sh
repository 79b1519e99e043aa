#!/bin/bash
# ncu --set full of selected kernels (regex K) in one bench step (ARGS), after a plain run exits 0.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
CMD="python bench.py $ARGS --steps 1 --warmup 3 --no-e2e --no-cpu-baseline"
$CMD > gpurun_out/plain_prof.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:$K" -s ${SKIP:-0} -c ${COUNT:-5} -o gpurun_out/${OUT:-prof} -f $CMD > gpurun_out/ncu_prof.log 2>&1
echo "exit $?"; tail -3 gpurun_out/ncu_prof.log
