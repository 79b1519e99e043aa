#!/bin/bash
# ncu captures: --set full of the step's main kernels (C2 default bench; C4 at half scale), after plain runs exit 0.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
K='regex:k_extract<|k_hist|k_open3d_reg|k_extract_runs|k_union_local|k_binarize|k_range'
C2="python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
C4="python bench.py --config C4 --scale 0.5 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline"
$C2 > gpurun_out/plain_C2.log 2>&1 && $C4 > gpurun_out/plain_C4h.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "$K" -s 7 -c 7 -o gpurun_out/prof_C2 -f $C2 > gpurun_out/ncu_C2.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k "$K" -s 6 -c 6 -o gpurun_out/prof_C4h -f $C4 > gpurun_out/ncu_C4h.log 2>&1
echo "exit $?"; tail -3 gpurun_out/ncu_C2.log gpurun_out/ncu_C4h.log
