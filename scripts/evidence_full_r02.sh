#!/bin/bash
# Round-2 ncu --set full captures of the top kernels (one GPU; each command ran without ncu first),
# and the C5 bench line.  Outputs in gpurun_out/ev2/.
mkdir -p gpurun_out/ev2
python bench.py --config C5 > gpurun_out/ev2/bench_C5.json 2> gpurun_out/ev2/bench_C5.err
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
ncu --set full --import-source on --clock-control none -k "regex:k_binarize|k_open2d_w|k_hist_u16|k_ck_extract|k_union_local|k_extract_runs" \
    -c 6 -o gpurun_out/ev2/full_C3 $B --config C3 > gpurun_out/ev2/full_C3.log 2>&1
ncu --set full --import-source on --clock-control none -k "regex:k_ck_extract|k_open3d_rows|k_extract_runs_rows|k_union_local|k_hist_u16" \
    -c 5 -o gpurun_out/ev2/full_C4 $B --config C4 > gpurun_out/ev2/full_C4.log 2>&1
