#!/bin/bash
# Round-2 ncu --set full captures of the dominant kernels per config (one GPU; each command ran
# without ncu first).  Outputs in gpurun_out/ev2/.
mkdir -p gpurun_out/ev2
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
# C3: a4 + a5 (binarisation chunk, register-row opening), histogram, compaction
ncu --set full --import-source on --clock-control none -k "regex:k_binarize|k_open2d_w|k_hist_u16|k_ck_extract" \
    -c 4 -o gpurun_out/ev2/full_C3 $B --config C3 > gpurun_out/ev2/full_C3.log 2>&1
# C4: compaction (dominant), histogram, run extraction, union-find
ncu --set full --import-source on --clock-control none -k "regex:k_ck_extract|k_hist_u16|k_extract_runs_rows|k_union_local" \
    -c 4 -o gpurun_out/ev2/full_C4 $B --config C4 > gpurun_out/ev2/full_C4.log 2>&1
# C5: histogram (dominant), compaction
ncu --set full --import-source on --clock-control none -k "regex:k_hist_u16|k_ck_extract" \
    -c 2 -o gpurun_out/ev2/full_C5 $B --config C5 > gpurun_out/ev2/full_C5.log 2>&1
