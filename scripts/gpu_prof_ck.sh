#!/bin/bash
# ncu --set full (with source) of the compaction kernel at C4 and C5 (half scale), after plain runs
# exit 0; the source pages are exported to CSV on the box for scripts/sass_mix.py.
set -u
mkdir -p gpurun_out/ck
for c in C4 C5; do
  CMD="python bench.py --config $c --scale 0.5 --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
  $CMD > gpurun_out/ck/plain_$c.json 2> gpurun_out/ck/plain_$c.err || exit 1
  ncu --set full --clock-control none --import-source on -k "regex:k_ck_extract" -s 3 -c 1 \
      -o gpurun_out/ck/prof_$c -f $CMD > gpurun_out/ck/ncu_$c.log 2>&1
  ncu -i gpurun_out/ck/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/ck/src_$c.csv 2>&1
  ncu -i gpurun_out/ck/prof_$c.ncu-rep --page details > gpurun_out/ck/details_$c.txt 2>&1
done
echo done
