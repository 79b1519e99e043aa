#!/bin/bash
# ncu --set full of the run-driven extraction (k_rx_runs) at C4 and C5 (one step each, after a plain run).
O=gpurun_out/ev5
mkdir -p $O
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
for c in C4 C5; do
  $B --config $c > $O/plain_$c.json 2> $O/plain_$c.err || continue
  ncu --set full --import-source on --clock-control none -k "regex:k_rx_runs" -s 3 -c 1 -o $O/full_${c}_rx $B --config $c > $O/full_${c}_rx.log 2>&1
  ncu -i $O/full_${c}_rx.ncu-rep --page details > $O/full_${c}_rx.txt 2>&1
done
echo done
