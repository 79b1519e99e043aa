#!/bin/bash
# Round-2 evidence refresh (final): GPU tests, smoke, bench lines, ncu launch lists, a full capture of
# the run-driven extraction at C5.  Outputs in gpurun_out/ev6/
set -x
O=gpurun_out/ev6
mkdir -p $O
python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1; echo "rc=$?" >> $O/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1; echo "rc=$?" >> $O/smoke.txt
python bench.py > $O/bench_default.json 2> $O/bench_default.err
for c in C1 C2 C4 C5; do
  python bench.py --config $c > $O/bench_$c.json 2> $O/bench_$c.err
done
python bench.py --impl reference > $O/bench_reference.json 2> $O/bench_reference.err
for c in C2 C3 C4 C5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file $O/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4 \
      > $O/ncu_launches_$c.log 2>&1
done
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
ncu --set full --import-source on --clock-control none -k "regex:k_rx_runs" -s 3 -c 1 -o $O/full_C5_rx $B --config C5 > $O/full_C5_rx.log 2>&1
ncu -i $O/full_C5_rx.ncu-rep --page details > $O/full_C5_rx.txt 2>&1
echo done
