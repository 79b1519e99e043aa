#!/bin/bash
# Round-2 evidence on one B200: tests, bench lines, ncu launch lists and
# full captures.  Outputs land in gpurun_out/ev/; the summaries are copied to profiles/r02/.
set -x
mkdir -p gpurun_out/ev
python -m pytest tests -m gpu -q > gpurun_out/ev/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/ev/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/ev/smoke.txt 2>&1
python bench.py > gpurun_out/ev/bench_default.json 2> gpurun_out/ev/bench_default.err
for c in C1 C2 C4 C5; do
  python bench.py --config $c > gpurun_out/ev/bench_$c.json 2> gpurun_out/ev/bench_$c.err
done
python bench.py --impl reference > gpurun_out/ev/bench_reference.json 2> gpurun_out/ev/bench_reference.err
for c in C2 C3 C4 C5; do
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv \
      --log-file gpurun_out/ev/launches_$c.csv python bench.py --config $c --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4 \
      > gpurun_out/ev/ncu_launches_$c.log 2>&1
done
