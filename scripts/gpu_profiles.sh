#!/bin/bash
# Round profile set: bench lines (C2 default, C4), ncu launch lists of one step (C2, C4), and one
# ncu --set full capture of the dominant kernel (k_extract) on C2 and on C4 at half scale.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
python bench.py > gpurun_out/bench_C2.json 2> gpurun_out/bench_C2.err; echo "bench C2 $?"
python bench.py --config C4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C4.json 2> gpurun_out/bench_C4.err; echo "bench C4 $?"
python bench.py --config C3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3.json 2> gpurun_out/bench_C3d.err; echo "bench C3 $?"
python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_C5.json 2> gpurun_out/bench_C5.err; echo "bench C5 $?"
python bench.py --config C1 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/bench_C1.json 2> gpurun_out/bench_C1.err; echo "bench C1 $?"
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv"
A="--steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-graph"
python bench.py $A > gpurun_out/plain1.log 2>&1 && ncu $M --log-file gpurun_out/launches_C2.csv python bench.py $A > /dev/null 2>&1; echo "launches C2 $?"
python bench.py $A --config C4 > gpurun_out/plain2.log 2>&1 && ncu $M --log-file gpurun_out/launches_C4.csv python bench.py $A --config C4 > /dev/null 2>&1; echo "launches C4 $?"
F="--set full --clock-control none --import-source on -k regex:^k_extract(_seg)?$ -s 1 -c 1"
ncu $F -o gpurun_out/full_extract_C2 -f python bench.py $A > gpurun_out/ncu_full_C2.log 2>&1; echo "full C2 $?"
python bench.py $A --config C4 --scale 0.5 > gpurun_out/plain3.log 2>&1 && ncu $F -o gpurun_out/full_extract_C4h -f python bench.py $A --config C4 --scale 0.5 > gpurun_out/ncu_full_C4h.log 2>&1; echo "full C4h $?"
A3="--config C3 --frames --background rev --classes 3 $A"
python bench.py $A3 > gpurun_out/plain4.log 2>&1 && ncu $M --log-file gpurun_out/launches_C3_next3.csv python bench.py $A3 > /dev/null 2>&1; echo "launches C3 next3 $?"
python bench.py --config C3 --frames --background rev --classes 3 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_C3_next3.json 2> gpurun_out/bench_C3.err; echo "bench C3 next3 $?"
