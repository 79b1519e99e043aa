#!/bin/bash
# ncu --set full (with source) of one kernel (regex K) for the working tree's libroix.so and a saved one
# (LIB_B), one bench config (CFG); source pages exported to CSV on the box.
set -u
O=gpurun_out/${OUT:-pab}
mkdir -p $O
L=paper_2602_15917_b200/libroix.so
cp $L /tmp/lib_a.so
CMD="python bench.py --config ${CFG:-C3} ${SCALE:+--scale $SCALE} --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
for v in a b; do
  if [ $v = b ]; then cp $LIB_B $L; else cp /tmp/lib_a.so $L; fi
  $CMD > $O/plain_$v.json 2> $O/plain_$v.err || continue
  ncu --set full --clock-control none --import-source on -k "regex:$K" -s ${SKIP:-3} -c 1 -o $O/prof_$v -f $CMD > $O/ncu_$v.log 2>&1
  ncu -i $O/prof_$v.ncu-rep --page source --csv --print-source sass > $O/src_$v.csv 2>&1
  ncu -i $O/prof_$v.ncu-rep --page details > $O/details_$v.txt 2>&1
done
cp /tmp/lib_a.so $L
echo done
