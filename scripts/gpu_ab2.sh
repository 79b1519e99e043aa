#!/bin/bash
# Same-box A/B: the working tree's libroix.so against a saved one (LIB_B), C3 / C4 / C5 bench lines.
set -u
O=gpurun_out/${OUT:-ab2}
mkdir -p $O
L=paper_2602_15917_b200/libroix.so
cp $L /tmp/lib_a.so
[ -n "${TESTK:-}" ] && { python -m pytest tests -m gpu -q -x -k "$TESTK" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt; }
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
for c in ${CFGS:-C3 C4 C5}; do
  cp /tmp/lib_a.so $L; python bench.py --config $c $B > $O/a_$c.json 2> $O/a_$c.err
  cp $LIB_B $L;        python bench.py --config $c $B > $O/b_$c.json 2> $O/b_$c.err
  cp /tmp/lib_a.so $L; python bench.py --config $c $B > $O/a2_$c.json 2> $O/a2_$c.err
done
cp /tmp/lib_a.so $L
echo done
