#!/bin/bash
# Same-box A/B/..: each saved library in LIBS (space-separated "path" or "path|bench args") timed on
# C3 / C4 / C5, two rounds in rotation; TESTK runs those GPU tests against the working tree's
# libroix.so first.
set -u
O=gpurun_out/${OUT:-abn}
mkdir -p $O
L=paper_2602_15917_b200/libroix.so
cp $L /tmp/lib_cur.so
[ -n "${TESTK:-}" ] && { python -m pytest tests -m gpu -q -x -k "$TESTK" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt; }
B="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-next4"
for c in ${CFGS:-C3 C4 C5}; do
  for r in 1 2; do
    for ent in $LIBS; do
      lib=${ent%%|*}; args=""; [ "$ent" != "$lib" ] && args=${ent#*|}
      t=$(basename $lib .so)$(echo "$args" | tr -d ' -')
      cp $lib $L; python bench.py --config $c $B $args > $O/${t}_${c}_$r.json 2> $O/${t}_${c}_$r.err
    done
  done
done
cp /tmp/lib_cur.so $L
echo done
