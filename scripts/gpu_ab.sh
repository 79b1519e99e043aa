#!/bin/bash
# Quick A/B on one B200: the compaction / pipeline GPU tests, then C3 / C4 / C5 bench lines (no e2e).
set -u
O=gpurun_out/${OUT:-ab}
mkdir -p $O
python -m pytest tests -m gpu -q -x -k "${TESTK:-extract or pipeline or fullsize or sharded}" > $O/pytest.txt 2>&1; echo "rc=$?" >> $O/pytest.txt
for c in ${CFGS:-C3 C4 C5}; do
  python bench.py --config $c --steps 10 --warmup 3 --no-e2e --no-cpu-baseline --no-next4 ${BARGS:-} > $O/bench_$c.json 2> $O/bench_$c.err
done
echo done
