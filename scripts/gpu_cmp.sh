#!/bin/bash
# Compare bench variants (C2 / C4, --extract mask / runs); optional test subset first.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
if [ -n "${TESTS:-}" ]; then timeout 900 python -m pytest -x -q -m gpu $TESTS > gpurun_out/gputests.log 2>&1; echo "tests exit $?"; tail -2 gpurun_out/gputests.log; fi
for cfg in ${CFGS:-C2 C4}; do for ex in ${EXS:-mask runs}; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --extract $ex > gpurun_out/cmp_${cfg}_${ex}.json 2>gpurun_out/cmp_${cfg}_${ex}.err
  python -c "import json;d=json.load(open('gpurun_out/cmp_${cfg}_${ex}.json'));print('$cfg $ex', round(d['value'],1), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()})"
done; done
