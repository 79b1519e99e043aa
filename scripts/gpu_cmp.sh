#!/bin/bash
# Compare bench variants: C2 and C4 with --extract mask / runs.
set -u
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1 || exit 1
for cfg in C2 C4; do for ex in mask runs; do
  timeout 300 python bench.py --config $cfg --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --extract $ex > gpurun_out/cmp_${cfg}_${ex}.json 2>&1
  python -c "import json;d=json.load(open('gpurun_out/cmp_${cfg}_${ex}.json'));print('$cfg $ex', round(d['value'],1), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()})"
done; done
