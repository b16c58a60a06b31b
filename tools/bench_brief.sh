#!/bin/bash
# usage: tools/bench_brief.sh N [extra bench args]
python bench.py --n $1 --steps 3 --warmup 3 --no-cpu-baseline "${@:2}" 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms/step %.1f  e2e %.3f/s  gflops %.2f' % (d['ms_per_step'], d['e2e']['value'], d['fp64_gflops_effective']))
print({k:(round(v['ms'],1),v['launches']) for k,v in d['kernel_time_by_kind'].items()})"
