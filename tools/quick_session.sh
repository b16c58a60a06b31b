#!/bin/bash
# kernel tests of the changed kernels + a short bench
OUT=gpurun_out
mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "${K:-skinny or applyq}" > $OUT/quick_tests.log 2>&1
tail -3 $OUT/quick_tests.log
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_quick.json 2> $OUT/bench_quick.err
tail -3 $OUT/bench_quick.err
python -c "
import json
d=json.loads(open('$OUT/bench_quick.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], 'rerr', d['r_sketch_rel_err_matrix0'], 'norm', d['norm_estimate'])
print({k:round(v['ms'],1) for k,v in d['kernel_time_by_kind'].items()})
print({k:(round(v['achieved'],1), round(v['frac'],3)) for k,v in d['roofline_by_kind'].items()})
"
