#!/bin/bash
# applyq A/B: kernel tests, micro-benchmark per chunk width / buffer count, bench
OUT=gpurun_out
mkdir -p $OUT
python -m pytest tests/test_gpu_kernels.py -x -q -m gpu -k "applyq" > $OUT/applyq_tests.log 2>&1
tail -3 $OUT/applyq_tests.log
{
echo "== default"; python tools/applyq_batch_micro.py
echo "== nbuf 1"; HQ_APQ_NBUF=1 python tools/applyq_batch_micro.py
echo "== cw<=16"; HQ_APQ_CW=16 python tools/applyq_batch_micro.py
echo "== cw<=8"; HQ_APQ_CW=8 python tools/applyq_batch_micro.py
} > $OUT/applyq_micro.txt 2>&1
cat $OUT/applyq_micro.txt
python bench.py --steps 3 --warmup 3 --no-cpu-baseline > $OUT/bench_apq.json 2> $OUT/bench_apq.err
python -c "
import json
d=json.loads(open('$OUT/bench_apq.json').read().strip().splitlines()[-1])
print('value', d['value'], 'e2e', d['e2e']['value'], 'ms', d['ms_per_step'], 'rerr', d['r_sketch_rel_err_matrix0'])
print({k:round(v['ms'],1) for k,v in d['kernel_time_by_kind'].items()})
"
