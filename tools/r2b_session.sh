#!/bin/bash
# batch-scaling experiment (n = 8192 so that large batches fit), per-op times of
# the bench workload, QR phase cycle counts (debug-timing build)
OUT=gpurun_out
mkdir -p $OUT
for b in 28 57 86 114 148; do
  python bench.py --n 8192 --batch $b --steps 3 --warmup 3 --no-cpu-baseline --no-instrument 2>/dev/null | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read()); print('n8192 batch', $b, 'ms/step %.1f value %.2f e2e %.2f' % (d['ms_per_step'], d['value'], d['e2e']['value']))" 
done > $OUT/batch_scaling.txt 2>&1
python tools/op_times.py 2 0 57 192 $OUT/op_times_b57.tsv > $OUT/op_times.log 2>&1
for spec in "256 200 1" "512 200 1" "700 256 1" "160 160 1" "1024 300 1"; do
  set -- $spec
  echo "== m $1 k $2 cl $3"; HQ_LIB=tools/libhq_qrdbg.so python tools/qr_timing.py $1 $2 $3 2>&1 | head -2
done > $OUT/qr_phases.txt 2>&1
cat $OUT/batch_scaling.txt; tail -2 $OUT/op_times.log
