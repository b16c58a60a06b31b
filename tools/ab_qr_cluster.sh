for t in ${QR_THRESHOLDS:-74 148 100000}; do
  echo "T=$t" >> gpurun_out/ab.log
  HQ_QR_ONE_CTA_ABOVE=$t timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('ms/step %.1f  value %.3f e2e %.3f/s' % (d['ms_per_step'], d['value'], d['e2e']['value']))
print({k:(round(v['ms'],1),v['launches']) for k,v in d['kernel_time_by_kind'].items()})" >> gpurun_out/ab.log 2>&1
done
