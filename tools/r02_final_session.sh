#!/bin/bash
# Round-2 final evidence on one box: GPU tests, the bench line (with the CPU
# leg), the reference arm, per-config latencies, the launch list of the bench
# workload.  (Per-kernel ncu --set full: tools/r02_sel_session.sh.)
set -u
OUT=gpurun_out
R=/tmp/ncu
mkdir -p $OUT $R
timeout 1200 python -m pytest tests -x -q -m gpu > $OUT/gpu_tests.log 2>&1
tail -2 $OUT/gpu_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > $OUT/r02_bench_config2_with_cpu.json 2> $OUT/bench_final.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > $OUT/r02_bench_reference_arm.json 2>> $OUT/bench_final.err
timeout 600 python tools/config_latency.py > $OUT/r02_config_latency.txt 2>&1
timeout 900 ncu --clock-control none --profile-from-start off --metrics gpu__time_duration.sum --csv --log-file $R/ll.csv python tools/prof_one.py 2 0 ${B:-74} bench > $OUT/ncu_ll2.log 2>&1
python tools/launch_summary.py $R/ll.csv > $OUT/r02_launches_cfg2_b${B:-74}.txt 2>&1
tail -1 $OUT/r02_bench_config2_with_cpu.json | cut -c1-300
cat $OUT/r02_config_latency.txt
