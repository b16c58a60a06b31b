#!/bin/bash
# Round-2 final evidence on one box: the bench line (with the CPU leg), the
# reference arm, launch list + ncu --set full per kernel class of the bench
# workload (74 matrices, bench capacity profile), per-config latencies.
set -u
OUT=gpurun_out
R=/tmp/ncu
mkdir -p $OUT $R
B=${B:-74}
python bench.py --steps 5 --warmup 3 > $OUT/r02_bench_config2_with_cpu.json 2> $OUT/bench_final.err
python bench.py --impl reference --steps 2 --warmup 1 > $OUT/r02_bench_reference_arm.json 2>> $OUT/bench_final.err
python tools/config_latency.py > $OUT/r02_config_latency.txt 2>&1
NCU="ncu --clock-control none --profile-from-start off"
$NCU --metrics gpu__time_duration.sum --csv --log-file $R/ll.csv python tools/prof_one.py 2 0 $B bench > $OUT/ncu_ll2.log 2>&1
python tools/launch_summary.py $R/ll.csv > $OUT/r02_launches_cfg2_b$B.txt 2>&1
cap() {  # name regex skip
  $NCU --set full --import-source on -k "regex:$2" --launch-skip $3 --launch-count 1 -o $R/ncu_$1 -f \
    python tools/prof_one.py 2 0 $B bench > $R/ncu_$1.log 2>&1
  python tools/ncu_summary.py $R/ncu_$1.ncu-rep > $OUT/r02_ncu_$1.txt 2>&1
}
for spec in "gemm64:gemm_kernel<64:300" "gemm32:gemm_kernel<32:100" "gemmskinny:gemm_skinny_kernel:50" "applyq:applyq_kernel:100" "concat:concat_kernel:100" "gemvflat:gemv_flat_kernel:20" "qr:qr_kernel:200" "qrcluster:qr_cluster_kernel:60" "qrcp:qrcp_kernel:100" "svdcl:svd_cluster_kernel:100" "svdsmall:svd_small_kernel:20"; do
  IFS=: read -r n k s <<< "$spec"
  cap "$n" "$k" "$s"
done
du -sh $OUT
echo done
