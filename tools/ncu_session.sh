#!/bin/bash
# Per-kernel-class ncu captures of the bench workload (config 2, batch B,
# rank capacity 192, one non-graph factorization pass) and of config 3:
# launch lists (gpu__time_duration) and --set full captures of one
# representative launch per kernel class.  Reports stay in /tmp/ncu on the
# box; only their text summaries land in gpurun_out/ (size limit).
set -u
OUT=gpurun_out
R=/tmp/ncu
mkdir -p $R
B=${B:-32}
NCU="ncu --clock-control none --profile-from-start off"
if [ "${LL:-1}" = 1 ]; then
  $NCU --metrics gpu__time_duration.sum --csv --log-file $R/launches_cfg2_b$B.csv python tools/prof_one.py 2 0 $B 192 > $OUT/ncu_ll2.log 2>&1
  python tools/launch_summary.py $R/launches_cfg2_b$B.csv > $OUT/r02_launches_cfg2_b$B.txt 2>&1
  $NCU --metrics gpu__time_duration.sum --csv --log-file $R/launches_cfg3.csv python tools/prof_one.py 3 0 1 512 > $OUT/ncu_ll3.log 2>&1
  python tools/launch_summary.py $R/launches_cfg3.csv > $OUT/r02_launches_cfg3.txt 2>&1
fi
cap() {  # name regex skip config batch kcap
  $NCU --set full --import-source on -k "regex:$2" --launch-skip $3 --launch-count 1 -o $R/ncu_$1 -f \
    python tools/prof_one.py $4 0 $5 $6 > $R/ncu_$1.log 2>&1
  python tools/ncu_summary.py $R/ncu_$1.ncu-rep > $OUT/r02_ncu_$1.txt 2>&1
}
for spec in ${CAPS:-"gemm64:gemm_kernel<64:300:2:$B:192" "gemm32:gemm_kernel<32:100:2:$B:192" "applyq:applyq_kernel:100:2:$B:192" "concat:concat_kernel:100:2:$B:192" "gemvflat:gemv_flat_kernel:20:2:$B:192" "qr:qr_kernel:200:2:$B:192" "svdcl:svd_cluster_kernel:100:2:$B:192" "svdblock3:svd_block_kernel:2:3:1:512"}; do
  IFS=: read -r n k s c b kc <<< "$spec"
  cap "$n" "$k" "$s" "$c" "$b" "$kc"
done
du -sh $OUT
echo done
