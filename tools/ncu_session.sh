#!/bin/bash
# Per-kernel-class ncu captures of the bench workload (config 2, batch 32,
# rank capacity 192, one non-graph factorization pass) and of config 3:
# launch lists (gpu__time_duration) and --set full captures of one
# representative launch per kernel class.  Output: gpurun_out/ncu_*.
set -u
OUT=gpurun_out
B=${B:-32}
NCU="ncu --clock-control none --profile-from-start off"
$NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_cfg2_b$B.csv python tools/prof_one.py 2 0 $B 192 > $OUT/ncu_ll2.log 2>&1
$NCU --metrics gpu__time_duration.sum --csv --log-file $OUT/launches_cfg3.csv python tools/prof_one.py 3 0 1 512 > $OUT/ncu_ll3.log 2>&1
cap() {  # name regex skip config batch kcap
  $NCU --set full --import-source on -k "regex:$2" --launch-skip $3 --launch-count 1 -o $OUT/ncu_$1 -f \
    python tools/prof_one.py $4 0 $5 $6 > $OUT/ncu_$1.log 2>&1
}
cap gemm64 "gemm_kernel<64" 300 2 $B 192
cap gemm32 "gemm_kernel<32" 100 2 $B 192
cap applyq "applyq_kernel" 100 2 $B 192
cap concat "concat_kernel" 100 2 $B 192
cap gemvflat "gemv_flat_kernel" 20 2 $B 192
cap gemv "gemv_kernel<2, 1>" 20 2 $B 192
cap qr "qr_kernel" 200 2 $B 192
cap qrcl "qr_cluster_kernel" 100 2 $B 192
cap svdcl "svd_cluster_kernel" 100 2 $B 192
cap svdblock3 "svd_block_kernel" 2 3 1 512
echo done
