#!/bin/bash
# ONE ncu --set full run capturing one launch per kernel class of the bench
# workload (tools/prof_sel.py brackets only the selected ops).  Each captured
# kernel costs about a minute at batch 74 (ncu saves and restores the 150 GB
# of device memory around its replay passes), so the run carries its own
# timeout well inside gpurun's.
OUT=gpurun_out
R=/tmp/ncu
mkdir -p $OUT $R
SEL=${SEL:-"gemm64:300,gemm64:1200,gemm32:5,gemv:20,gemv:21,gemv:22,applyq:100,concat:100,qr:200,qrcpcl:100,svdcl2:100,svdsmall:5"}
timeout 1800 ncu --clock-control none --profile-from-start off --set full --import-source on -o $R/sel -f \
  python tools/prof_sel.py 2 0 ${B:-74} bench "$SEL" > $OUT/ncu_sel.log 2>&1
echo "ncu rc $?"
timeout 400 python tools/ncu_summary.py $R/sel.ncu-rep > $OUT/r02_ncu_classes.txt 2>&1
tail -3 $OUT/ncu_sel.log
grep -c kernel: $OUT/r02_ncu_classes.txt
