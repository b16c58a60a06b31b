#!/bin/bash
# one ncu --set full run capturing one launch per kernel class of the bench workload
OUT=gpurun_out
R=/tmp/ncu
mkdir -p $OUT $R
SEL=${SEL:-"gemm64:300,gemm64:1200,gemm32:5,gemv:20,gemv:21,gemv:22,applyq:100,applyq:300,concat:100,qr:200,qr:30,qrcl:10,qrcp:50,qrcpcl:100,svdcl2:100,svdcl4:3,svdcl1:2,svdsmall:5"}
ncu --clock-control none --profile-from-start off --set full --import-source on -o $R/sel -f \
  python tools/prof_sel.py 2 0 ${B:-74} bench "$SEL" > $OUT/ncu_sel.log 2>&1
python tools/ncu_summary.py $R/sel.ncu-rep > $OUT/r02_ncu_classes.txt 2>&1
tail -5 $OUT/ncu_sel.log
grep -c kernel: $OUT/r02_ncu_classes.txt
