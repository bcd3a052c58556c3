#!/bin/bash
# SpMM timing for library variants: SOS="lib1 lib2" CASES="C2u:16 C3:16"
for so in ${SOS:-paper_2301_04792_b200/_lib/liblwb200.so}; do
  for cs in ${CASES:-"C2u:16" "C3:16" "C3:4" "C3:64"}; do
    IFS=: read m n <<< "$cs"
    echo "$(basename $so) $(LWB200_LIB=$so timeout 300 python tools/spmm_one.py $m $n ${SCHED:-work_oriented} ${DT:-float32} 2>&1 | tail -1)"
  done
done
