#!/bin/bash
# Round-2 ncu captures of the kernels without one yet: fp64 C3 chunk kernel, the
# C5 (2^26) chunk kernel inside the power loop, group_mapped block tiles on C2b/C2u,
# thread_mapped on C1/C2b. Outputs in gpurun_out/.
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
run() { tag=$1; k=$2; s=$3; shift 3; timeout 600 $N -k regex:$k -s $s -c 1 -o gpurun_out/prof_r2_$tag "$@" > gpurun_out/ncu_$tag.log 2>&1; echo "$tag=$?"; }
run c3_fp64 k_wo_chunk 2 python tools/spmv_one.py C3 work_oriented fp64
run c2b_block k_group_block 2 python tools/spmv_one.py C2b group_block
run c2u_block k_group_block 2 python tools/spmv_one.py C2u group_block
run c1_thread k_spmv_thread_mapped 2 python tools/spmv_one.py C1 thread_mapped
run c2u_thread k_spmv_thread_mapped 2 python tools/spmv_one.py C2u thread_mapped
run c5_chunk k_wo_chunk 70 python bench.py --mode power --steps 1 --warmup 3 --no-cpu-baseline --no-e2e
for f in gpurun_out/prof_r2_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}_summary.txt 2>&1; done
echo done
