#!/bin/bash
# ptxas register / spill summary of one csrc file: tools/regs.sh spmv_work_oriented.cu [filter] [-Dextra...]
f=$1; shift; filt=${1:-.}; shift
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xptxas -v -I include -I paper_2301_04792_b200/csrc "$@" \
  -c paper_2301_04792_b200/csrc/$f -o /tmp/regs.o 2>&1 | python3 -c '
import sys,re,subprocess
name=None
for l in sys.stdin:
    m=re.search(r"Compiling entry function .(\S+).", l)
    if m: name=subprocess.run(["c++filt",m.group(1).rstrip("\x27")],capture_output=True,text=True).stdout.strip(); continue
    m=re.search(r"Used (\d+) registers", l)
    if m and name and re.search(sys.argv[1], name): print(m.group(1), "regs", name[:150])
    m=re.search(r"(\d+) bytes spill stores", l)
    if m and int(m.group(1)) and name and re.search(sys.argv[1], name): print("  SPILL", l.strip())
' "$filt"
