#!/bin/bash
# ptxas register / spill summary of one csrc file: tools/ptxas_regs.sh render.cu [regex]
cd "$(dirname "$0")/../paper_2408_12677_b200/csrc"
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC -I../../include -Xptxas -v \
  -c "$1" -o /dev/null 2>&1 | awk -v re="${2:-.}" '
  /Compiling entry function/ {match($0, /_Z[^'"'"']*/); f=substr($0, RSTART, RLENGTH)}
  /spill stores/ {sp=$0; sub(/.*stack frame, /, "", sp)}
  /Used [0-9]+ registers/ {match($0, /Used [0-9]+ registers/); r=substr($0, RSTART+5, RLENGTH-15);
     if (f ~ re) { cmd="c++filt " f; cmd | getline d; close(cmd); printf "%4s regs | %-40s | %s\n", r, sp, substr(d,1,110)} }'
