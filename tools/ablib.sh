#!/bin/bash
# Build an A/B variant of libcurast_b200.so with extra nvcc flags:
#   bash tools/ablib.sh NAME -DFOO=1 ...   ->  tools/ab/NAME.so  (CURAST_LIB=... in tools/s1_ab.py)
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p "$ROOT/tools/ab"
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 \
    -Xcompiler -fPIC -shared "$@" -o "$ROOT/tools/ab/$name.so" \
    "$ROOT/paper_2604_21749_b200/csrc/curast.cu" "$ROOT/paper_2604_21749_b200/csrc/resolve.cu"
