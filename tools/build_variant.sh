#!/bin/bash
# Build an experimental variant of libb200tally.so with extra -D flags:
#   tools/build_variant.sh NAME -DBT_RELOAD=0 ...  -> build/variants/libb200tally_NAME.so
# then run with BT_LIB_PATH=build/variants/libb200tally_NAME.so (same C ABI).
set -e
cd "$(dirname "$0")/.."
name=$1; shift
mkdir -p build/variants
nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -lineinfo -std=c++17 \
  -Xcompiler -fPIC -shared -Xptxas -v "$@" -I include \
  -o build/variants/libb200tally_$name.so paper_2504_19048_b200/csrc/b200tally.cu \
  > build/variants/$name.log 2>&1 || { tail -20 build/variants/$name.log; exit 1; }
grep -A3 "walk_staged_kernelILi\(256ELi1\|192ELi2\|256ELi2\)E" build/variants/$name.log | grep -E "Used|spill" | paste - - | sed "s/^/$name: /" | cut -c1-200
