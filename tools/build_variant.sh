#!/bin/bash
# Build an experimental libnasch_b200 variant with extra nvcc defines:
#   tools/build_variant.sh NAME -DNB_TB_WIDE=1 ...   ->  variants/libnasch_NAME.so
# Select it at run time with NASCH_B200_LIB=variants/libnasch_NAME.so.
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
NAME=$1; shift
BASE="-O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC -Xptxas -v -I$ROOT/include -I$ROOT/paper_2309_14311_b200/csrc -ccbin /usr/bin/g++"
make -s -C "$ROOT/paper_2309_14311_b200/csrc" OUT="$ROOT/variants/libnasch_$NAME.so" \
  BUILD="$ROOT/variants/build_$NAME/" CLI="$ROOT/variants/bin_$NAME/nasch" NVFLAGS="$BASE $*" \
  "$ROOT/variants/libnasch_$NAME.so"
grep -A2 "nasch_tb_kernelIhLi128ELi16ELi16ELb1" "$ROOT/variants/build_$NAME/ptxas_engine.txt" | grep -o "Used [0-9]* registers.*" | head -1
