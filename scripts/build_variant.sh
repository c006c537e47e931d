#!/bin/bash
# Tuning builds: recompile one source with extra -D flags and link a separate library
# (scripts/variants/liblsk_<name>.so, selected at run time with LSK_LIB_PATH).
# usage: scripts/build_variant.sh <name> <source.cu> [nvcc flags...]
set -e
name=$1; src=$2; shift 2
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2006_07057_b200/build/tuning   # objects of `build.py --tuning`
mkdir -p $R/scripts/variants /tmp/lskvar
obj=/tmp/lskvar/${name}_$(basename $src .cu).o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I$R/include -I$(python -c 'import sys; sys.path.insert(0,"'$R'/paper_2006_07057_b200"); import build; print(build.nccl_include())') \
  -DLSK_TUNING "$@" -c $R/paper_2006_07057_b200/csrc/$src -o $obj
objs=$(ls $B/*.o | grep -v "/$(basename $src .cu).o$")
nvcc -shared -o $R/scripts/variants/liblsk_$name.so $objs $obj -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -ldl
echo $R/scripts/variants/liblsk_$name.so
