#!/bin/bash
# A/B variants of one source: scripts/build_ab.sh <name> <path/to/source.cu> <replaces.o> [nvcc flags]
# compiles the given file (any path; includes resolve against csrc/) with -DLSK_TUNING and links it
# with the tuning build's other objects (`build.py --tuning`) into scripts/variants/liblsk_<name>.so
set -e
name=$1; src=$2; rep=$3; shift 3
R=$(cd "$(dirname "$0")/.." && pwd)
B=$R/paper_2006_07057_b200/build/tuning
mkdir -p $R/scripts/variants /tmp/lskvar
obj=/tmp/lskvar/ab_${name}.o
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC \
  -I$R/include -I$R/paper_2006_07057_b200/csrc -I$(python -c 'import sys; sys.path.insert(0,"'$R'/paper_2006_07057_b200"); import build; print(build.nccl_include())') \
  -DLSK_TUNING "$@" -c $src -o $obj
objs=$(ls $B/*.o | grep -v "/$rep$")
nvcc -shared -o $R/scripts/variants/liblsk_$name.so $objs $obj -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC -ldl
echo $R/scripts/variants/liblsk_$name.so
