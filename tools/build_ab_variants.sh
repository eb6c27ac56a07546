#!/bin/bash
# Builds ab/<name>.so: the shipped library with one source recompiled under extra -D flags.
#   tools/build_ab_variants.sh <source.cu> name1 "-DFOO=1 -DBAR=2" [name2 "..."] ...
set -eu
SRC=$1; shift
CS=paper_2602_21626_b200/csrc
B=paper_2602_21626_b200/build
mkdir -p ab
make -C $CS -j8 > /dev/null
ARCH="-gencode arch=compute_100a,code=sm_100a"
FLAGS="$ARCH -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -I$PWD/include -I$CS --expt-relaxed-constexpr"
base=$(basename $SRC .cu)
while [ $# -ge 2 ]; do
  name=$1; defs=$2; shift 2
  /usr/local/cuda/bin/nvcc $FLAGS $defs -c $CS/$SRC -o /tmp/ab_$name.o
  objs=$(ls $B/*.o | grep -v "/$base.o$")
  /usr/local/cuda/bin/nvcc $ARCH -shared -o ab/$name.so $objs /tmp/ab_$name.o -lcudart
  echo "built ab/$name.so ($defs)"
done
