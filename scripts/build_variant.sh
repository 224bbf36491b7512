#!/bin/bash
# build an experiment variant of the library: scripts/build_variant.sh NAME "-DFOO=1 ..."
set -e -o pipefail
cd "$(dirname "$0")/.."
NAME=$1; DEFS=$2
OBJ=paper_2507_19427_b200/_obj_$NAME; mkdir -p $OBJ
for f in paper_2507_19427_b200/csrc/*.cu paper_2507_19427_b200/csrc/*.cpp; do
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 --expt-relaxed-constexpr -Xcompiler -fPIC -I include $DEFS -c $f -o $OBJ/$(basename $f).o &
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2507_19427_b200/libafdk_$NAME.so $OBJ/*.o -cudart static -lrt -ldl -lpthread
rm -rf $OBJ
echo paper_2507_19427_b200/libafdk_$NAME.so
