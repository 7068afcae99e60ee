#!/bin/bash
# Build a variant of the CUDA library from a patched copy of csrc/ into
# build/variants/<name>/liblorbpano_b200.so (A/B experiments; the product
# build is untouched). usage: variant.sh NAME 'sed-expression' FILE [...]
set -e
ROOT="$(cd "$(dirname "$0")/.." && pwd)"
NAME=$1; shift
D=$ROOT/build/variants/$NAME
rm -rf $D && mkdir -p $D/csrc
cp $ROOT/paper_1810_03988_b200/csrc/* $D/csrc/
while [ $# -ge 2 ]; do sed -i "$1" $D/csrc/$2; shift 2; done
FLAGS="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo --fmad=false -std=c++17 -I$ROOT/include -Xcompiler -fPIC,-ffp-contract=off -Xcudafe --diag_suppress=177"
for f in capi lorb match homography compositor; do nvcc $FLAGS -c $D/csrc/$f.cu -o $D/$f.o & done; wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $D/liblorbpano_b200.so $D/*.o
echo $D/liblorbpano_b200.so
