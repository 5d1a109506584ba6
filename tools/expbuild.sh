#!/bin/bash
# Kernel-experiment build: tools/expbuild.sh NAME K "EXTRA NVCC FLAGS"
# Rebuilds only the apply translation units (one 3D degree K, fp64) with the
# extra flags and links _exp/NAME/libdgx.so against the regular objects
# of build/obj (run `make -C paper_1711_03590_b200/csrc` first). Load it with
# DGX_LIB=_exp/NAME/libdgx.so (bench.py / tests).
set -e
NAME=$1; K=$2; shift 2; EXTRA="$*"
ROOT=$(cd "$(dirname "$0")/.." && pwd)
SRC=$ROOT/paper_1711_03590_b200/csrc
OUT=$ROOT/_exp/$NAME
mkdir -p $OUT
FL="-std=c++17 -O3 -lineinfo -gencode arch=compute_100a,code=sm_100a -Xcompiler -fPIC,-ffp-contract=off -Xptxas -warn-spills --expt-relaxed-constexpr -DDGX_DEV_K=$K $EXTRA"
for f in sipg sipg_gl sipg_gauss sipg_hermite; do
  /usr/local/cuda/bin/nvcc $FL -c $SRC/$f.cu -o $OUT/$f.o &
done
wait
OBJ=$ROOT/build/obj
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $OUT/libdgx.so \
  $OBJ/setup.o $OBJ/capi.o $OBJ/geometry.o $OBJ/operator.o $OBJ/advection.o $OBJ/exchange.o \
  $OBJ/nccl_exchange.o $OBJ/solvers.o $OUT/sipg.o $OUT/sipg_gl.o $OUT/sipg_gauss.o $OUT/sipg_hermite.o -ldl
echo built $OUT/libdgx.so
