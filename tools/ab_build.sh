#!/bin/bash
# Builds an A/B variant of libtexforge_cuda.so: tools/ab/lib_NAME.so with
# extra nvcc flags (e.g. -DTFG_SOMETHING=1). Select it at run time with
# TEXFORGE_CUDA_LIB=$PWD/tools/ab/lib_NAME.so (tools/ab_sweep.sh does that).
# Usage: bash tools/ab_build.sh NAME "-DFOO=1 -DBAR=2"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
mkdir -p $ROOT/tools/ab
make -s -j8 -C $ROOT/paper_1710_06189_b200/csrc OUT=$ROOT/tools/ab/lib_$name.so OBJ=$ROOT/tools/ab/build_$name \
  EXTRA_NVFLAGS="$*" 2>&1 | grep -i "error" || true
ls -la $ROOT/tools/ab/lib_$name.so
