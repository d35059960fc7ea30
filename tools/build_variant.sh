#!/bin/bash
# Build a variant of the library with extra nvcc flags into _lib/variants/<name>.so
#   tools/build_variant.sh <name> "<EXTRA_NVFLAGS>"
set -e
HERE=$(cd "$(dirname "$0")/.." && pwd)
name=$1; flags=$2
out=$HERE/paper_1811_01110_b200/_lib/variants/$name.so
make -s -C $HERE/paper_1811_01110_b200/csrc -j8 OUT=$out OBJDIR=$HERE/paper_1811_01110_b200/_lib/variants/obj_$name EXTRA_NVFLAGS="$flags" >/dev/null
echo $out
