#!/bin/bash
# Build a compile-time variant of the library into variants/<name>/ (git-
# ignored, travels with gpurun); select it with MKNN_LIB=variants/<name>/libmknn_b200.so.
# usage: tools/build_variant.sh <name> "<nvcc flags, e.g. -DMKNN_BS_U=1>"
set -e
cd "$(dirname "$0")/.."
name=$1; flags=$2
rm -rf variants/$name && mkdir -p variants/$name/a/b
cp -r paper_1412_6170_b200/csrc variants/$name/a/b/csrc && rm -rf variants/$name/a/b/csrc/build
mkdir -p variants/$name/a/include && cp include/mknn_b200.h variants/$name/a/include/
make -s -j4 -C variants/$name/a/b/csrc EXTRA="$flags" OUT=$PWD/variants/$name/libmknn_b200.so
rm -rf variants/$name/a
