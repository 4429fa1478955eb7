#!/bin/bash
# Build the product library with extra nvcc defines into _lib/variants/<name>.so
# for A/B runs (select with RKMF_LIB_PATH). Usage: tools/build_variant.sh name -DFOO=1 ...
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
name=$1; shift
tmp=$(mktemp -d)
mkdir -p "$tmp/paper_2503_22631_b200" "$ROOT/paper_2503_22631_b200/_lib/variants"
cp -r "$ROOT/paper_2503_22631_b200/csrc" "$tmp/paper_2503_22631_b200/"
rm -rf "$tmp/paper_2503_22631_b200/csrc/build"
ln -s "$ROOT/include" "$tmp/include"
make -s -C "$tmp/paper_2503_22631_b200/csrc" -j8 \
  OUT="$ROOT/paper_2503_22631_b200/_lib/variants/$name.so" \
  NVCC="/usr/local/cuda/bin/nvcc $*" "$ROOT/paper_2503_22631_b200/_lib/variants/$name.so"
rm -rf "$tmp"
echo "built _lib/variants/$name.so"
