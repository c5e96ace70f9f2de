#!/bin/bash
# Kernel-variant experiments (not the product): builds csrc/ with extra -D flags into
# build_variants/lib_<name>.so; load it with DCAT_LIB_PATH=build_variants/lib_<name>.so.
# usage: tools/build_variant.sh <name> "<nvcc flags>"
set -e
ROOT=$(cd "$(dirname "$0")/.." && pwd)
V=$ROOT/paper_2507_12704_b200/_vb_$1
mkdir -p "$V" "$ROOT/build_variants"
cp "$ROOT"/paper_2507_12704_b200/csrc/*.cu "$ROOT"/paper_2507_12704_b200/csrc/*.cuh "$ROOT"/paper_2507_12704_b200/csrc/*.h "$ROOT"/paper_2507_12704_b200/csrc/*.hpp "$ROOT"/paper_2507_12704_b200/csrc/Makefile "$V"/
make -s -C "$V" EXTRA="$2" OUT="$ROOT/build_variants/lib_$1.so"
