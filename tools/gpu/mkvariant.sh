#!/bin/bash
# Build a whole-library A/B variant: tools/gpu/mkvariant.sh NAME "-DFLAG=1 ..."
# -> paper_2101_08825_b200/_variants/NAME/libmollifem_b200.so (git-ignored,
# travels with gpurun; tools/ab_time.py / tools/gpu/ab.sh load it through
# MF_LIB_PATH)
set -e
cd "$(dirname "$0")/../../paper_2101_08825_b200/csrc"
V=../_variants/$1
mkdir -p $V/build
make -s -j8 BUILD=$V/build OUT=$V/libmollifem_b200.so EXTRA="$2"
echo "built $V"
