#!/bin/bash
# Dev tool: build compile-time variants of the library into build/variants/
# (name:flags pairs), for tests/emu/variants.py.  build/ is git-ignored but
# travels to the GPU box with gpurun.
set -e
cd "$(dirname "$0")/../../paper_2309_03912_b200/csrc"
mkdir -p ../../build/variants
for spec in "$@"; do
  name="${spec%%:*}"; flags="${spec#*:}"
  /usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 --extended-lambda -O3 \
    -lineinfo -Xcompiler -fPIC -shared -diag-suppress 550,177 $flags \
    -o ../../build/variants/libexs_$name.so exspace_b200.cu 2>&1 | grep -v "deprecated\|CountingInputIterator\|^ *[0-9]* |\|^ *|\|note: declared" || true
  echo "built $name ($flags)"
done
