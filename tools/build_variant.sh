#!/bin/bash
# Build a variant of the native library into exp_libs/<name>.so with extra
# nvcc flags (kernel A/B experiments; tools/ab_libs.sh runs them). The object
# cache is cleared before and after, so flags always take effect and the
# in-tree library is rebuilt from the plain sources by the next build().
#   tools/build_variant.sh <name> "<nvcc flags>"
set -e
mkdir -p exp_libs
rm -rf paper_1904_05717_b200/build
TILEMUL_B200_NVFLAGS="$2" python -c "from paper_1904_05717_b200 import build as B; B.build()" >/dev/null
cp paper_1904_05717_b200/lib/libtilemul_b200.so exp_libs/$1.so
rm -rf paper_1904_05717_b200/build
