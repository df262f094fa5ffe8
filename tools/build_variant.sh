#!/bin/bash
# Build a copy of the package with extra nvcc -D flags into _variants/<name>/ (untracked).
#   tools/build_variant.sh name "-DWASABI_KD=8 -DWASABI_MINB=5" [name2 "defs2" ...]
# Time them on the GPU with tools/prof_superpose.py --pkg _variants/<name>.
set -e
cd "$(dirname "$0")/.."
mkdir -p _variants
while [ $# -ge 2 ]; do
  n=$1; defs=$2; shift 2
  rm -rf _variants/$n; mkdir -p _variants/$n
  cp -r paper_1708_04233_b200 include _variants/$n/
  rm -rf _variants/$n/paper_1708_04233_b200/*.so _variants/$n/paper_1708_04233_b200/build
  (cd _variants/$n && WASABI_NVCC_DEFS="$defs" python -c "import paper_1708_04233_b200.build as B; B.build()" 2>&1 \
     | grep -E "error|spill" | sed "s/^/[$n] /" | cut -c1-160) || true
done
