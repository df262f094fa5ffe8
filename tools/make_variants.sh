#!/bin/bash
# Build superpose variants into _variants/<name>/ (untracked): each is a copy of the package with
# sed edits applied to kernels_superpose.cu, built in place.  Usage:
#   tools/make_variants.sh name1 'sed-expr1' name2 'sed-expr2' ...
# Time them on the GPU with tools/prof_superpose.py --pkg _variants/<name>.
set -e
cd "$(dirname "$0")/.."
mkdir -p _variants
while [ $# -ge 2 ]; do
  n=$1; e=$2; shift 2
  rm -rf _variants/$n; mkdir -p _variants/$n
  cp -r paper_1708_04233_b200 include _variants/$n/
  rm -rf _variants/$n/paper_1708_04233_b200/*.so _variants/$n/paper_1708_04233_b200/build
  K=_variants/$n/paper_1708_04233_b200/csrc/kernels_superpose.cu
  case "$e" in
    file:*) cp "${e#file:}" "$K" ;;      # whole-file variant
    *) sed -i "$e" "$K" ;;
  esac
  (cd _variants/$n && python -c "import paper_1708_04233_b200.build as B; B.build()" 2>&1 | grep -E "error|spill" | sed "s/^/[$n] /" | cut -c1-160) || true
done
