#!/bin/bash
# dev helper: build the library with extra nvcc flags into lib/ab/<name>.so
#   tools/dev/build_variant.sh <name> "-DGR_PIX_NP_BIG=6 -DGR_PIX_NC_BIG=6"
set -e
name=$1; shift
GR_NVCC_EXTRA="$*" python -c "from paper_2402_16801_b200 import _build; _build.build(force=True)"
mkdir -p paper_2402_16801_b200/lib/ab
cp paper_2402_16801_b200/lib/libgridrogue_b200.so paper_2402_16801_b200/lib/ab/$name.so
echo "built lib/ab/$name.so ($*)"
