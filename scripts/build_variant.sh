#!/bin/bash
# Build an A/B variant of the C-ABI library with extra nvcc flags:
#   scripts/build_variant.sh NAME "-DPC_X=0 ..."
# -> paper_2109_09056_b200/libparticula_b200_NAME.so (load it with
#    PARTICULA_B200_LIB=libparticula_b200_NAME.so; same ABI as the default build)
set -e
R=$(cd "$(dirname "$0")/.." && pwd)
T=/tmp/pcvar_$1
rm -rf "$T"; mkdir -p "$T/pkg/csrc" "$T/include"
cp "$R"/paper_2109_09056_b200/csrc/*.cu "$R"/paper_2109_09056_b200/csrc/*.cuh \
   "$R"/paper_2109_09056_b200/csrc/Makefile "$T/pkg/csrc/"
cp "$R"/include/*.h "$R"/include/*.cuh "$T/include/" 2>/dev/null || true
make -C "$T/pkg/csrc" -j8 EXTRA="$2" > "$T/build.log" 2>&1 || { tail -20 "$T/build.log"; exit 1; }
cp "$T/pkg/libparticula_b200.so" "$R/paper_2109_09056_b200/libparticula_b200_$1.so"
echo "built libparticula_b200_$1.so ($2)"
