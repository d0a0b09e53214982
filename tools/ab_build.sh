#!/usr/bin/env bash
# Build a variant of libmetro_b200.so with extra nvcc flags into abtest/lib<NAME>.so
# (A/B timing: tools/ab_libs.sh).  ./tools/ab_build.sh B "-DSOME_VARIANT_FLAG"
set -eu
name=$1; shift
out=$PWD/abtest/build_$name
make -s -j8 -C paper_2512_09277_b200/csrc OUTDIR="$out" EXTRA="$*" > /dev/null
cp "$out/libmetro_b200.so" "abtest/lib$name.so"
echo "abtest/lib$name.so <- EXTRA=$*"
