#!/bin/bash
# Same-box A/B of build variants: bash tools/ab_variants.sh "<layer_bench args>" lib1 lib2 ...
ARGS=$1; shift
for lib in "$@"; do
  echo "== $lib"
  BPX_LIB=$lib timeout 300 python tools/layer_bench.py $ARGS 2>&1 | grep -vE "^\[\{" | cut -c1-200
done
