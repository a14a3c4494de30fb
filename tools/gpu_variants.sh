# Build the library with each -D variant in turn and time one layer/op.
# usage: bash tools/gpu_variants.sh "<layer> <op>" "-DA=1" "-DB=2" ...
LO=$1; shift
for v in "" "$@"; do
  echo "== variant: '$v'"
  BPX_NVCC_EXTRA="$v" python -c "from paper_2112_10065_b200 import build; build.build(force=True)" 2>&1 | grep -i error
  for l in $LO; do :; done
  timeout 120 python tools/layer_bench.py $LO | grep -v "^\[{" | head -20
done
