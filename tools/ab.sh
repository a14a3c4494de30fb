# A/B timing on one box: BPX_LIB=<a.so> vs <b.so>, layer_bench args after --
# usage: bash tools/ab.sh a.so b.so [layer_bench args]
A=$1; B=$2; shift 2
for lib in "$A" "$B"; do
  echo "== $lib"
  BPX_LIB=$lib timeout 300 python tools/layer_bench.py "$@" | grep -v "^\[{"
done
