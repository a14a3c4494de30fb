for lib in paper_2112_10065_b200/libbpx.so ./ab_FNOMMA.so ./ab_FNOCONV.so ./ab_FTMA.so; do
  echo "== $lib"
  for op in fwd dgrad; do
  BPX_LIB=$lib timeout 300 python tools/layer_bench.py --op $op 2>&1 | grep -E "conv1_2|conv2_2|conv3_2|conv4_2|conv5_2|rror" | cut -c1-200
  done
done
