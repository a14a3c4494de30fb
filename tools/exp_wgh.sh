for lib in paper_2112_10065_b200/libbpx.so ./ab_NOMMA.so ./ab_NOCONV.so ./ab_TMA.so; do
  echo "== $lib"
  BPX_LIB=$lib timeout 300 python tools/layer_bench.py --op wgrad 2>&1 | grep -E "conv1_2|conv2_2|conv3_2|conv4_2|conv5_2|Error|error" | cut -c1-300
done
