mkdir -p gpurun_out
: > gpurun_out/exp20.log
for v in lbw16 nt512lbw16 nt512; do
  for c in "c1 1024" "c4 1024"; do set -- $c; UG_LIB_OVERRIDE=build_variants/libunigpu_$v.so OPS=utf8_to_utf16le,utf16le_to_utf8 timeout 300 python tools/opbench.py $1 $2 10 >> gpurun_out/exp20.log 2>&1; done
done
