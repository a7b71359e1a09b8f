L=s1b1_1x1a,s1b1_1x1b,s2b2_1x1b,s3b2_1x1a,s3b2_1x1b,s4b2_1x1a,s1b1_3x3,s3b2_3x3
for v in "" _noepi _nomma _none; do
  echo "== lib$v" >> gpurun_out/bis13.log
  ICV_LIB=$PWD/paper_1907_02129_b200/_lib/libicv$v.so timeout 300 python tools/ab_knob.py $L pdl 1 >> gpurun_out/bis13.log 2>&1
done
timeout 120 python tools/repro_layer.py s3b2_1x1a 256 dense_cs=2 win_debug=1 >> gpurun_out/bis13.log 2>&1
timeout 120 python tools/repro_layer.py s3b2_1x1a 256 dense_cs=1 win_debug=1 >> gpurun_out/bis13.log 2>&1
