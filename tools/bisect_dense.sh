# Bisection of the tensor-core kernels on cfg5 layers: the shipped library vs
# debug builds without the epilogue stores (noepi), without the MMAs (nomma)
# or without both (none) -- make -C paper_1907_02129_b200/csrc variant NAME=...
L=${1:-s1b1_1x1a,s1b1_1x1b,s3b2_1x1a,s3b2_1x1b,s4b2_1x1a,s1b1_3x3,s2b2_3x3,s3b2_3x3,s4b2_3x3,s2b1_3x3}
OUT=${2:-gpurun_out/bisect.log}
for v in "" _noepi _nomma _none; do
  echo "== lib$v" >> $OUT
  ICV_LIB=$PWD/paper_1907_02129_b200/_lib/libicv$v.so timeout 300 python tools/ab_knob.py $L pdl 1 >> $OUT 2>&1
done
