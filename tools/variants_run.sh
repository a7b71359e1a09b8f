# Time configs under each experiment build of libicv (made by `make variant`).
#   bash tools/variants_run.sh "cfg4 cfg2" OUT suffix...   (suffix "base" = libicv.so)
CFGS=$1; OUT=$2; shift 2
for v in "$@"; do
  lib=$PWD/paper_1907_02129_b200/_lib/libicv_$v.so
  [ "$v" = "base" ] && lib=$PWD/paper_1907_02129_b200/_lib/libicv.so
  echo "== $v" >> $OUT
  ICV_LIB=$lib ICV_NO_GATE=1 timeout 300 python tools/time_conv.py $CFGS >> $OUT 2>&1
done
