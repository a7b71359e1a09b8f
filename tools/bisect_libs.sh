# Time cfg5 layers with alternative builds of libicv (debug / experiment
# variants made by `make -C paper_1907_02129_b200/csrc variant NAME=...`).
#   bash tools/bisect_libs.sh LAYERS OUT lib_suffix...
L=$1; OUT=$2; shift 2
for v in "$@"; do
  [ "$v" = "base" ] && v=""
  echo "== lib$v" >> $OUT
  ICV_LIB=$PWD/paper_1907_02129_b200/_lib/libicv$v.so timeout 300 python tools/ab_knob.py $L pdl 1 >> $OUT 2>&1
done
