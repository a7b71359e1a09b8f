#!/bin/bash
# Time the conv kernel of each config for every libicv variant present in _lib/.
cd "$(dirname "$0")/.."
for lib in paper_1907_02129_b200/_lib/libicv*.so; do
  case "$lib" in *stats*) continue;; esac
  echo "== $lib"
  case "$lib" in *_no*) export ICV_NO_GATE=1;; *) unset ICV_NO_GATE;; esac
  ICV_LIB=$PWD/$lib timeout -s KILL 120 python tools/time_conv.py "$@" || echo "FAILED rc=$?"
done
