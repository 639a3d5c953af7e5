#!/bin/bash
# Time config(s) under every built variant: tools/var_time.sh "c2 c4" v0 v1 ...
cfgs=$1; shift
for v in "$@"; do
  echo "== $v"
  for r in 1 2; do GZ_LIB=build/var/$v/libgzb200.so python tools/quick_time.py $cfgs 2>&1 | grep -v policy; done
done
