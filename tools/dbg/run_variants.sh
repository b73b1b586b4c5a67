#!/bin/bash
# on the GPU box: run CMD with each variant library swapped in:  tools/dbg/run_variants.sh "CMD" base v1 v2 ...
cmd=$1; shift
lib=paper_2104_10949_b200/libmpc3b200.so
cp $lib /tmp/lib_base.so
for v in "$@"; do
  if [ "$v" = base ]; then cp /tmp/lib_base.so $lib; else cp tools/dbg/variants/lib_$v.so $lib; fi
  echo "== $v"; eval "$cmd"
done
cp /tmp/lib_base.so $lib
