#!/bin/bash
# A/B of propagation-blocked builds: scripts/pb_ab.sh "<configs>" v1 v2 ...
# (v = a pbvariant name under paper_2203_09284_b200/csrc/build, or "main")
cfgs="$1"; shift
for c in $cfgs; do
  for v in "$@"; do
    if [ "$v" = main ]; then lib=""; else lib=paper_2203_09284_b200/csrc/build/libfpr_b200_$v.so; fi
    echo "== $v cfg$c"
    FPR_B200_LIB=$lib GEOMS=${GEOMS:-13:21} PB_ONLY=1 timeout -s KILL 300 python scripts/pb_probe.py $c 2>&1 | grep -v "^$" | sed 's/; per-iter.*//' | tail -2
  done
done
