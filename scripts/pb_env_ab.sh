#!/bin/bash
# PB sweep time under environment settings: scripts/pb_env_ab.sh "<configs>" "ENV=.. ENV=.." ...
cfgs="$1"; shift
for c in $cfgs; do
  for envs in "$@"; do
    echo "== [$envs] cfg$c"
    env $envs GEOMS=${GEOMS:-13:21} PB_ONLY=1 timeout -s KILL 300 python scripts/pb_probe.py $c 2>&1 | grep -v "^$" | sed 's/; per-iter.*//' | tail -1
  done
done
