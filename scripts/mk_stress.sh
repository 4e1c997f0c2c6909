#!/bin/bash
cd "$(dirname "$0")/.."
for args in "tiny 40 1024" "tiny 40 512" "tiny 8 1024"; do
  fails=0
  for i in 1 2 3 4; do
    timeout 60 python scripts/mk_one.py $args > /tmp/one.log 2>&1 || { fails=$((fails+1)); tail -2 /tmp/one.log; }
  done
  echo "$args: $fails/4 failed"
done
