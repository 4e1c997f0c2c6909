#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/u.jsonl; : > $O
for v in base db2 db3 base db2 db3; do
  if [ "$v" = base ]; then unset SSD_B200_LIB; else export SSD_B200_LIB=$PWD/paper_2603_03251_b200/libssd_b200_$v.so; fi
  SSD_B200_PROFILE_PART=s timeout 120 python scripts/fwd_ablate.py d5,d20 | sed "s/\"env\"/\"lib\": \"$v\", \"env\"/" >> $O 2>&1
  timeout 120 python scripts/round_profile.py | sed "s/\"env\"/\"lib\": \"$v\", \"env\"/" >> $O 2>&1
done
cat $O
