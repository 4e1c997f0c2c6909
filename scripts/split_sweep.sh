#!/bin/bash
cd "$(dirname "$0")/.."
for sp in 148,148 100,48 84,64 74,74 64,84; do
  echo "SPLIT=$sp"; SSD_B200_SPLIT_SMS=$sp timeout 300 python scripts/pf_sweep.py 16 2>&1 | tail -1 | grep -o "SSD=.*"
done
