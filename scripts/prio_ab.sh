#!/bin/bash
cd "$(dirname "$0")/.."
for pr in 0 1; do echo "SPEC_PRIO=$pr"; SSD_B200_SPEC_PRIO=$pr timeout 300 python scripts/pf_sweep.py 16 2>&1 | tail -1 | grep -o "SSD=.*"; done
