#!/bin/bash
cd "$(dirname "$0")/.."
for acl in 0 1; do echo "ATTN_CL=$acl"; SSD_B200_ATTN_CL=$acl timeout 300 python scripts/pf_sweep.py 16 2>&1 | tail -1; done
timeout 900 python -m pytest tests -m gpu -q -x --timeout 800 -p no:cacheprovider -rf 2>&1 | tail -3
