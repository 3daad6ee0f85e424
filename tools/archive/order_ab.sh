#!/bin/bash
# A/B of the CTA orders (TT_CTA_ORDER bit0 fwd head-major, bit1 bwd head-major)
O=gpurun_out/ab; mkdir -p $O
for m in 0 1 2 3; do
  echo "== TT_CTA_ORDER=$m" >> $O/order.txt
  TT_CTA_ORDER=$m timeout 300 python tools/timeall.py agentic8k deep32k wide >> $O/order.txt 2>&1
done
