#!/bin/bash
O=gpurun_out/lab; mkdir -p $O; rm -f $O/loss.txt
for v in 1 6 7 8; do
  echo "== TT_LOSS_VARIANT=$v" >> $O/loss.txt
  TT_LOSS_DEBUG=1 TT_LOSS_VARIANT=$v timeout 120 python tools/timeloss.py 2>&1 | sort | uniq >> $O/loss.txt
  TT_LOSS_VARIANT=$v timeout 300 python -m pytest tests/test_gpu_loss.py tests/test_gpu_weights.py -x -q -k "loss" 2>&1 | tail -1 >> $O/loss.txt
done
