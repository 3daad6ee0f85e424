#!/bin/bash
O=gpurun_out/lprof; mkdir -p $O
for v in 1 2 3; do TT_LOSS_DEBUG=1 TT_LOSS_VARIANT=$v timeout 120 python tools/timeloss.py > $O/dbg_$v.txt 2>&1; done
TT_LOSS_VARIANT=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:loss_cluster --launch-skip 3 --launch-count 1 -o $O/lc -f python tools/timeloss.py > $O/ncu.log 2>&1
