set -u
O=gpurun_out/${1:-lossgrp}; mkdir -p $O
for g in 256 320 384 448; do
  echo "== group $g" >> $O/loss.txt
  TT_EXTRA_NVCC_FLAGS="-DTT_LOSS_GROUP=$g" python -m paper_2511_00413_b200.build --force > $O/build_$g.log 2>&1 || { echo build failed >> $O/loss.txt; continue; }
  timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
  timeout 300 python -m pytest tests/test_gpu_loss.py -x -q 2>&1 | tail -1 >> $O/loss.txt
done
echo done
