set -u
O=gpurun_out/${1:-lossv}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for v in ${VARS}; do
  echo "== TT_LOSS_VARIANT=$v" >> $O/loss.txt
  TT_LOSS_VARIANT=$v timeout 600 python -m pytest tests/test_gpu_loss.py tests/test_gpu_random_sweep.py -x -q -k "loss" 2>&1 | tail -1 >> $O/loss.txt
  TT_LOSS_VARIANT=$v timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
  TT_LOSS_VARIANT=$v timeout 120 python tools/timeloss.py >> $O/loss.txt 2>&1
done
echo done
