# final-build robustness: random attention sweep x32 (2048 forests), loss sweep x8, persistent tests x5
set -u
O=gpurun_out/${1:-r2x}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
TT_SWEEP_SCALE=32 timeout 2400 python -m pytest tests/test_gpu_random_sweep.py -m gpu -q -k "attention" > $O/random_attn_x32.log 2>&1; echo "exit $?" >> $O/random_attn_x32.log
TT_SWEEP_SCALE=8 timeout 2400 python -m pytest tests/test_gpu_random_sweep.py -m gpu -q -k "loss" > $O/random_loss_x8.log 2>&1; echo "exit $?" >> $O/random_loss_x8.log
for r in 1 2 3 4 5; do
  timeout 900 python -m pytest tests/test_gpu_persistent.py -m gpu -q > $O/persistent_$r.log 2>&1; echo "exit $?" >> $O/persistent_$r.log
done
echo done > $O/done.txt
