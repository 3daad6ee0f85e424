# boundary-mode fix check: loss/lmhead/sweep (incl. extended sweep) + loss diag on the failing seeds
set -u
O=gpurun_out/bfix; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loss.py tests/test_gpu_lmhead.py tests/test_gpu_weights.py tests/test_gpu_random_sweep.py -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
TT_SWEEP_SCALE=8 timeout 900 python -m pytest tests/test_gpu_random_sweep.py -q -k loss > $O/sweep8.txt 2>&1; echo "exit $?" >> $O/sweep8.txt
timeout 300 python tools/loss_diag.py 35 47 83 > $O/diag.txt 2>&1
echo done
