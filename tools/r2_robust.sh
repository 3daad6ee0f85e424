# robustness of the persistent kernels: multi-item forest tests (x3 runs), extended random sweep
set -u
O=gpurun_out/${1:-r2u}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
for r in 1 2 3; do
  timeout 900 python -m pytest tests/test_gpu_persistent.py -m gpu -q > $O/persistent_$r.log 2>&1; echo "exit $?" >> $O/persistent_$r.log
done
TT_SWEEP_SCALE=8 timeout 2400 python -m pytest tests/test_gpu_random_sweep.py -m gpu -q -k "attention" > $O/random_sweep_x8.log 2>&1; echo "exit $?" >> $O/random_sweep_x8.log
echo done > $O/done.txt
