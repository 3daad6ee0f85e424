set -u
O=gpurun_out/${1:-r2z}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_persistent.py -m gpu -q > $O/persistent.log 2>&1; echo "exit $?" >> $O/persistent.log
echo done > $O/done.txt
