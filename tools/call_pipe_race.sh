# racecheck / memcheck of loss_pipe_kernel (alone: V = 262,144; split tail rows) + loss parity + timing
set -u
O=gpurun_out/${1:-piperace}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loss.py -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_loss.py -x -q -k "V262144 or tail_split" > $O/racecheck.txt 2>&1; echo "exit $?" >> $O/racecheck.txt
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_loss.py -x -q -k "V262144 or tail_split" > $O/memcheck.txt 2>&1; echo "exit $?" >> $O/memcheck.txt
TT_LOSS_VARIANT=0 timeout 120 python tools/timeloss.py > $O/time.txt 2>&1
timeout 120 python tools/timeloss.py >> $O/time.txt 2>&1
echo done
