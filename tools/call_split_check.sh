# loss split: parity (all loss tests incl. capture), then memcheck / synccheck / racecheck of the split path
set -u
O=gpurun_out/${1:-splitchk}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_loss.py tests/test_gpu_lmhead.py -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_loss.py -x -q -k "tail_split or kernel_paths or capture" > $O/split_$tool.txt 2>&1; echo "exit $?" >> $O/split_$tool.txt
done
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_loss.py -x -q -k "tail_split or kernel_paths or capture" > $O/split_racecheck.txt 2>&1; echo "exit $?" >> $O/split_racecheck.txt
echo done
