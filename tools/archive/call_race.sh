set -u
O=gpurun_out/${1:-race}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 1500 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_attn.py -x -q -k "one_partial_block or exactly_128" > $O/attn_racecheck.txt 2>&1; echo "exit $?" >> $O/attn_racecheck.txt
timeout 900 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_loss.py -x -q -k "small_vocab" > $O/loss_racecheck.txt 2>&1; echo "exit $?" >> $O/loss_racecheck.txt
echo done
