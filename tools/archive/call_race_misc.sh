# racecheck of the LM-head, RoPE / Gradient Scaler, block and weights paths
set -u
O=gpurun_out/${1:-racemisc}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 2000 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_block.py tests/test_gpu_lmhead.py tests/test_gpu_weights.py -x -q -k "agentic700 or restore_grad or rope or term_boundary or weights" > $O/misc_racecheck.txt 2>&1; echo "exit $?" >> $O/misc_racecheck.txt
echo done
