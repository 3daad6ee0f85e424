# final check A: full GPU suite, smoke, compute-sanitizer over the backward changes (V in TMEM, fold, walk)
set -u
O=gpurun_out/${1:-r2fa}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=15 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
for tool in memcheck racecheck synccheck; do
  extra=""; [ $tool = racecheck ] && extra="--racecheck-report hazard"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_attn.py -x -q -k "one_partial_block or exactly_128 or fused_sqnorm" > $O/attn_$tool.txt 2>&1; echo "exit $?" >> $O/attn_$tool.txt
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_weights.py -x -q -k "unit_weights or attention" > $O/weights_$tool.txt 2>&1; echo "exit $?" >> $O/weights_$tool.txt
done
echo done > $O/done.txt
