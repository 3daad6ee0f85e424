set -u
O=gpurun_out/${1:-sanitize}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for tool in memcheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_attn.py -x -q -k "agentic1500_mha or one_partial_block or forest_zero_len" > $O/attn_$tool.txt 2>&1; echo "exit $?" >> $O/attn_$tool.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_loss.py -x -q -k "small_vocab or many_continuations" > $O/loss_$tool.txt 2>&1; echo "exit $?" >> $O/loss_$tool.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_block.py tests/test_gpu_lmhead.py -x -q -k "agentic700 or restore_grad" > $O/misc_$tool.txt 2>&1; echo "exit $?" >> $O/misc_$tool.txt
done
echo done
