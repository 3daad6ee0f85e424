set -u
O=gpurun_out/${1:-pers}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_attn.py -x -q -k "bf16_tensor_core and agentic1500" > $O/smoke_test.txt 2>&1; echo "exit $?" >> $O/smoke_test.txt
if grep -q "passed" $O/smoke_test.txt && ! grep -q failed $O/smoke_test.txt; then
  timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_weights.py tests/test_gpu_block.py tests/test_gpu_plan.py tests/test_gpu_random_sweep.py -x -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
  timeout 300 python tools/timeall.py deep32k agentic8k wide > $O/time.txt 2>&1
fi
echo done
