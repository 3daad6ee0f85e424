set -u
O=gpurun_out/${1:-ktmem}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_weights.py -x -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
echo "== default" > $O/time.txt; timeout 200 python tools/timeall.py deep32k agentic8k wide >> $O/time.txt 2>&1
TT_EXTRA_NVCC_FLAGS="${ALT:--DTT_BWD_KTMEM=0}" python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
echo "== ALT $ALT" >> $O/time.txt; timeout 200 python tools/timeall.py deep32k agentic8k wide >> $O/time.txt 2>&1
echo done
