set -u
O=gpurun_out/${1:-redv4}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
TT_DEBUG_BWD=64 timeout 600 python -m pytest tests/test_gpu_attn.py -x -q -k "bf16_tensor_core or fused_sqnorm or full_size" > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
for d in 0 64; do echo "dbg=$d"; TT_DEBUG_BWD=$d timeout 200 python tools/timeall.py deep32k agentic8k wide 2>&1; done > $O/time.txt
echo done
