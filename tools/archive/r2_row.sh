# forward softmax layout A/B: one thread per row (TT_FWD_ROW=1, shipped) vs per (row, half) (0)
set -u
O=gpurun_out/${1:-r2row}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for r in 1 2; do echo "== ROW=1 run $r" >> $O/time.txt; timeout 300 python tools/timeall.py agentic8k deep32k wide batch64k >> $O/time.txt 2>&1; done
for c in deep32k batch64k agentic8k; do timeout 120 python tools/attn_power.py $c row1 >> $O/power.txt 2>&1; done
TT_EXTRA_NVCC_FLAGS="-DTT_FWD_ROW=0" python -m paper_2511_00413_b200.build --dev --force > $O/build0.log 2>&1
for r in 1 2; do echo "== ROW=0 run $r" >> $O/time.txt; timeout 300 python tools/timeall.py agentic8k deep32k wide batch64k >> $O/time.txt 2>&1; done
for c in deep32k batch64k agentic8k; do timeout 120 python tools/attn_power.py $c row0 >> $O/power.txt 2>&1; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
