# bwd CTA-pair dQ pre-reduction (DSMEM) A/B: parity (shipped: pairs on head-major trees) + sustained power
set -u
O=gpurun_out/${1:-r2pq}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
timeout 600 python tools/timeall.py deep32k > $O/smoke_time.txt 2>&1; echo "exit $?" >> $O/smoke_time.txt
timeout 1500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py tests/test_gpu_multirank_bench.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for r in 1 2; do for c in deep32k batch64k; do
  TT_BWD_PAIRQ=1 timeout 120 python tools/attn_power.py $c pairq1 >> $O/power.txt 2>&1
  TT_BWD_PAIRQ=0 timeout 120 python tools/attn_power.py $c pairq0 >> $O/power.txt 2>&1
done; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/power.txt
