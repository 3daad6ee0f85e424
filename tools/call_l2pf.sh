# next-CTA L2 prefetch A/B (TT_L2_PREFETCH=0 disables) on attention fwd / bwd + attention parity
set -u
O=gpurun_out/${1:-l2pf}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py -q -k "not loss" > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
for r in 1 2; do
  for v in 0 1; do
    echo "== TT_L2_PREFETCH=$v (round $r)" >> $O/time.txt
    TT_L2_PREFETCH=$v timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
  done
done
echo done
