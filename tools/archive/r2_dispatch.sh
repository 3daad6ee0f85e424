# bwd dispatch (persistent kernel for short items, flat kernel for long ones): parity of both paths, same-box
# A/B against the round-2-start build (ab_old), forced-kernel A/B (dev TT_BWD_FLAT=0/1)
set -u
O=gpurun_out/${1:-r2r}; mkdir -p $O
python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
(cd ab_old && python -m paper_2511_00413_b200.build --force > ../$O/build_old.log 2>&1)
timeout 1500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_persistent.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py tests/test_gpu_block.py tests/test_gpu_multirank_bench.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for r in 1 2; do
  for d in /root/repo /root/repo/ab_old; do
    TT_ROOT=$d timeout 300 python tools/timeab.py batch64k deep32k:1 deep32k:0 agentic8k wide >> $O/time.txt 2>&1
  done
done
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
for f in 0 1; do echo "== TT_BWD_FLAT=$f" >> $O/time_flat.txt; TT_BWD_FLAT=$f timeout 300 python tools/timeab.py agentic8k wide deep32k:0 >> $O/time_flat.txt 2>&1; done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/time.txt
