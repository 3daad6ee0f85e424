# bwd probe: parity tests, ablations (TT_DEBUG_BWD 1 = skip dQ reduce, 4 = skip elementwise math, 5 = both) and role counters
set -u
O=gpurun_out/${1:-bwdprobe}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_weights.py -x -q > $O/pytest.txt 2>&1; echo "exit $?" >> $O/pytest.txt
for d in ${DBGS:-0 1 4 5}; do echo "dbg=$d"; TT_DEBUG_BWD=$d timeout 120 python tools/timeall.py deep32k agentic8k wide 2>&1; done > $O/ablate.txt
TT_PROFILE_COUNTERS=1 python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
timeout 300 python tools/bwdcount.py > $O/counters.txt 2>&1
echo done
