# dQ accumulator layout A/B: [N][hq][d] (default) vs [hq][N][d] (TT_DQ_HND=1): parity under HND, short-burst and
# sustained timing of the backward on the same box (dev builds)
set -u
O=gpurun_out/${1:-r2v}; mkdir -p $O
TT_EXTRA_NVCC_FLAGS="-DTT_DQ_HND=1" python -m paper_2511_00413_b200.build --dev --force > $O/build_hnd.log 2>&1
timeout 900 python -m pytest tests/test_gpu_attn.py tests/test_gpu_persistent.py -m gpu -x -q > $O/pytest_hnd.log 2>&1; echo "exit $?" >> $O/pytest_hnd.log
for r in 1 2; do
  echo "== HND" >> $O/time.txt; timeout 300 python tools/timeab.py batch64k deep32k:1 agentic8k >> $O/time.txt 2>&1
done
TT_SUSTAINED=1 timeout 300 python tools/timeab.py batch64k > $O/sustained_hnd.txt 2>&1
python -m paper_2511_00413_b200.build --dev --force > $O/build_nhd.log 2>&1
for r in 1 2; do
  echo "== NHD" >> $O/time.txt; timeout 300 python tools/timeab.py batch64k deep32k:1 agentic8k >> $O/time.txt 2>&1
done
TT_SUSTAINED=1 timeout 300 python tools/timeab.py batch64k > $O/sustained_nhd.txt 2>&1
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/time.txt
