set -u
O=gpurun_out/${1:-poly}; mkdir -p $O
for f in "-DTT_FWD_POLY=1 -DTT_BWD_POLY=1" "-DTT_FWD_POLY=2 -DTT_BWD_POLY=2" "-DTT_FWD_POLY=0 -DTT_BWD_POLY=0"; do
  echo "== $f" >> $O/sweep.txt
  TT_EXTRA_NVCC_FLAGS="$f" python -m paper_2511_00413_b200.build --force > $O/build.log 2>&1
  timeout 200 python tools/timeall.py deep32k agentic8k wide >> $O/sweep.txt 2>&1
done
echo done
