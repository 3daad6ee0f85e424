# persistent bwd per-tile cost on long items: K/V copy code inline vs out of line (dev TT_BWD_CP_NOINLINE),
# each against the flat kernel (dev TT_BWD_FLAT=1) on the same box
set -u
O=gpurun_out/${1:-r2t}; mkdir -p $O
for nl in 0 1; do
  TT_EXTRA_NVCC_FLAGS="-DTT_BWD_CP_NOINLINE=$nl" python -m paper_2511_00413_b200.build --dev --force > $O/build_$nl.log 2>&1
  for r in 1 2; do
    for f in 0 1; do
      echo "== noinline=$nl flat=$f" >> $O/time.txt
      TT_BWD_FLAT=$f timeout 300 python tools/timeab.py batch64k deep32k:1 agentic8k >> $O/time.txt 2>&1
    done
  done
done
python -m paper_2511_00413_b200.build --force > /dev/null 2>&1
echo done >> $O/time.txt
