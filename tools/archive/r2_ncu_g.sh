# persistent kernels: fwd sub-diagonal mask A/B (dev TT_DEBUG_FWD=128 = full test on every partial tile),
# launch list of the default bench, ncu --set full of the attention / loss kernels on batch64k tree 0,
# agentic8k, deep32k, wide
set -u
O=gpurun_out/${1:-r2n}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build_dev.log 2>&1
timeout 600 python -m pytest tests/test_gpu_attn.py tests/test_gpu_persistent.py -m gpu -x -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
for r in 1 2; do
  echo "== sub-diagonal fast mask" >> $O/time.txt; timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
  echo "== full mask" >> $O/time.txt; TT_DEBUG_FWD=128 timeout 300 python tools/timeall.py agentic8k wide deep32k >> $O/time.txt 2>&1
done
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_batch64k.csv \
  python bench.py --trees 4 --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' --launch-skip 12 --launch-count 4 \
  -o $O/full_batch64k -f python bench.py --trees 1 --steps 1 --warmup 3 --no-extras > $O/ncu_full.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' \
  --launch-skip 12 --launch-count 4 -o $O/full_agentic8k -f \
  python bench.py --config agentic8k --steps 1 --warmup 3 --no-extras > $O/ncu_a8k.log 2>&1
for c in deep32k wide; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100' \
  --launch-skip 6 --launch-count 2 -o $O/full_$c -f \
  python bench.py --config $c --steps 1 --warmup 3 --no-extras --no-loss > $O/ncu_$c.log 2>&1
done
echo done > $O/done.txt
