# final check B: synccheck re-run after the dp_free fix, attention parity, bench lines (driver-style),
# reference arm, launch list, ncu --set full of tree 0
set -u
O=gpurun_out/${1:-r2fb}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_attn.py -x -q -k "one_partial_block or exactly_128 or fused_sqnorm" > $O/attn_synccheck.txt 2>&1; echo "exit $?" >> $O/attn_synccheck.txt
timeout 900 compute-sanitizer --tool synccheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_weights.py -x -q -k "unit_weights or weighted_bwd" > $O/weights_synccheck.txt 2>&1; echo "exit $?" >> $O/weights_synccheck.txt
timeout 1500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_random_sweep.py tests/test_gpu_weights.py tests/test_gpu_multirank_bench.py -m gpu -q > $O/pytest_attn.log 2>&1; echo "pytest exit $?" >> $O/pytest_attn.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
for c in agentic8k deep32k wide; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_batch64k.csv \
  python bench.py --trees 4 --steps 1 --warmup 3 --no-extras > /dev/null 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' --launch-skip 12 --launch-count 4 \
  -o $O/full_batch64k -f python bench.py --trees 1 --steps 1 --warmup 3 --no-extras > $O/ncu_full.log 2>&1
echo done > $O/done.txt
