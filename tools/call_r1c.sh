set -u
O=gpurun_out/r1c; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 120 ./tools/mma_rate.bin > $O/mma_rate.txt 2>&1
timeout 600 python bench.py --config batch64k --trees 4 --steps 3 --no-e2e --no-cpu > $O/bench_b4.json 2> $O/bench_b4.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster' \
  --launch-skip 9 --launch-count 3 -o $O/full_agentic8k -f \
  python bench.py --steps 1 --warmup 3 --no-cpu --no-e2e --no-linear > $O/ncu_full.log 2>&1
echo done
