# final ncu --set full captures of the other configs (agentic8k: fwd / loss / bwd; deep32k and wide: fwd / bwd)
set -u
O=gpurun_out/${1:-r2fn}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100|loss_cluster|loss_pipe' \
  --launch-skip 12 --launch-count 4 -o $O/full_agentic8k -f \
  python bench.py --config agentic8k --steps 1 --warmup 3 --no-extras > $O/ncu_a8k.log 2>&1
for c in deep32k wide; do
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:'tree_attn_fwd_sm100|tree_attn_bwd_sm100' \
  --launch-skip 6 --launch-count 2 -o $O/full_$c -f \
  python bench.py --config $c --steps 1 --warmup 3 --no-extras --no-loss > $O/ncu_$c.log 2>&1
done
echo done > $O/done.txt
