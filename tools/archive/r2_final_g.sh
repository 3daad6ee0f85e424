# round-2 third-session check: full GPU suite, smoke, sanitizers over the persistent attention kernels,
# driver-style bench lines (default batch64k + agentic8k / deep32k / wide), reference arm
set -u
O=gpurun_out/${1:-r2g_final}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv > $O/smi.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q --durations=10 > $O/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
for tool in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_attn.py -x -q -k "one_partial_block or exactly_128 or fused_sqnorm or bf16" > $O/attn_$tool.txt 2>&1; echo "exit $?" >> $O/attn_$tool.txt
done
timeout 1500 python bench.py --steps 20 --warmup 5 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
for c in agentic8k deep32k wide; do
  timeout 600 python bench.py --config $c --steps 20 --warmup 5 --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
echo done > $O/done.txt
