# bench lines: default (batch64k) + optional configs; gemm tests + timing
set -u
O=gpurun_out/${1:-r2b}; shift || true
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_lmhead.py tests/test_gpu_block.py -x -q > $O/pytest_some.log 2>&1; echo "exit $?" >> $O/pytest_some.log
timeout 1200 python bench.py --steps 5 --warmup 3 > $O/bench_batch64k.json 2> $O/bench_batch64k.err
for c in "$@"; do timeout 600 python bench.py --config $c --no-cpu > $O/bench_$c.json 2> $O/bench_$c.err; done
echo done
