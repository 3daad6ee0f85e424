set -u
O=gpurun_out/${1:-r2ae}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_attn.py tests/test_gpu_persistent.py tests/test_gpu_multirank_bench.py tests/test_gpu_bench_records.py -m gpu -q > $O/pytest.log 2>&1; echo "exit $?" >> $O/pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke exit $?" >> $O/smoke.log
echo done > $O/done.txt
