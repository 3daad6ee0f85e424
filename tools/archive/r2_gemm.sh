set -u
O=gpurun_out/${1:-r2gemm}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
timeout 300 python -m pytest tests/test_gpu_gemm.py -x -q > $O/pytest_gemm.log 2>&1; echo "exit $?" >> $O/pytest_gemm.log
timeout 300 python -m pytest tests/test_gpu_lmhead.py -x -q > $O/pytest_lmhead.log 2>&1; echo "exit $?" >> $O/pytest_lmhead.log
timeout 300 python tools/timegemm.py > $O/timegemm.txt 2>&1
echo done
