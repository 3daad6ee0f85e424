# compute-sanitizer over the round-2 code: tcgen05 GEMM + LM head, pack (forest scan, staging ring,
# capture refusal), bench records, the root-key star case
set -u
O=gpurun_out/${1:-r2san}; mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_lmhead.py -x -q -k "not 2048" > $O/gemm_$tool.txt 2>&1; echo "exit $?" >> $O/gemm_$tool.txt
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_pack.py tests/test_gpu_bench_records.py -x -q > $O/pack_$tool.txt 2>&1; echo "exit $?" >> $O/pack_$tool.txt
done
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 --error-exitcode 9 python -m pytest tests/test_gpu_rope_none.py tests/test_gpu_block.py -x -q > $O/block_memcheck.txt 2>&1; echo "exit $?" >> $O/block_memcheck.txt
echo done
