set -u
O=gpurun_out/lmrep8; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
timeout 600 python -m pytest tests -m gpu -x -q -k lmhead > $O/a.txt 2>&1
timeout 600 python -m pytest tests/test_gpu_lmhead.py tests/test_multi_rank.py -x -q -k "lmhead" > $O/b.txt 2>&1
timeout 600 python -m pytest tests/test_multi_rank.py tests/test_gpu_lmhead.py -x -q > $O/c.txt 2>&1
timeout 600 python -m pytest tests/test_oracle_lmhead.py tests/test_gpu_lmhead.py -x -q > $O/d.txt 2>&1
echo done
