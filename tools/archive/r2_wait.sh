set -u
O=gpurun_out/${1:-r2wait}; mkdir -p $O
python -m paper_2511_00413_b200.build --dev --force > $O/build.log 2>&1
for rep in 1 2; do for w in 0 1 2; do TT_GEMM_WAIT=$w timeout 120 python tools/gemm_sustained.py >> $O/sustained.txt 2>&1; done; done
timeout 120 python tools/gemm_sustained.py --cublas >> $O/sustained.txt 2>&1
python -m paper_2511_00413_b200.build --force >> $O/build.log 2>&1
echo done
