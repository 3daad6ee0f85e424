set -u
O=gpurun_out/${1:-persab}; mkdir -p $O
python -m paper_2511_00413_b200.build > $O/build.log 2>&1
for r in 1 2; do
echo "== persistent run $r" >> $O/time.txt; timeout 300 python tools/timeall.py deep32k agentic8k wide >> $O/time.txt 2>&1
done
cp paper_2511_00413_b200/csrc/attn_sm100_bwd.cu /tmp/pers.cu
cp tools/attn_sm100_bwd_nonpersistent.cu.txt paper_2511_00413_b200/csrc/attn_sm100_bwd.cu
python -m paper_2511_00413_b200.build >> $O/build.log 2>&1
for r in 1 2; do
echo "== non-persistent run $r" >> $O/time.txt; timeout 300 python tools/timeall.py deep32k agentic8k wide >> $O/time.txt 2>&1
done
cp /tmp/pers.cu paper_2511_00413_b200/csrc/attn_sm100_bwd.cu
echo done
