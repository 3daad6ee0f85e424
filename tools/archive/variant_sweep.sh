cp paper_2511_00413_b200/libtt.so /tmp/libtt_orig.so
for v in tools/variants/libtt_*.so; do
  cp $v paper_2511_00413_b200/libtt.so
  echo "== $v"; timeout 100 python tools/timeall.py deep32k agentic8k wide 2>&1 | grep -o "^[a-z0-9]*: N=[0-9]*.*bwd [0-9.]* ms ([0-9]* TF/s)"
done
cp /tmp/libtt_orig.so paper_2511_00413_b200/libtt.so
